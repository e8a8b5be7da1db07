"""Times the big cfg5-shaped ozf products (NN 16384x552x262144, TN
262144x552x16384) through gemm_dev with XB_GEMM_OZF=1; meant to run under
ncu -k regex:ozf_kernel with XB_OZF_DBG variants."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for M, N, K, trans in [(16384, 552, 262144, False), (262144, 552, 16384, True)]:
        a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float32)
        b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32)
        c = torch.empty(M, N, device="cuda", dtype=torch.float32)
        for _ in range(2):
            ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), a.shape[1], b.data_ptr(), N,
                         c.data_ptr(), N)
        torch.cuda.synchronize()
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
