"""One int8-slice FP64 product (XB_GEMM_OZ=1 path) for ncu captures."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1907_06470_b200 import _lib

    os.environ.setdefault("XB_GEMM_OZ", "1")
    M, N, K = 65536, 120, 16384
    ctx = _lib.load(0)
    a = torch.randn(M, K, device="cuda", dtype=torch.float64)
    b = torch.randn(K, N, device="cuda", dtype=torch.float64)
    c = torch.empty(M, N, device="cuda", dtype=torch.float64)
    for _ in range(2):
        ctx.gemm_dev(np.float64, False, M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
