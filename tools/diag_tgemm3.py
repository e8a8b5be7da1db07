"""tcgen05 kernel: error vs f32 accumulation chain length (XB_TG_CHAIN)."""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for M, N, K in [(4096, 224, 65536), (2048, 552, 262144)]:
        a = torch.randn(M, K, device="cuda", generator=g)
        b = torch.randn(K, N, device="cuda", generator=g)
        c = torch.empty(M, N, device="cuda")
        ctx.gemm_dev(np.float32, False, M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.gemm_dev(np.float32, False, M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ref = a.double() @ b.double()
        err = (c.double() - ref).abs()
        print(f"chain={os.environ.get('XB_TG_CHAIN')} {M}x{N}x{K}: max_abs={err.max().item():.3e} "
              f"mean_abs={err.mean().item():.3e} bias={(c.double() - ref).mean().item():.2e} "
              f"ref_std={ref.std().item():.1f} {dt*1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
