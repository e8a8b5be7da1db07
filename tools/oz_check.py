"""Accuracy and speed of the int8-slice (Ozaki) FP64 GEMM against a torch f64
reference:  XB_GEMM_OZ=1 python tools/oz_check.py"""

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
    tag = f"oz={os.environ.get('XB_GEMM_OZ')} S={os.environ.get('XB_OZ_SLICES', 6)}"
    for M, N, K, trans in [(128, 64, 32, False), (200, 70, 100, False), (300, 30, 520, True),
                           (1000, 120, 3000, False), (1000, 120, 3000, True),
                           (65536, 120, 16384, False), (16384, 120, 65536, True)]:
        a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float64)
        b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float64)
        c = torch.empty(M, N, device="cuda", dtype=torch.float64)
        lda = a.shape[1]
        ctx.gemm_dev(np.float64, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ctx.gemm_dev(np.float64, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N,
                         c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        ref = (a.T if trans else a) @ b
        scale = ((a.abs().T if trans else a.abs()) @ b.abs())
        err = (c - ref).abs()
        rel = float((err / scale).max())
        print(f"{tag} {'TN' if trans else 'NN'} {M}x{N}x{K}: err/(|A||B|) max {rel:.2e}, "
              f"max_abs {err.max().item():.2e}, {dt * 1e3:.2f} ms, {2 * M * N * K / dt / 1e12:.1f} TF/s",
              flush=True)
        del a, b, c, ref, scale, err
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
