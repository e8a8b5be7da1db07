"""float32 A on the int8 pipe (ozf_gemm, XB_GEMM_OZF=1) vs torch f64 and the
default 3xTF32 path:  XB_GEMM_OZF=1 python tools/ozf_check.py"""

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
    tag = f"ozf={os.environ.get('XB_GEMM_OZF')}"
    shapes = [(128, 64, 32, False), (300, 120, 1000, True), (1000, 552, 3000, False),
              (2000, 220, 5000, True), (16384, 552, 262144, False), (262144, 552, 16384, True)]
    for M, N, K, trans in shapes:
        a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float32)
        b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32) / np.sqrt(K)
        c = torch.empty(M, N, device="cuda", dtype=torch.float32)
        lda = a.shape[1]
        ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        reps = 3 if M * K < 1e10 else 2
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N,
                         c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        a64, b64 = a.double(), b.double()
        op = a64.T if trans else a64
        ref = op @ b64
        scale = op.abs() @ b64.abs()
        err = float(((c.double() - ref).abs() / scale).max())
        rel = float((c.double() - ref).norm() / ref.norm())
        print(f"{tag} {'TN' if trans else 'NN'} {M}x{N}x{K}: err/(|A||B|) {err:.2e} "
              f"fro-rel {rel:.2e}  {dt * 1e3:.2f} ms {2 * M * N * K / dt / 1e12:.1f} TF/s",
              flush=True)
        del a, b, c, a64, b64, op, ref, scale
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
