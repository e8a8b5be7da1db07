"""Quick numerics + speed check of the float32 GEMM path (tcgen05 3xTF32),
run on the GPU box with a short timeout:  python tools/check_tgemm.py"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    rng = np.random.default_rng(0)
    shapes = [(128, 64, 32), (300, 30, 520), (1000, 120, 3000), (777, 224, 999), (4096, 552, 3000),
              (129, 200, 65)]
    for m, n, k in shapes:
        for trans in (False, True):
            a = rng.standard_normal((k, m) if trans else (m, k)).astype(np.float32)
            b = rng.standard_normal((k, n)).astype(np.float32)
            t0 = time.perf_counter()
            got = ctx.gemm(a, b, trans_a=trans)
            dt = time.perf_counter() - t0
            ref = (a.T if trans else a).astype(np.float64) @ b.astype(np.float64)
            err = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), np.sqrt(k)))
            print(f"m={m} n={n} k={k} trans={trans} rel_err={err:.2e} ({dt*1e3:.1f} ms)", flush=True)
    # throughput on a cfg5-like product
    import torch

    for trans in (False, True):
        M, N, K = (16384, 552, 262144) if not trans else (262144, 552, 16384)
        a = torch.randn((K, M) if trans else (M, K), device="cuda", dtype=torch.float32)
        b = torch.randn(K, N, device="cuda", dtype=torch.float32)
        c = torch.empty(M, N, device="cuda", dtype=torch.float32)
        lda = a.shape[1]
        for _ in range(2):
            ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N,
                         c.data_ptr(), N)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N,
                         c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        ref = (a.T if trans else a).double() @ b.double()
        err = float(((c.double() - ref).abs().max() / ref.abs().max()).item())
        print(f"{'TN' if trans else 'NN'} {M}x{N}x{K}: {dt*1e3:.1f} ms, "
              f"{2*M*N*K/dt/1e12:.1f} TF/s (useful), rel_err {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
