"""tcgen05 kernel: product error and time vs XB_TG_DRAIN / XB_TG_CHAIN (set in the env)."""

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
    tag = f"drain={os.environ.get('XB_TG_DRAIN')} chain={os.environ.get('XB_TG_CHAIN')}"
    for M, N, K, trans in [(300, 30, 520, False), (1000, 120, 3000, True), (4096, 224, 65536, False),
                           (2048, 552, 262144, False), (16384, 552, 262144, False),
                           (262144, 552, 16384, True)]:
        a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g)
        b = torch.randn(K, N, device="cuda", generator=g)
        c = torch.empty(M, N, device="cuda")
        lda = a.shape[1]
        ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N, c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        ad = a.double()
        ref = (ad.T if trans else ad) @ b.double()
        err = (c.double() - ref).abs()
        norm = float((err / torch.clamp(ref.abs(), min=K ** 0.5)).max())
        # f32 round-to-nearest reference (cuBLAS SGEMM without TF32)
        torch.backends.cuda.matmul.allow_tf32 = False
        s32 = ((a.T if trans else a) @ b).double()
        e32 = float(((s32 - ref).abs() / torch.clamp(ref.abs(), min=K ** 0.5)).max())
        print(f"{tag} {'TN' if trans else 'NN'} {M}x{N}x{K}: norm_err={norm:.2e} (sgemm {e32:.2e}) "
              f"mean_abs={err.mean().item():.2e} {dt*1e3:.2f} ms {2*M*N*K/dt/1e12:.0f} TF/s", flush=True)
        del a, b, c, ad, ref, err, s32
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
