"""One float32 product through the tcgen05 path, for ncu captures.

    python tools/tgemm_one.py --m 16384 --n 552 --k 262144 [--trans]
"""

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--n", type=int, default=552)
    ap.add_argument("--k", type=int, default=262144)
    ap.add_argument("--trans", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pad", type=int, default=0, help="extra elements per row of A (lda)")
    ap.add_argument("--f64", action="store_true", help="float64 A (the DMMA path)")
    args = ap.parse_args()
    import torch

    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    M, N, K = args.m, args.n, args.k
    rows, cols = (K, M) if args.trans else (M, K)
    dt = torch.float64 if args.f64 else torch.float32
    a = torch.randn(rows, cols + args.pad, device="cuda", dtype=dt)[:, :cols]
    b = torch.randn(K, N, device="cuda", dtype=dt)
    c = torch.empty(M, N, device="cuda", dtype=dt)
    lda = a.stride(0)
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.gemm_dev(np.float64 if args.f64 else np.float32, args.trans, M, N, K, a.data_ptr(), lda, b.data_ptr(), N,
                     c.data_ptr(), N)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{'TN' if args.trans else 'NN'} {M}x{N}x{K}: {dt * 1e3:.2f} ms "
              f"{2 * M * N * K / dt / 1e12:.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
