"""Diagnostics for the tcgen05 3xTF32 kernel: error per shape and term mode."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    rng = np.random.default_rng(0)
    for m, n, k in [(128, 64, 32), (128, 128, 32), (128, 224, 32), (128, 192, 32), (128, 120, 32),
                    (1000, 120, 3000), (1000, 224, 3000), (128, 256, 32), (256, 64, 64)]:
        a = rng.standard_normal((m, k)).astype(np.float32)
        b = rng.standard_normal((k, n)).astype(np.float32)
        got = ctx.gemm(a, b)
        ref = a.astype(np.float64) @ b.astype(np.float64)
        e = np.abs(got - ref)
        rows = np.unique(np.nonzero(e > 1e-4 * np.sqrt(k))[0])
        cols = np.unique(np.nonzero(e > 1e-4 * np.sqrt(k))[1])
        print(f"mode={os.environ.get('XB_TG_MODE', '3')} m={m} n={n} k={k} "
              f"max_abs={e.max():.2e} bad_rows={rows[:8].tolist()}..{len(rows)} "
              f"bad_cols={cols[:8].tolist()}..{len(cols)}", flush=True)
        # exactly tf32-representable inputs: the hi*hi term alone is exact
        at = (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        bt = (b.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        got2 = ctx.gemm(at, bt)
        ref2 = at.astype(np.float64) @ bt.astype(np.float64)
        print(f"   tf32-exact inputs: max_abs={np.abs(got2 - ref2).max():.2e}", flush=True)


if __name__ == "__main__":
    main()
