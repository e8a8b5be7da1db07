"""tcgen05 kernel diagnostics: isolate multi-CTA vs multi-k-tile effects."""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    rng = np.random.default_rng(1)
    for m, k, n in [(128, 64, 64), (256, 32, 64), (256, 64, 64), (128, 96, 64), (384, 32, 64)]:
        for trial in range(2):
            a = rng.standard_normal((m, k)).astype(np.float32)
            b = rng.standard_normal((k, n)).astype(np.float32)
            at = a if os.environ.get("RAWA") else (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
            got = ctx.gemm(at, b)
            ref = at.astype(np.float64) @ b.astype(np.float64)
            e = np.abs(got - ref)
            per_tile = [float(e[i * 128:(i + 1) * 128].max()) for i in range(m // 128)]
            print(f"mode={os.environ.get('XB_TG_MODE')} m={m} k={k} trial={trial} "
                  f"err per m-tile={['%.1e' % x for x in per_tile]}", flush=True)


if __name__ == "__main__":
    main()
