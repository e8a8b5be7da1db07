"""Out-of-core streamer on a pageable numpy A (forced streaming of a
cfg2-sized matrix: q + 1 = 3 staged passes).   python tools/stream_probe.py"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    m, n = 65536, 16384
    rng = np.random.default_rng(1)
    a = np.empty((m, n), dtype=np.float32)
    blk = rng.standard_normal((1024, n)).astype(np.float32)
    for r in range(0, m, 1024):
        a[r:r + 1024] = blk
    for i in range(3):
        t0 = time.perf_counter()
        st = ctx.rsvd_dense_streamed(a, 100, 20, 2, 2)[4]
        dt = time.perf_counter() - t0
        print(f"streamed pageable f32 {m}x{n}: {dt:.3f} s, copy stage {st[0]:.3f} s "
              f"({3 * a.nbytes / st[0] / 1e9:.1f} GB/s over 3 passes)", flush=True)


if __name__ == "__main__":
    main()
