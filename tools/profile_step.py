"""Run W warm-up + K device-resident factorisations of a config-shaped A, for
ncu launch lists / --set full captures (A is seeded Gaussian: kernel timing
does not depend on the spectrum).

    python tools/profile_step.py --config 2 --warmup 2 --steps 1
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    args = ap.parse_args()
    import torch

    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    ctx = _lib.load(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(w.cfg)
    dt = torch.float64 if w.precision == "double" else torch.float32
    a = torch.randn(w.m, w.n, generator=g, device="cuda", dtype=dt)
    u = torch.empty((w.m, w.k), dtype=dt, device="cuda")
    v = torch.empty((w.n, w.k), dtype=dt, device="cuda")
    s = torch.empty((w.k,), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    import time
    walls = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, stages = ctx.rsvd_dense_dev(np.float64 if w.precision == "double" else np.float32, w.m, w.n, a.data_ptr(), w.n, w.k, w.p, w.q,
                                       w.cfg, u.data_ptr(), s.data_ptr(), v.data_ptr())
        walls.append(round((time.perf_counter() - t0) * 1e3, 3))
    print("wall ms per call", walls)
    print("stage seconds", np.round(stages, 5).tolist(), "launches", ctx.launches)


if __name__ == "__main__":
    main()
