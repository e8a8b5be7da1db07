"""Pageable-host ingest through the staging ring (engine.cu HostStager):
xb_rsvd_dense on a pageable numpy A, per worker-thread count (experiment
build: XB_STAGE_THREADS), against a pinned A.

    XB_BUILD_EXPERIMENTS=1 python -m paper_1907_06470_b200.build
    python tools/stage_probe.py [threads ...]
"""

import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one():
    import torch

    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import CONFIGS

    w = CONFIGS[int(os.environ.get("PROBE_CFG", "2"))]
    dt = np.float64 if w.precision == "double" else np.float32
    ctx = _lib.load(0)
    rng = np.random.default_rng(1)
    a = np.empty((w.m, w.n), dtype=dt)
    blk = rng.standard_normal((1024, w.n)).astype(dt)
    for r in range(0, w.m, 1024):
        a[r:r + 1024] = blk[: min(1024, w.m - r)]
    times = []
    for i in range(4):
        t0 = time.perf_counter()
        st = ctx.rsvd_dense(a, w.k, w.p, w.q, w.cfg)[4]
        times.append(time.perf_counter() - t0)
    print(f"threads={os.environ.get('XB_STAGE_THREADS', 'default')} "
          f"slot={os.environ.get('XB_STAGE_SLOT_MB', '64')}MB x{os.environ.get('XB_STAGE_SLOTS', '4')} "
          f"piece={os.environ.get('XB_STAGE_PIECE_KB', '2048')}KB pageable: "
          f"{[round(t, 3) for t in times]} s, ingest stage {st[0]:.3f} s", flush=True)
    if os.environ.get("PROBE_PINNED"):
        hp = torch.empty((w.m, w.n), dtype=torch.float64 if dt == np.float64 else torch.float32,
                         pin_memory=True)
        hp.numpy()[:] = a
        ap = hp.numpy()
        times = []
        for i in range(3):
            t0 = time.perf_counter()
            st = ctx.rsvd_dense(ap, w.k, w.p, w.q, w.cfg)[4]
            times.append(time.perf_counter() - t0)
        print(f"pinned: {[round(t, 3) for t in times]} s, ingest stage {st[0]:.3f} s", flush=True)


if __name__ == "__main__":
    if os.environ.get("PROBE_CHILD"):
        one()
    else:
        print("host cpus:", os.cpu_count(), flush=True)
        # threads:slotMB:slots:pieceKB
        for i, spec in enumerate(sys.argv[1:] or ["16:64:4:2048", "16:8:6:1024", "16:4:8:512",
                                                  "16:16:4:1024", "12:8:6:1024", "15:8:6:512"]):
            t, mb, ns, kb = spec.split(":")
            env = dict(os.environ, PROBE_CHILD="1", XB_STAGE_THREADS=t, XB_STAGE_SLOT_MB=mb,
                       XB_STAGE_SLOTS=ns, XB_STAGE_PIECE_KB=kb)
            if i == 0:
                env["PROBE_PINNED"] = "1"
            subprocess.run([sys.executable, __file__], env=env, check=False)
