"""Where does the cfg3 host-COO call (xb_rsvd_coo) spend its time?
python tools/coo_e2e_probe.py   (XB_TRACE=1 for the library's own lines)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_06470_b200 import _lib  # noqa: E402
from paper_1907_06470_b200.workloads import CONFIGS, sparse_uniform_np  # noqa: E402

w = CONFIGS[3]
ctx = _lib.load(0)
rowptr, col, val = sparse_uniform_np(w.m, w.n, 20, 3003)
rows = np.repeat(np.arange(w.m, dtype=np.int64), np.diff(rowptr))
cols = col.astype(np.int64)
for i in range(3):
    t0 = time.perf_counter()
    r, c, v = ctx._coo(rows, cols, val)
    t1 = time.perf_counter()
    out = ctx.rsvd_coo(rows, cols, val, (w.m, w.n), w.k, w.p, w.q, w.cfg)
    t2 = time.perf_counter()
    print(f"_coo {t1 - t0:.3f} s, rsvd_coo {t2 - t1:.3f} s, stages {np.round(out[4], 4).tolist()} "
          f"sum {out[4].sum():.3f}", flush=True)
