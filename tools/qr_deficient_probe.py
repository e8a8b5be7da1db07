"""Probe: R diagonal and deficient columns of the device thin QR for an exactly
dependent column (tests/test_gpu_reference_suite.py)."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
from paper_1907_06470_b200 import _lib
ctx = _lib.load(0)
rng = np.random.default_rng(1)
a = rng.standard_normal((30, 6)); a[:, 3] = 2.0 * a[:, 1] - a[:, 0]
q, r, d = ctx.thin_qr(a)
print("diag", np.abs(np.diag(r)), "thr", np.finfo(float).eps * np.linalg.norm(r), "def", d)
