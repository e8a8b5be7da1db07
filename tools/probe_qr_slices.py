"""Accuracy probe for the f32 configs' n-side QR products on the int8 pipe
(oz_gemm64) at a reduced slice count: run under XB_OZ_QR_SLICES=S (3..6)
and compare one cfg5-like factorisation with the CPU oracle.

    XB_OZ_QR_SLICES=4 python tools/probe_qr_slices.py

n*l must be >= 2^24 for the n-side products to take the int8 path, so the
shape is wider than tests/test_gpu_f32_large_l.py's cfg5-like case. Prints
one JSON line: sigma relative error and sine angles of U, V (north star
float32 targets 1e-4 / 1e-3).
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import metrics as M  # noqa: E402
from oracle import pipeline as OP  # noqa: E402
from paper_1907_06470_b200 import _lib  # noqa: E402
from paper_1907_06470_b200.workloads import dense_lowrank_np  # noqa: E402


def main():
    m, n, k, p, q = 2048, 65536, 500, 50, 3
    a = dense_lowrank_np(m, n, "inv", 1e-4, 1005, 2005, 1000, np.float32)
    lib = _lib.load()
    u, s, v, _, _ = lib.rsvd_dense(a, k, p, q, 5)
    ref = OP.rsvd_reorth(a, k, p, q, 5, "single", fast=True)
    print(json.dumps({"slices": os.environ.get("XB_OZ_QR_SLICES", "default"),
                      "shape": [m, n], "sigma_rel": float(M.sigma_rel(s, ref.s)),
                      "angle_u": float(M.sin_angle(u, ref.u)),
                      "angle_v": float(M.sin_angle(v, ref.v))}))


if __name__ == "__main__":
    main()
