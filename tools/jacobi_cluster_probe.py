"""Cluster Jacobi (small.cu jacobi_cluster_kernel) against the single-CTA
kernel and numpy: accuracy over a range of l (odd, tiny, 128) and the
wall time of xb_svd_small per variant (experiment build: XB_JACOBI).

    XB_BUILD_EXPERIMENTS=1 python -m paper_1907_06470_b200.build
    python tools/jacobi_cluster_probe.py
"""

import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LS = [1, 2, 3, 5, 8, 17, 30, 31, 32, 33, 48, 63, 64, 65, 96, 100, 119, 120, 121, 127, 128]


def one():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    worst = 0.0
    for l in LS:
        rng = np.random.default_rng(l)
        n = max(8 * l, 16)
        b = (rng.standard_normal((l, l)) * np.logspace(0, -3, l)) @ np.linalg.qr(
            rng.standard_normal((n, l)))[0].T
        ctx.svd_small(b)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            u, s, v = ctx.svd_small(b)
            ts.append(time.perf_counter() - t0)
        s_ref = np.linalg.svd(b, compute_uv=False)
        rel = np.max(np.abs(s - s_ref) / s_ref[0])
        orth = max(np.max(np.abs(u.T @ u - np.eye(l))), np.max(np.abs(v.T @ v - np.eye(l))))
        rec = np.max(np.abs((u * s) @ v.T - b)) / s_ref[0]
        desc = bool(np.all(np.diff(s) <= 0))
        # sign rule: largest |entry| of every U column positive
        sg = bool(np.all(u[np.argmax(np.abs(u), axis=0), np.arange(l)] > 0))
        worst = max(worst, rel, orth, rec)
        print(f"  l={l:4d}: {min(ts) * 1e3:7.3f} ms  sigma_rel={rel:.1e} orth={orth:.1e} "
              f"recon={rec:.1e} sorted={desc} sign={sg}", flush=True)
        assert desc and sg
    # rank-deficient input: zero singular values, ties
    l = 96
    rng = np.random.default_rng(7)
    b = rng.standard_normal((l, 40)) @ rng.standard_normal((40, 4 * l))
    try:
        u, s, v = ctx.svd_small(b)
    except Exception as e:  # noqa: BLE001
        print("  rank-deficient case raised:", e, flush=True)
        return
    s_ref = np.linalg.svd(b, compute_uv=False)
    print(f"  rank-40 of {l}: sigma err {np.max(np.abs(s - s_ref)) / s_ref[0]:.1e}, "
          f"orth U {np.max(np.abs(u.T @ u - np.eye(l))):.1e}", flush=True)
    print(f"variant {os.environ.get('XB_JACOBI', 'auto')}: worst {worst:.1e}", flush=True)


if __name__ == "__main__":
    if os.environ.get("PROBE_CHILD"):
        one()
    else:
        for var in sys.argv[1:] or ["cluster", "rr"]:
            print(f"XB_JACOBI={var}", flush=True)
            subprocess.run([sys.executable, __file__],
                           env=dict(os.environ, PROBE_CHILD="1", XB_JACOBI=var), check=False)
