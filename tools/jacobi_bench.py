"""Small-SVD (CholQR2 of B^T + Jacobi) timing and accuracy vs numpy, per l.
XB_JACOBI=single|coop|pairs selects the Jacobi variant.

    python tools/jacobi_bench.py 120 220 552
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_1907_06470_b200 import _lib

    ctx = _lib.load(0)
    for l in [int(x) for x in sys.argv[1:]] or [120, 220, 552]:
        rng = np.random.default_rng(l)
        n = 8 * l
        b = (rng.standard_normal((l, l)) * np.logspace(0, -3, l)) @ np.linalg.qr(
            rng.standard_normal((n, l)))[0].T
        ctx.svd_small(b)
        t0 = time.perf_counter()
        u, s, v = ctx.svd_small(b)
        dt = time.perf_counter() - t0
        s_ref = np.linalg.svd(b, compute_uv=False)
        rel = np.max(np.abs(s - s_ref) / s_ref[0])
        orth = np.max(np.abs(u.T @ u - np.eye(l)))
        rec = np.max(np.abs((u * s) @ v.T - b)) / s_ref[0]
        print(f"jacobi={os.environ.get('XB_JACOBI', 'auto')} l={l}: {dt * 1e3:.2f} ms  "
              f"sigma_rel={rel:.1e} orth={orth:.1e} recon={rec:.1e}", flush=True)


if __name__ == "__main__":
    main()
