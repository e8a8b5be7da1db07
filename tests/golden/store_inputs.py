"""Seeded inputs shared by make_golden_store.py and tests/test_store_*.py
(no dependency on the reference, so the GPU box can rebuild them)."""

import numpy as np


def mtx_text(seed: int, m: int, n: int) -> str:
    """Seeded low-rank dense matrix written as coordinate general real."""
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal((m, 6)) * (0.7 ** np.arange(6))) @ rng.standard_normal((6, n))
    a += 1e-6 * rng.standard_normal((m, n))
    lines = ["%%MatrixMarket matrix coordinate real general", f"{m} {n} {m * n}"]
    for i in range(m):
        for j in range(n):
            lines.append(f"{i + 1} {j + 1} {a[i, j]:.17g}")
    return "\n".join(lines) + "\n"
