"""Parity metrics — TEST INFRASTRUCTURE ONLY.

Sine-form principal angle: for orthonormal X, Y,
sin(theta_max) = ||Y - X (X^T Y)||_2. The arccos(sigma_min(X^T Y)) form
floors near 1.5e-8 in f64, above the 1e-8 target, so it is not used.
"""

import numpy as np


def orthonormal(x: np.ndarray) -> np.ndarray:
    q, _ = np.linalg.qr(np.asarray(x, dtype=np.float64))
    return q


def sin_angle(x: np.ndarray, y: np.ndarray) -> float:
    """Largest principal angle (sine) between range(x) and range(y)."""
    qx, qy = orthonormal(x), orthonormal(y)
    resid = qy - qx @ (qx.T @ qy)
    return float(np.linalg.norm(resid, 2))


def sigma_rel(s: np.ndarray, ref: np.ndarray) -> float:
    """max_i |s_i - ref_i| / ref_i (zero ref_i: relative to ref_0)."""
    s = np.asarray(s, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = np.where(ref > 0, ref, max(float(ref[0]), 1e-300))
    return float(np.max(np.abs(s - ref) / scale))


def sigma_rel_top(s: np.ndarray, ref: np.ndarray) -> float:
    """max_i |s_i - ref_i| / ref_0 (the reference tests' form)."""
    s = np.asarray(s, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(s - ref)) / max(float(ref[0]), 1e-300))


def ortho_defect(q: np.ndarray) -> float:
    q = np.asarray(q, dtype=np.float64)
    return float(np.max(np.abs(q.T @ q - np.eye(q.shape[1]))))
