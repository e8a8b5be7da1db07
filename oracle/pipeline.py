"""rSVD drivers restated on arrays — TEST INFRASTRUCTURE ONLY.

  randomized_svd   the SHIPPED reference driver, src/pipeline.py:442-625
                   (fixed power, gram_path=False): 2q+1 raw products, one
                   thin_qr, projection B = Q^T A, svd_small, U = Q U_B.
  rsvd_reorth      "xsvd-reorth": the same Omega and the
                   reference primitives, with thin_qr after EVERY product —
                   the oracle for configs 2-5, where the north star asks for
                   re-orthonormalisation (the shipped driver does not
                   re-orthonormalise, src/pipeline.py:321-371).

Operands: A is either a dense ndarray (m x n) or a `Coo` (rows, cols, vals,
shape). `precision` is "double" or "single" (src/core.py:26-46: storage
dtype <f8/<f4, compute dtype f64/f32).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import kernels as K
from .rng import gaussian_band

STORAGE = {"double": np.float64, "single": np.float32}
COMPUTE = {"double": np.float64, "single": np.float32}


@dataclass
class Coo:
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    shape: tuple

    @property
    def T(self) -> "Coo":
        return Coo(self.cols, self.rows, self.vals, (self.shape[1], self.shape[0]))

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape, dtype=np.asarray(self.vals).dtype)
        np.add.at(out, (np.asarray(self.rows, np.int64), np.asarray(self.cols, np.int64)), self.vals)
        return out


@dataclass
class OracleResult:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray
    deficient_columns: tuple


_THREADS = [1]  # cell workers for the restated block_multiply (set per driver call)


def _mul(x, y, precision, fast):
    """x @ y with the reference's density dispatch (kernels.py:79-112)."""
    cdt, sdt = COMPUTE[precision], STORAGE[precision]
    if isinstance(x, Coo):
        if fast:
            import scipy.sparse as sp

            a = sp.csr_matrix((np.asarray(x.vals, cdt), (x.rows, x.cols)), shape=x.shape)
            return np.asarray(a @ np.asarray(y, cdt)).astype(sdt)
        return K.sparse_dense_multiply(x.rows, x.cols, x.vals, x.shape, y, cdt, sdt)
    if isinstance(y, Coo):
        # dense x sparse (kernels.py:98-112) == (sparse^T x dense^T)^T
        if fast:
            import scipy.sparse as sp

            b = sp.csr_matrix((np.asarray(y.vals, cdt), (y.cols, y.rows)), shape=(y.shape[1], y.shape[0]))
            return np.ascontiguousarray(np.asarray(b @ np.asarray(x, cdt).T).T).astype(sdt)
        return dense_sparse_multiply(x, y, cdt, sdt)
    if fast:
        return K.block_multiply_fast(x, y, cdt, sdt)
    return K.block_multiply(x, y, cdt, sdt, threads=_THREADS[0])


def dense_sparse_multiply(x, y: Coo, cdt, sdt) -> np.ndarray:
    """Dense x sparse per output cell (kernels.py:98-112): entries of the
    sparse cell sorted by (k, c), scattered into acc^T."""
    m, k = x.shape
    k2, n = y.shape
    if k != k2:
        raise K.OracleShapeError(f"inner dimensions disagree: {x.shape} x {y.shape}")
    rows = np.asarray(y.rows, np.int64)
    cols = np.asarray(y.cols, np.int64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], np.asarray(y.vals)[order]
    out = np.empty((m, n), dtype=sdt)
    for r0, r1 in K._spans(m):
        for c0, c1 in K._spans(n):
            acc = np.zeros((r1 - r0, c1 - c0), dtype=cdt)
            acc_t = acc.T
            for k0, k1 in K._spans(k):
                lo, hi = np.searchsorted(rows, k0), np.searchsorted(rows, k1)
                br, bc, bv = rows[lo:hi], cols[lo:hi], vals[lo:hi]
                mask = (bc >= c0) & (bc < c1)
                ek, ec, ev = br[mask], bc[mask], bv[mask]
                if len(ev) == 0:
                    continue
                at = np.ascontiguousarray(x[r0:r1, k0:k1]).astype(cdt).T
                ev = ev.astype(cdt)
                ek = ek - k0
                ec = ec - c0
                for s in range(0, len(ev), 8192):
                    sl = slice(s, s + 8192)
                    np.add.at(acc_t, ec[sl], ev[sl, None] * at[ek[sl], :])
            out[r0:r1, c0:c1] = acc.astype(sdt)
    return out


def _transpose(a):
    return a.T if isinstance(a, Coo) else np.asarray(a).T


def _qr(y, precision, fast):
    sdt, cdt = STORAGE[precision], COMPUTE[precision]
    return (K.thin_qr_fast if fast else K.thin_qr)(y, sdt, cdt)


def _svd(b, fast):
    return (K.svd_small_fast if fast else K.svd_small)(np.asarray(b, dtype=np.float64))


def _check(a, k, p):
    m, n = a.shape
    if k < 1:
        raise ValueError(f"rank must be at least 1, got {k}")
    if k + p > min(m, n):
        raise K.OracleShapeError(f"rank {k} (+{p} oversampling) exceeds min{a.shape} = {min(m, n)}")


def omega(seed: int, n: int, l: int, precision: str) -> np.ndarray:
    """Omega = gaussian_band(seed, 0, n, l) cast to storage (pipeline.py:259-284)."""
    return gaussian_band(seed, 0, n, l).astype(STORAGE[precision])


def randomized_svd(a, k, p, q, seed, precision="double", *, fast=False, om=None,
                   threads: int = 1) -> OracleResult:
    """The shipped driver, src/pipeline.py:442-625 (fixed power)."""
    _THREADS[0] = max(1, int(threads))
    _check(a, k, p)
    m, n = a.shape
    l = k + p
    o = omega(seed, n, l, precision) if om is None else om
    y = _mul(a, o, precision, fast)                      # sketch, 321-330
    for _ in range(q):
        z = _mul(_transpose(a), y, precision, fast)      # power-left, 340-348
        y = _mul(a, z, precision, fast)                  # power-right, 350-360
    qm, _, deficient = _qr(y, precision, fast)           # orthogonalize, 511-523
    b = _mul(qm.T, a, precision, fast)                   # project, 550-553
    u_b, s, v = _svd(b, fast)                            # svd0, 582-591
    u = _mul(qm, u_b[:, :k], precision, fast)            # postprocess, 603-616
    return OracleResult(u, s[:k].astype(np.float64), v[:, :k].astype(STORAGE[precision]), deficient)


def rsvd_reorth(a, k, p, q, seed, precision="double", *, fast=False, om=None,
                threads: int = 1) -> OracleResult:
    """xsvd-reorth: thin_qr after every product."""
    _THREADS[0] = max(1, int(threads))
    _check(a, k, p)
    m, n = a.shape
    l = k + p
    o = omega(seed, n, l, precision) if om is None else om
    qm, _, deficient = _qr(_mul(a, o, precision, fast), precision, fast)
    for _ in range(q):
        qz, _, _ = _qr(_mul(_transpose(a), qm, precision, fast), precision, fast)
        qm, _, deficient = _qr(_mul(a, qz, precision, fast), precision, fast)
    b = _mul(qm.T, a, precision, fast)
    u_b, s, v = _svd(b, fast)
    u = _mul(qm, u_b[:, :k], precision, fast)
    return OracleResult(u, s[:k].astype(np.float64), v[:, :k].astype(STORAGE[precision]), deficient)


def sketch_power_auto(a, k, p, seed, precision="double", *, q_max=5, tau=1e-6, fast=False,
                      om=None):
    """power="auto" of _sketch_and_power (src/pipeline.py:295-372): raw
    products Y = (A A^T)^q A Omega, nu_q = ||Y_q||_F / sqrt(m l); stop when
    nu_q < tau nu_0 or consecutive ratios agree to 1%, or at q_max; a zero
    sketch stops at q = 0. Returns (chosen q, [nu_0, ..., nu_chosen])."""
    _check(a, k, p)
    m, n = a.shape
    l = k + p
    o = omega(seed, n, l, precision) if om is None else om
    scale = 1.0 / np.sqrt(m * l)
    y = _mul(a, o, precision, fast)
    nus = [float(np.sqrt(np.sum(np.asarray(y, dtype=np.float64) ** 2))) * scale]
    if not nus[0] > 0.0:
        return 0, nus
    chosen, prev_rho = 0, 1.0
    for q in range(1, q_max + 1):
        z = _mul(_transpose(a), y, precision, fast)
        y = _mul(a, z, precision, fast)
        chosen = q
        nus.append(float(np.sqrt(np.sum(np.asarray(y, dtype=np.float64) ** 2))) * scale)
        nu = nus[-1]
        if nu < tau * nus[0]:
            break
        rho = nu / nus[q - 1]
        if abs(rho - prev_rho) <= 0.01 * rho:
            break
        prev_rho = rho
    return chosen, nus


def rsvd_reorth_gram(a, k, p, q, seed, precision="double", *, fast=True, om=None):
    """xsvd-reorth range finder + the gram_path projection and small SVD of
    src/pipeline.py:526-580: B^T = (Q^T (A A^T)^q A)^T by 2q raw products,
    G = B B^T, svd_small(G) (eigen-decomposition, sign rule), sigma =
    sqrt(max(eig, 0))^(1/(2q+1)) (q > 0), V = B^T U_B with unit columns."""
    _check(a, k, p)
    m, n = a.shape
    l = k + p
    o = omega(seed, n, l, precision) if om is None else om
    qm, _, deficient = _qr(_mul(a, o, precision, fast), precision, fast)
    for _ in range(q):
        qz, _, _ = _qr(_mul(_transpose(a), qm, precision, fast), precision, fast)
        qm, _, deficient = _qr(_mul(a, qz, precision, fast), precision, fast)
    w = _mul(_transpose(a), qm, precision, fast)             # B^T
    for _ in range(q):
        w = _mul(_transpose(a), _mul(a, w, precision, fast), precision, fast)
    w = np.asarray(w, dtype=np.float64)
    g = w.T @ w
    u_b, eig, _ = _svd(g, fast)
    sig = np.sqrt(np.maximum(eig, 0.0))
    s = sig ** (1.0 / (2 * q + 1)) if q > 0 else sig
    v = w @ u_b
    norms = np.sqrt(np.sum(v * v, axis=0))
    nz = norms > 0
    v[:, nz] /= norms[nz]
    u = _mul(qm, u_b[:, :k], precision, fast)
    return OracleResult(u, s[:k].astype(np.float64), v[:, :k].astype(STORAGE[precision]), deficient)
