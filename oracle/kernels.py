"""Block kernels restated on plain arrays — TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/xsvd/kernels.py on in-memory numpy arrays
(the reference's StoredMatrix/BlockPool indirection only moves bytes; the
arithmetic sequence is what is restated here):

  block_multiply      kernels.py:145-193 + _cell_accumulate 71-112
                      (256x256 output cells, k-chunks ascending, acc in the
                      compute dtype, stored at the storage dtype)
  thin_qr             kernels.py:297-351 (+ _house 247-266,
                      _householder_qr 269-282, _apply_reflectors 285-294)
  svd_small           kernels.py:542-562 (+ _bidiagonalize 373-409,
                      _gk_step 412-449, chases 452-476, _bidiagonal_svd
                      479-523, _svd_tall 526-539)

`*_fast` variants use LAPACK/one-shot BLAS instead of the cell walk; they
agree with the restatement to ~1e-15 relative (checked in the oracle tests)
and are what the large parity cases use.
"""

from __future__ import annotations

import math

import numpy as np

CELL = 256  # CANONICAL_CELL, src/core.py:23


class OracleShapeError(ValueError):
    pass


class OracleConvergenceError(RuntimeError):
    pass


def _spans(extent: int, step: int = CELL):
    return [(lo, min(extent, lo + step)) for lo in range(0, extent, step)]


# -- multiply ---------------------------------------------------------------


def block_multiply(x: np.ndarray, y: np.ndarray, cdt, out_dtype, threads: int = 1) -> np.ndarray:
    """Dense x dense on the canonical cell grid (kernels.py:80-84, 172-193).

    `threads` > 1 runs output cells on a thread pool like the reference's
    _run_tasks (kernels.py:231-236); each cell's k-chunks stay in ascending
    order, so the bits do not depend on the thread count."""
    m, k = x.shape
    k2, n = y.shape
    if k != k2:
        raise OracleShapeError(f"inner dimensions disagree: {x.shape} x {y.shape}")
    out = np.empty((m, n), dtype=out_dtype)
    kk = _spans(k)

    def cell(task):
        r0, r1, c0, c1 = task
        acc = np.zeros((r1 - r0, c1 - c0), dtype=cdt)
        for k0, k1 in kk:
            a = np.ascontiguousarray(x[r0:r1, k0:k1]).astype(cdt)
            b = np.ascontiguousarray(y[k0:k1, c0:c1]).astype(cdt)
            acc += a @ b
        out[r0:r1, c0:c1] = acc.astype(out_dtype)

    tasks = [(r0, r1, c0, c1) for r0, r1 in _spans(m) for c0, c1 in _spans(n)]
    if threads <= 1 or len(tasks) <= 1:
        for t in tasks:
            cell(t)
    else:
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        # the reference's fast mode: cell threads with OPENBLAS_NUM_THREADS=1
        # (SURVEY §8d); avoids oversubscribing cores with nested BLAS threads
        with threadpool_limits(limits=1, user_api="blas"):
            with ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(cell, tasks))
    return out


def sparse_dense_multiply(rows, cols, vals, shape, y, cdt, out_dtype) -> np.ndarray:
    """Sparse x dense (kernels.py:85-97): per cell, entries sorted by
    (row, col) (pool.py:420-445), np.add.at in 8192-entry chunks."""
    m, k = shape
    k2, n = y.shape
    if k != k2:
        raise OracleShapeError(f"inner dimensions disagree: {shape} x {y.shape}")
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], np.asarray(vals)[order]
    out = np.empty((m, n), dtype=out_dtype)
    kk = _spans(k)
    for r0, r1 in _spans(m):
        lo, hi = np.searchsorted(rows, r0), np.searchsorted(rows, r1)
        br, bc, bv = rows[lo:hi], cols[lo:hi], vals[lo:hi]
        for c0, c1 in _spans(n):
            acc = np.zeros((r1 - r0, c1 - c0), dtype=cdt)
            for k0, k1 in kk:
                mask = (bc >= k0) & (bc < k1)
                er, ek, ev = br[mask], bc[mask], bv[mask]
                if len(ev) == 0:
                    continue
                b = np.ascontiguousarray(y[k0:k1, c0:c1]).astype(cdt)
                ev = ev.astype(cdt)
                er = er - r0
                ek = ek - k0
                for s in range(0, len(ev), 8192):
                    sl = slice(s, s + 8192)
                    np.add.at(acc, er[sl], ev[sl, None] * b[ek[sl], :])
            out[r0:r1, c0:c1] = acc.astype(out_dtype)
    return out


def block_multiply_fast(x, y, cdt, out_dtype) -> np.ndarray:
    """One-shot BLAS product in the compute dtype (not cell-ordered)."""
    return (np.asarray(x).astype(cdt, copy=False) @ np.asarray(y).astype(cdt, copy=False)).astype(
        out_dtype, copy=False)


# -- thin QR ----------------------------------------------------------------


def _house(x: np.ndarray):
    """Householder vector with v[0]=1 and beta (kernels.py:247-266)."""
    v = np.array(x, dtype=np.float64, copy=True)
    x0 = float(v[0])
    sigma = float(v[1:] @ v[1:])
    v[0] = 1.0
    if sigma == 0.0:
        return v, 0.0 if x0 >= 0.0 else 2.0
    mu = math.sqrt(x0 * x0 + sigma)
    v0 = x0 - mu if x0 <= 0.0 else -sigma / (x0 + mu)
    beta = 2.0 * v0 * v0 / (sigma + v0 * v0)
    v[1:] /= v0
    return v, beta


def _householder_qr(s: np.ndarray):
    """In-place QR (kernels.py:269-282)."""
    rows, r = s.shape
    V = np.zeros((rows, r), dtype=s.dtype)
    betas = np.zeros(r, dtype=np.float64)
    for j in range(min(r, rows)):
        v, beta = _house(s[j:, j])
        V[j:, j] = v
        betas[j] = beta
        if beta != 0.0:
            w = beta * (v @ s[j:, j:])
            s[j:, j:] -= np.outer(v, w)
    return np.triu(s[:r, :r]).copy(), V, betas


def _apply_reflectors(V, betas, m):
    """m <- H_0 ... H_{r-1} m (kernels.py:285-294)."""
    for j in range(V.shape[1] - 1, -1, -1):
        beta = betas[j]
        if beta == 0.0:
            continue
        v = V[j:, j]
        w = beta * (v @ m[j:, :])
        m[j:, :] -= np.outer(v, w)
    return m


def thin_qr(y: np.ndarray, storage_dtype, compute_dtype):
    """Streaming panel Householder QR in f64 (kernels.py:297-351).

    Returns (Q at storage dtype, R f64, deficient column tuple)."""
    m, r = y.shape
    if m < r or r < 1:
        raise OracleShapeError(f"thin QR needs rows >= cols >= 1, got {m}x{r}")
    spans = _spans(m, max(r, CELL))
    R = None
    stashes = []
    for p0, p1 in spans:
        w = np.asarray(y[p0:p1, :]).astype(np.float64)
        stacked = w if R is None else np.vstack([R, w])
        R, V, betas = _householder_qr(stacked)
        stashes.append((V, betas))
    norm = float(np.sqrt(np.sum(R * R)))
    eps = float(np.finfo(compute_dtype).eps)
    deficient = tuple(i for i in range(r) if abs(float(R[i, i])) <= eps * norm)
    q = np.empty((m, r), dtype=storage_dtype)
    carry = np.eye(r)
    for idx in range(len(spans) - 1, -1, -1):
        p0, p1 = spans[idx]
        V, betas = stashes[idx]
        mbuf = np.zeros((V.shape[0], r))
        mbuf[:r, :] = carry
        g = _apply_reflectors(V, betas, mbuf)
        if idx == 0:
            q[p0:p1] = g.astype(storage_dtype)
        else:
            carry = g[:r, :].copy()
            q[p0:p1] = g[r:, :].astype(storage_dtype)
    return q, R, deficient


def thin_qr_fast(y: np.ndarray, storage_dtype, compute_dtype):
    """LAPACK QR with the reference's sign convention (diag R >= 0)."""
    m, r = y.shape
    if m < r or r < 1:
        raise OracleShapeError(f"thin QR needs rows >= cols >= 1, got {m}x{r}")
    q, R = np.linalg.qr(np.asarray(y, dtype=np.float64))
    sgn = np.where(np.diag(R) < 0, -1.0, 1.0)
    q = q * sgn
    R = R * sgn[:, None]
    norm = float(np.sqrt(np.sum(R * R)))
    eps = float(np.finfo(compute_dtype).eps)
    deficient = tuple(i for i in range(r) if abs(float(R[i, i])) <= eps * norm)
    return q.astype(storage_dtype), R, deficient


# -- small SVD ----------------------------------------------------------------


def _rot(f, g):
    if g == 0.0:
        return 1.0, 0.0, f
    if f == 0.0:
        return 0.0, 1.0, g
    r = math.hypot(f, g)
    return f / r, g / r, r


def _rot_cols(m, i, j, c, s):
    ci = c * m[:, i] + s * m[:, j]
    m[:, j] = -s * m[:, i] + c * m[:, j]
    m[:, i] = ci


def _bidiagonalize(a):
    """Householder bidiagonalization (kernels.py:373-409)."""
    a = a.astype(np.float64, copy=True)
    m, n = a.shape
    left, right = [], []
    for k in range(n):
        v, beta = _house(a[k:, k])
        left.append((v, beta))
        if beta != 0.0:
            w = beta * (v @ a[k:, k:])
            a[k:, k:] -= np.outer(v, w)
        if k < n - 2:
            v, beta = _house(a[k, k + 1:])
            right.append((v, beta))
            if beta != 0.0:
                w = beta * (a[k:, k + 1:] @ v)
                a[k:, k + 1:] -= np.outer(w, v)
    d = np.diagonal(a).copy()
    e = np.diagonal(a, offset=1).copy() if n > 1 else np.empty(0)
    u = np.eye(m, n)
    for k in range(n - 1, -1, -1):
        v, beta = left[k]
        if beta != 0.0:
            w = beta * (v @ u[k:, k:])
            u[k:, k:] -= np.outer(v, w)
    vmat = np.eye(n)
    for k in range(len(right) - 1, -1, -1):
        v, beta = right[k]
        if beta != 0.0:
            w = beta * (v @ vmat[k + 1:, k + 1:])
            vmat[k + 1:, k + 1:] -= np.outer(v, w)
    return u, d, e, vmat


def _gk_step(d, e, p, q, u_rot, v_rot):
    """Implicit-shift bidiagonal QR sweep (kernels.py:412-449)."""
    dm, dn = float(d[q - 1]), float(d[q])
    em = float(e[q - 1])
    em1 = float(e[q - 2]) if q - 1 > p else 0.0
    t11 = dm * dm + em1 * em1
    t12 = dm * em
    t22 = dn * dn + em * em
    delta = 0.5 * (t11 - t22)
    if delta == 0.0 and t12 == 0.0:
        mu = t22
    else:
        denom = delta + math.copysign(math.hypot(delta, t12), delta if delta != 0.0 else 1.0)
        mu = t22 - (t12 * t12) / denom if denom != 0.0 else t22
    y = float(d[p]) * float(d[p]) - mu
    z = float(d[p]) * float(e[p])
    for k in range(p, q):
        c, s, r = _rot(y, z)
        if k > p:
            e[k - 1] = r
        f = c * d[k] + s * e[k]
        e[k] = c * e[k] - s * d[k]
        g = s * d[k + 1]
        d[k + 1] = c * d[k + 1]
        d[k] = f
        _rot_cols(v_rot, k, k + 1, c, s)
        c, s, r = _rot(float(d[k]), float(g))
        d[k] = r
        f = c * e[k] + s * d[k + 1]
        d[k + 1] = c * d[k + 1] - s * e[k]
        e[k] = f
        if k < q - 1:
            g = s * e[k + 1]
            e[k + 1] = c * e[k + 1]
        _rot_cols(u_rot, k, k + 1, c, s)
        if k < q - 1:
            y = float(e[k])
            z = float(g)


def _zero_row_chase(d, e, k, q, u_rot):
    """kernels.py:452-463."""
    f = float(e[k])
    e[k] = 0.0
    for j in range(k + 1, q + 1):
        c, s, r = _rot(float(d[j]), f)
        d[j] = r
        _rot_cols(u_rot, j, k, c, s)
        if j < q:
            f = -s * float(e[j])
            e[j] = c * float(e[j])


def _zero_col_chase(d, e, p, q, v_rot):
    """kernels.py:466-476."""
    f = float(e[q - 1])
    e[q - 1] = 0.0
    for j in range(q - 1, p - 1, -1):
        c, s, r = _rot(float(d[j]), f)
        d[j] = r
        _rot_cols(v_rot, j, q, c, s)
        if j > p:
            f = -s * float(e[j - 1])
            e[j - 1] = c * float(e[j - 1])


def _bidiagonal_svd(d, e, eps):
    """kernels.py:479-523."""
    n = len(d)
    d = d.astype(np.float64, copy=True)
    e = e.astype(np.float64, copy=True)
    u_rot = np.eye(n)
    v_rot = np.eye(n)
    if n == 1:
        return d, u_rot, v_rot
    anorm = float(np.max(np.abs(d))) + (float(np.max(np.abs(e))) if len(e) else 0.0)
    max_steps = 30 * n
    steps = 0
    while True:
        for i in range(n - 1):
            if abs(e[i]) <= eps * (abs(d[i]) + abs(d[i + 1])):
                e[i] = 0.0
        q = n - 1
        while q > 0 and e[q - 1] == 0.0:
            q -= 1
        if q == 0:
            break
        p = q - 1
        while p > 0 and e[p - 1] != 0.0:
            p -= 1
        if anorm > 0.0:
            zeroed = False
            for k in range(p, q):
                if abs(d[k]) <= eps * anorm:
                    _zero_row_chase(d, e, k, q, u_rot)
                    zeroed = True
                    break
            if zeroed:
                continue
            if abs(d[q]) <= eps * anorm:
                _zero_col_chase(d, e, p, q, v_rot)
                continue
        steps += 1
        if steps > max_steps:
            raise OracleConvergenceError(f"bidiagonal SVD did not converge in {max_steps} sweeps")
        _gk_step(d, e, p, q, u_rot, v_rot)
    return d, u_rot, v_rot


def _svd_tall(a):
    """kernels.py:526-539."""
    u0, d, e, v0 = _bidiagonalize(a)
    s, u_rot, v_rot = _bidiagonal_svd(d, e, float(np.finfo(np.float64).eps))
    neg = s < 0
    s = np.abs(s)
    u_rot[:, neg] = -u_rot[:, neg]
    order = np.argsort(-s, kind="stable")
    return u0 @ u_rot[:, order], s[order], v0 @ v_rot[:, order]


def sign_fix(u, v):
    """Largest-|entry| of each U column positive, earliest row on ties;
    the matching V column flips with it (kernels.py:556-561)."""
    for j in range(u.shape[1]):
        i = int(np.argmax(np.abs(u[:, j])))
        if u[i, j] < 0:
            u[:, j] = -u[:, j]
            v[:, j] = -v[:, j]
    return u, v


def svd_small(b: np.ndarray):
    """B (r x n, r <= n) = U diag(s) V^T (kernels.py:542-562)."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2:
        raise OracleShapeError(f"svd_small expects a matrix, got shape {b.shape}")
    r, n = b.shape
    if r > n:
        raise OracleShapeError(f"svd_small expects r <= n, got {r}x{n}")
    ut, s, vt = _svd_tall(b.T.copy())
    u, v = sign_fix(vt, ut)
    return u, s, v


def svd_small_fast(b: np.ndarray):
    """LAPACK SVD with the same sign rule."""
    b = np.asarray(b, dtype=np.float64)
    r, n = b.shape
    if r > n:
        raise OracleShapeError(f"svd_small expects r <= n, got {r}x{n}")
    u, s, vt = np.linalg.svd(b, full_matrices=False)
    u, v = sign_fix(u.copy(), vt.T.copy())
    return u, s, v
