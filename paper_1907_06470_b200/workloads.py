"""Seeded synthetic workloads for the five BASELINE.json configs.

No public dataset is involved: each config's A is built from
seeds with the shape, spectrum and noise BASELINE.json names. Seeds follow
SURVEY.md §8d: A-construction 1000+c, noise 2000+c, CSR pattern 3000+c, and
the Omega seed is RsvdConfig.seed = c. "N(0, x)" noise is read as std x.
Haar factors are Q * sign(diag R) of the QR of an N(0,1) matrix.

Small instances are built in numpy (bit-reproducible on one numpy build);
the large ones (cfg2 upward) are built on the GPU with torch — this is
input generation for tests and the benchmark, not part of the product path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    cfg: int
    m: int
    n: int
    k: int
    p: int
    q: int
    precision: str          # "double" | "single"
    density: str            # "dense" | "sparse"
    spectrum: str           # "geom0.9" | "pow-1.5" | "exp-50" | "inv"
    signal_rank: int | None  # None: full min(m, n) spectrum
    noise: float
    tile: tuple

    @property
    def l(self) -> int:
        return self.k + self.p

    @property
    def name(self) -> str:
        return f"cfg{self.cfg}-{self.m}x{self.n}-{self.density}-{self.precision}-k{self.k}p{self.p}q{self.q}"


CONFIGS = {
    1: Workload(1, 4096, 2048, 20, 10, 2, "double", "dense", "geom0.9", None, 1e-8, (512, 512)),
    2: Workload(2, 65536, 16384, 100, 20, 2, "double", "dense", "pow-1.5", None, 1e-8, (4096, 4096)),
    3: Workload(3, 1_000_000, 200_000, 100, 20, 3, "double", "sparse", "n01", None, 0.0, (65536, 200_000)),
    4: Workload(4, 1_048_576, 65_536, 200, 20, 2, "single", "dense", "exp-50", 500, 1e-3, (8192, 8192)),
    5: Workload(5, 16_384, 1_048_576, 500, 50, 3, "single", "dense", "inv", 1000, 1e-4, (16384, 131072)),
}


def spectrum(kind: str, count: int) -> np.ndarray:
    i = np.arange(count, dtype=np.float64)
    if kind == "geom0.9":
        return 0.9 ** i                      # s_i = 0.9^i, i = 0..
    if kind == "pow-1.5":
        return (i + 1.0) ** -1.5             # s_i = i^-1.5, i = 1..
    if kind == "exp-50":
        return np.exp(-i / 50.0)             # s_i = exp(-i/50)
    if kind == "inv":
        return 1.0 / (i + 1.0)               # s_i = 1/i, i = 1..
    raise ValueError(kind)


def haar_np(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    q, r = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q * np.where(np.diag(r) < 0, -1.0, 1.0)


def dense_lowrank_np(m: int, n: int, kind: str, noise: float, seed_a: int, seed_noise: int,
                     signal_rank: int | None = None, dtype=np.float64) -> np.ndarray:
    """A = U diag(s) V^T + noise * N(0,1), U/V Haar (numpy, small sizes)."""
    r = min(m, n) if signal_rank is None else signal_rank
    rng = np.random.default_rng(seed_a)
    u = haar_np(rng, m, r)
    v = haar_np(rng, n, r)
    a = (u * spectrum(kind, r)) @ v.T
    if noise:
        a += noise * np.random.default_rng(seed_noise).standard_normal((m, n))
    return a.astype(dtype)


def workload_dense_np(w: Workload, m: int | None = None, n: int | None = None) -> np.ndarray:
    """The config's construction at its own (or a reduced) shape."""
    return dense_lowrank_np(m or w.m, n or w.n, w.spectrum, w.noise, 1000 + w.cfg, 2000 + w.cfg,
                            w.signal_rank, np.float64 if w.precision == "double" else np.float32)


def dense_lowrank_torch(m: int, n: int, kind: str, noise: float, seed: int,
                        signal_rank: int | None = None, dtype=None, device="cuda",
                        rows: tuple | None = None, cols: tuple | None = None):
    """Same construction on the GPU via torch (cfg2+ sizes): the block
    A[rows[0]:rows[1], cols[0]:cols[1]] (default: all of A) as a torch tensor
    on `device`. Haar factors via torch.linalg.qr in f64; the noise is drawn
    per row chunk of fixed height from a generator keyed by the chunk index,
    so any row or column block of A — one rank's shard — is bitwise the same
    as the corresponding block of the whole matrix."""
    import torch

    dtype = dtype or torch.float64
    r0, r1 = rows if rows is not None else (0, m)
    c0, c1 = cols if cols is not None else (0, n)
    r = min(m, n) if signal_rank is None else signal_rank
    g = torch.Generator(device=device)
    g.manual_seed(1000 + seed)
    s = torch.from_numpy(spectrum(kind, r)).to(device)

    def haar(rr, cc):
        x = torch.randn(rr, cc, generator=g, device=device, dtype=torch.float64)
        q, R = torch.linalg.qr(x)
        del x
        return q * torch.where(torch.diagonal(R) < 0, -1.0, 1.0)

    u = haar(m, r)[r0:r1].clone()
    torch.cuda.empty_cache()
    u.mul_(s)
    v = haar(n, r)[c0:c1].clone()
    torch.cuda.empty_cache()
    a = torch.empty((r1 - r0, c1 - c0), dtype=dtype, device=device)
    # fixed chunk height (<= 2^28 elements of f64 per chunk): depends only on
    # (m, n), never on the requested block
    chunk = max(1, min(8192, (1 << 28) // max(n, 1)))
    gn = torch.Generator(device=device)
    for k0 in range((r0 // chunk) * chunk, r1, chunk):
        k1 = min(m, k0 + chunk)
        lo, hi = max(k0, r0), min(k1, r1)
        blk = u[lo - r0:hi - r0] @ v.T
        if noise:
            gn.manual_seed((2000 + seed) * 1_000_003 + k0 // chunk)
            z = torch.randn(k1 - k0, n, generator=gn, device=device, dtype=torch.float64)
            blk.add_(z[lo - k0:hi - k0, c0:c1], alpha=noise)
            del z
        a[lo - r0:hi - r0].copy_(blk)
        del blk
    del u, v
    return a


def sparse_uniform_np(m: int, n: int, per_row: int, seed: int):
    """CSR with exactly `per_row` distinct uniform columns per row and N(0,1)
    values (cfg3's stated density 1e-4 = 20 per row). Returns
    (rowptr int64, col int32, val f64) with columns sorted per row."""
    rng = np.random.default_rng(seed)
    cols = np.empty((m, per_row), dtype=np.int64)
    # rejection-free distinct sampling per row: sort + resample duplicates
    cols[:] = rng.integers(0, n, size=(m, per_row))
    cols.sort(axis=1)
    dup = np.any(cols[:, 1:] == cols[:, :-1], axis=1)
    while dup.any():
        idx = np.flatnonzero(dup)
        redo = rng.integers(0, n, size=(len(idx), per_row))
        redo.sort(axis=1)
        cols[idx] = redo
        dup = np.any(cols[:, 1:] == cols[:, :-1], axis=1)
    vals = rng.standard_normal(m * per_row)
    rowptr = np.arange(0, m * per_row + 1, per_row, dtype=np.int64)
    return rowptr, cols.reshape(-1).astype(np.int32), vals
