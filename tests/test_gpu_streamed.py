"""Out-of-core path (config 4's design): A stays in host memory and streams
through HBM in row tiles, q + 1 fused passes. Forced here with small tiles on
matrices that would fit, so the oracle can check them."""

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,q,tile", [("double", 2, 1024), ("double", 0, 700),
                                          ("single", 2, 2048), ("double", 1, 0)])
def test_streamed_matches_oracle(lib, dtype, q, tile):
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    npdt = np.float64 if dtype == "double" else np.float32
    if dtype == "double":
        a = dense_lowrank_np(9000, 1500, "pow-1.5", 1e-8, 41, 42).astype(npdt)
        tol_s, tol_a = 1e-10, 1e-8
    else:
        a = dense_lowrank_np(12000, 2000, "exp-50", 1e-3, 43, 44, 500, np.float32)
        tol_s, tol_a = 1e-4, 1e-3
    k, p = 60, 20
    u, s, v, deficient, stages = lib.rsvd_dense_streamed(a, k, p, q, 9, tile_rows=tile)
    ref = OP.rsvd_reorth(a, k, p, q, 9, dtype, fast=True)
    assert M.sigma_rel(s, ref.s) <= tol_s
    assert M.sin_angle(u, ref.u) <= tol_a
    assert M.sin_angle(v, ref.v) <= tol_a
    assert deficient == ()
    assert stages[0] > 0  # host->HBM streaming time is reported


def test_streamed_rank_deficient_falls_back(lib):
    """rank(A) < l: a Cholesky breaks down and Z = A^T Q comes from an extra
    TN-only pass; results still match the reference singular values."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((4000, 15)) @ rng.standard_normal((15, 900))
    u, s, v, _, _ = lib.rsvd_dense_streamed(a, 20, 5, 1, 3, tile_rows=512)
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(s[:15] - ref[:15])) / ref[0] <= 1e-10
    assert M.sin_angle(u[:, :15], np.linalg.svd(a, full_matrices=False)[0][:, :15]) <= 1e-8


def test_streamed_power_auto_matches_in_hbm(lib):
    """power="auto" out of core (pipeline.py:295-372): the stopping rule is
    evaluated on every fused pass's raw Y, so the chosen q and the nu
    sequence equal the in-HBM engine's and the oracle loop's."""
    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(6000, 1200, "geom0.9", 1e-8, 45, 46)
    lib.set_power_auto(5, 1e-6)
    u0, s0, v0, _, _ = lib.rsvd_dense(a, 30, 10, _lib.POWER_AUTO, 4)
    q0, nu0 = lib.last_power()
    u1, s1, v1, _, _ = lib.rsvd_dense_streamed(a, 30, 10, _lib.POWER_AUTO, 4, tile_rows=1024)
    q1, nu1 = lib.last_power()
    qref, nuref = OP.sketch_power_auto(a, 30, 10, 4, "double", q_max=5, tau=1e-6, fast=True)
    assert q1 == q0 == qref
    np.testing.assert_allclose(nu1, nuref, rtol=1e-10)
    ref = OP.rsvd_reorth(a, 30, 10, qref, 4, "double", fast=True)
    assert M.sigma_rel(s1, ref.s) <= 1e-10
    assert M.sin_angle(u1, ref.u) <= 1e-8 and M.sin_angle(v1, ref.v) <= 1e-8


def test_streamed_gram_path_matches_oracle(lib):
    """gram_path out of core (pipeline.py:526-580): the power-matrix
    projection's 2q raw products are q more fused passes. The Gram route
    carries sigma^(4q+2), so only sigma_i / sigma_1 above ~eps^(1/(4q+2))
    are meaningful in any implementation: spectrum 1/i, q = 1."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(5000, 1000, "inv", 1e-10, 47, 48)
    lib.set_gram_path(True)
    try:
        u, s, v, _, _ = lib.rsvd_dense_streamed(a, 40, 10, 1, 6, tile_rows=800)
        u0, s0, v0, _, _ = lib.rsvd_dense(a, 40, 10, 1, 6)
    finally:
        lib.set_gram_path(False)
    ref = OP.rsvd_reorth_gram(a, 40, 10, 1, 6, "double", fast=True)
    assert np.max(np.abs(s - ref.s)) / ref.s[0] <= 1e-9
    assert np.max(np.abs(s - s0)) / s0[0] <= 1e-9
    assert M.sin_angle(u[:, :20], ref.u[:, :20]) <= 1e-6
    assert M.sin_angle(v[:, :20], ref.v[:, :20]) <= 1e-6


@pytest.mark.parametrize("grid,transposed,stream", [((5, 3), False, False), ((7, 2), False, True),
                                                    ((3, 4), True, False), ((4, 4), True, True)])
def test_tile_grid_source_matches_oracle(lib, grid, transposed, stream):
    """A as the reference's tile grid (xb_rsvd_dense_tiles): tiles fetched one
    at a time from the pool and never assembled into one host array — in HBM
    (bands ingested as they land) or streamed (q + 1 fused passes over the
    grid) — including a transposed view, whose tile (ti, tj) is the stored
    (tj, ti) transposed (pool.py:390-418)."""
    import paper_1907_06470_b200 as X
    from paper_1907_06470_b200.pipeline import _tile_grid
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    arr = dense_lowrank_np(3000, 1300, "pow-1.5", 1e-8, 51, 52)
    pool = X.BlockPool()
    base = arr.T.copy() if transposed else arr
    ma = X.matrix_from_dense(pool, "A", base, precision=X.Precision.DOUBLE, grid=grid)
    a = ma.T if transposed else ma
    assert a.shape == arr.shape
    rows, cols, get_tile, release = _tile_grid(a)
    u, s, v, _, stages = lib.rsvd_dense_tiles(a.shape, rows, cols, get_tile, np.float64, 50, 10,
                                              2, 7, release=release, force_stream=stream)
    ref = OP.rsvd_reorth(arr, 50, 10, 2, 7, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10
    assert M.sin_angle(u, ref.u) <= 1e-8 and M.sin_angle(v, ref.v) <= 1e-8
    assert stages[0] > 0


def test_budgeted_store_backed_tiles_through_drop_in(lib, tmp_path):
    """A budgeted pool over a BlockStore (tiles spill to the workdir and come
    back on demand, pool.py:189-221): randomized_svd streams the tile grid
    from the pool — the path a matrix larger than host RAM takes."""
    import paper_1907_06470_b200 as X
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    arr = dense_lowrank_np(2400, 900, "geom0.9", 1e-8, 53, 54)
    pool = X.BlockPool(X.BlockStore(str(tmp_path)))
    ma = X.matrix_from_dense(pool, "A", arr, precision=X.Precision.DOUBLE, grid=(6, 3))
    res = X.randomized_svd(pool, ma, X.RsvdConfig(rank=20, oversample=10, power=2, seed=3))
    ref = OP.rsvd_reorth(arr, 20, 10, 2, 3, "double", fast=True)
    assert M.sigma_rel(res.s, ref.s) <= 1e-10
    assert M.sin_angle(res.u.to_array(), ref.u) <= 1e-8
