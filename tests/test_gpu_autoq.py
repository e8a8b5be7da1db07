"""power="auto" on the device (engine.cu AutoPower): the reference's
stopping rule (pipeline.py:295-372) evaluated on raw-product norms carried
through the re-orthonormalised iteration. Checked against goldens made by
the reference's own _sketch_and_power / auto_select_q / randomized_svd."""

import numpy as np
import pytest

from conftest import golden
from oracle import metrics as M
from oracle import pipeline as OP
from test_oracle_golden import AUTOQ_CASES, _autoq_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", AUTOQ_CASES)
def test_auto_power_matches_reference(lib, name):
    import paper_1907_06470_b200 as X

    g = golden("autoq")
    a, k, p, q_max, tau, seed = _autoq_case(g, name)
    pool = X.BlockPool()
    am = X.matrix_from_dense(pool, "A", a, precision=X.Precision.DOUBLE)
    res = X.randomized_svd(pool, am, X.RsvdConfig(rank=k, oversample=p, power="auto",
                                                  q_max=q_max, tau=tau, seed=seed))
    chosen = int(g[f"{name}_chosen"])
    assert res.chosen_q == chosen
    _, nus = lib.last_power()
    ref_nus = g[f"{name}_nus"]
    assert len(nus) == len(ref_nus)
    # raw-product norms from the triangular factors: ~u kappa relative
    assert np.allclose(nus, ref_nus, rtol=1e-9, atol=0.0)
    if name != "zero":
        ref = OP.rsvd_reorth(a, k, p, chosen, seed, "double", fast=True)
        assert M.sigma_rel(res.s, ref.s) <= 1e-10
        assert M.sin_angle(res.u.to_array(), ref.u) <= 1e-8
        assert M.sin_angle(res.v.to_array(), ref.v) <= 1e-8
    assert X.auto_select_q(pool, am, k, q_max=q_max, tau=tau, seed=seed) == \
        int(g[f"{name}_probe_chosen"])


def test_auto_power_sparse(lib):
    """Sparse A takes the same rule (xb_rsvd_coo with XB_POWER_AUTO)."""
    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import sparse_uniform_np

    m, n = 3000, 800
    rowptr, col, val = sparse_uniform_np(m, n, 6, 5)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    dense = np.zeros((m, n))
    dense[rows, col] = val
    lib.set_power_auto(5, 1e-6)
    u, s, v, _, _ = lib.rsvd_coo(rows, col, val, (m, n), 10, 5, _lib.POWER_AUTO, 3)
    chosen, nus = lib.last_power()
    ref_q, ref_nus = OP.sketch_power_auto(dense, 10, 5, 3, q_max=5, tau=1e-6, fast=True)
    assert chosen == ref_q
    assert np.allclose(nus, ref_nus, rtol=1e-9, atol=0.0)
    ref = OP.rsvd_reorth(dense, 10, 5, chosen, 3, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10


# -- the reference's own auto-q tests (tests/test_pipeline.py:77-111, 298-311),
#    through this package's drop-in ---------------------------------------------

def _dense(X, pool, arr):
    return X.matrix_from_dense(pool, "a", arr, precision=X.Precision.DOUBLE)


def test_auto_q_stops_early_on_flat_spectrum(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(2)
    q_mat, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    pool = X.BlockPool()
    assert X.auto_select_q(pool, _dense(X, pool, q_mat), 6, q_max=5, seed=0) <= 1


def test_auto_q_threshold_branch_fires(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(3)
    q_mat, _ = np.linalg.qr(rng.standard_normal((25, 25)))
    pool = X.BlockPool()
    assert X.auto_select_q(pool, _dense(X, pool, 1e-4 * q_mat), 5, q_max=5, tau=1e-6,
                           seed=0) == 1


def test_auto_q_zero_matrix(lib):
    import paper_1907_06470_b200 as X

    pool = X.BlockPool()
    assert X.auto_select_q(pool, _dense(X, pool, np.zeros((10, 10))), 3, seed=0) == 0


def test_auto_q_decaying_spectrum_needs_passes(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(4)
    u, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    v, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    s = np.array([0.9**i for i in range(40)])
    pool = X.BlockPool()
    assert 1 <= X.auto_select_q(pool, _dense(X, pool, (u * s) @ v.T), 8, q_max=5, seed=0) <= 5


def test_auto_power_beats_or_ties_fixed_zero(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(14)
    u, _ = np.linalg.qr(rng.standard_normal((100, 100)))
    v, _ = np.linalg.qr(rng.standard_normal((80, 80)))
    s = np.array([(i + 1) ** -0.5 for i in range(80)])
    a = (u[:, :80] * s) @ v.T

    def recon_err(res):  # the reference test's measure (test_pipeline.py:31-33)
        approx = res.u.to_array() @ np.diag(res.s) @ res.v.to_array().T
        return np.max(np.abs(approx - a)) / max(np.max(np.abs(a)), 1e-300)

    pool = X.BlockPool()
    ma = _dense(X, pool, a)
    fixed = X.randomized_svd(pool, ma, X.RsvdConfig(rank=10, power=0, seed=0))
    err_fixed = recon_err(fixed)  # before the next call re-registers U / V
    auto = X.randomized_svd(pool, ma, X.RsvdConfig(rank=10, power="auto", seed=0))
    assert auto.chosen_q >= 1
    assert recon_err(auto) <= err_fixed * 1.02
