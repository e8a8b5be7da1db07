"""RsvdConfig.gram_path=True on the device (engine.cu: power-matrix
projection, Gram, Jacobi, sigma^(1/(2q+1)), unit V columns) against the
reference's own outputs (tests/golden/gram.npz) and its tests
(test_pipeline.py:244-282)."""

import numpy as np
import pytest

from conftest import golden
from oracle import metrics as M
from oracle import pipeline as OP
from test_oracle_golden import GRAM_CASES

pytestmark = pytest.mark.gpu


def _run(a, k, p, q, seed, gram=True, dtype=np.float64):
    import paper_1907_06470_b200 as X

    prec = X.Precision.DOUBLE if dtype == np.float64 else X.Precision.SINGLE
    pool = X.BlockPool()
    ma = X.matrix_from_dense(pool, "a", a.astype(dtype), precision=prec)
    return X.randomized_svd(pool, ma, X.RsvdConfig(rank=k, oversample=p, power=q, seed=seed,
                                                   gram_path=gram, precision=prec))


def _recon(res, a):
    approx = res.u.to_array() @ np.diag(res.s) @ res.v.to_array().T
    return np.max(np.abs(approx - a)) / max(np.max(np.abs(a)), 1e-300)


@pytest.mark.parametrize("name", GRAM_CASES)
def test_gram_path_matches_reference(lib, name):
    g = golden("gram")
    a = g[f"{name}_a"]
    k, p, q, seed = (int(x) for x in g[f"{name}_cfg"])
    res = _run(a, k, p, q, seed)
    ref_s = g[f"{name}_s"]
    # the Gram squares the condition: the reference's own gram-vs-direct
    # bound is 1e-6 (test_pipeline.py:270); here against its gram outputs
    assert np.max(np.abs(res.s - ref_s)) / ref_s[0] <= 1e-10
    assert M.sin_angle(res.u.to_array(), g[f"{name}_u"]) <= 1e-8
    assert M.sin_angle(res.v.to_array(), g[f"{name}_v"]) <= 1e-8
    orc = OP.rsvd_reorth_gram(a, k, p, q, seed)
    assert np.max(np.abs(res.s - orc.s)) / orc.s[0] <= 1e-10


def test_gram_route_corrects_exponent(lib):
    res = _run(np.diag([2.0, 1.0]), 2, 0, 1, 0)
    assert np.allclose(res.s, [2.0, 1.0], atol=1e-10)


def test_gram_route_matches_direct_on_random_input(lib):
    rng = np.random.default_rng(12)
    a = rng.standard_normal((50, 8)) @ rng.standard_normal((8, 45))
    direct = _run(a, 8, 0, 1, 0, gram=False)
    grammed = _run(a, 8, 0, 1, 0)
    assert np.max(np.abs(direct.s - grammed.s)) / direct.s[0] <= 1e-6
    assert _recon(grammed, a) <= 1e-6


def test_gram_route_at_power_zero_matches_direct(lib):
    rng = np.random.default_rng(20)
    a = rng.standard_normal((40, 5)) @ rng.standard_normal((5, 35))
    direct = _run(a, 5, 0, 0, 0, gram=False)
    grammed = _run(a, 5, 0, 0, 0)
    assert np.max(np.abs(direct.s - grammed.s)) / direct.s[0] <= 1e-6


def test_gram_route_single_and_large(lib):
    """float32 storage and a size where the products run on the int8 path."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(4096, 4096, "geom0.9", 1e-8, 5, 6)
    res = _run(a, 10, 6, 1, 2)
    orc = OP.rsvd_reorth_gram(a, 10, 6, 1, 2)
    assert np.max(np.abs(res.s - orc.s)) / orc.s[0] <= 1e-10
    assert M.sin_angle(res.u.to_array(), orc.u) <= 1e-8
    r32 = _run(a, 10, 6, 1, 2, dtype=np.float32)
    orc32 = OP.rsvd_reorth_gram(a.astype(np.float32), 10, 6, 1, 2, "single")
    assert np.max(np.abs(r32.s - orc32.s)) / orc32.s[0] <= 1e-4


def test_gram_path_state_does_not_leak(lib):
    """A gram_path call leaves the context's default (direct) route."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((60, 40))
    _run(a, 5, 2, 1, 0, gram=True)
    u, s, v, _, _ = lib.rsvd_dense(a, 5, 2, 1, 0)
    ref = OP.rsvd_reorth(a, 5, 2, 1, 0, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10
