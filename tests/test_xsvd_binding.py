"""The reference-side binding of INTEGRATION.md, driven through the REAL
reference package `xsvd` (importable in the build container from
/root/reference/pkg/src; skipped where it is absent, e.g. on the GPU box).

* CPU (`-m "not gpu"`): the §1 dispatch a maintainer adds at the top of
  xsvd.pipeline.randomized_svd routes the reference's own objects (its
  BlockPool, StoredMatrix, RsvdConfig) into this package's randomized_svd,
  which registers U/S/V back into the reference's pool. The device call is
  stood in for by the oracle here (no GPU in this container) — only this
  test's monkeypatch does that; the product path has no CPU fallback.
  The §2 module patching resolves through xsvd.pipeline's globals.
* GPU (`-m gpu`): the same dispatch with the real device call, against the
  reference's own shipped driver output at config 1's shape.
"""

import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


def _xsvd():
    if os.path.isdir(REF_SRC) and REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    try:
        import xsvd  # noqa: F401
        import xsvd.pipeline
    except ImportError:
        pytest.skip("the reference package xsvd is not importable here")
    return sys.modules["xsvd"]


def _install_dispatch(monkeypatch, xsvd):
    """INTEGRATION.md §1, verbatim in spirit: the first lines of
    xsvd.pipeline.randomized_svd hand an unbudgeted call to the B200 path."""
    import paper_1907_06470_b200 as G

    shipped = xsvd.pipeline.randomized_svd
    calls = []

    def randomized_svd(pool, a, config, *, threads=1, runner=None, clock=None):
        if os.environ.get("XSVD_BACKEND") == "b200" and pool.store is None:
            calls.append(a.matrix_id)
            return G.randomized_svd(pool, a, config, threads=threads, runner=runner, clock=clock)
        return shipped(pool, a, config, threads=threads, runner=runner, clock=clock)

    monkeypatch.setattr(xsvd.pipeline, "randomized_svd", randomized_svd)
    monkeypatch.setenv("XSVD_BACKEND", "b200")
    return calls


def test_dispatch_routes_reference_objects_cpu(monkeypatch):
    xsvd = _xsvd()
    import paper_1907_06470_b200.pipeline as GP
    from oracle import pipeline as OP

    def device_standin(a, config, precision, clock):
        arr = np.asarray(GP._dense_input(a), dtype=np.float64)
        r = OP.rsvd_reorth(arr, config.rank, config.oversample, int(config.power), config.seed,
                           "double", fast=True)
        return r.u, r.s, r.v, r.deficient_columns, int(config.power)

    monkeypatch.setattr(GP, "_rsvd_device", device_standin)
    calls = _install_dispatch(monkeypatch, xsvd)
    pool = xsvd.BlockPool()
    arr = np.random.default_rng(1).standard_normal((200, 80))
    a = xsvd.matrix_from_dense(pool, "A", arr, precision=xsvd.Precision.DOUBLE)
    cfg = xsvd.RsvdConfig(rank=5, oversample=5, power=1, seed=3, precision=xsvd.Precision.DOUBLE)
    res = xsvd.pipeline.randomized_svd(pool, a, cfg)
    assert calls == ["A"]
    # the results live in the REFERENCE's pool, as its own matrix objects
    assert isinstance(res.u, xsvd.StoredMatrix) and isinstance(res.v, xsvd.StoredMatrix)
    assert pool.descriptor("U").rows == 200 and pool.descriptor("V").rows == 80
    assert pool.descriptor("S").rows == 5
    assert set(res.stage_seconds) == set(xsvd.STAGE_NAMES)
    ref = OP.rsvd_reorth(arr, 5, 5, 1, 3, "double", fast=True)
    np.testing.assert_allclose(res.s, ref.s, rtol=1e-12)
    np.testing.assert_allclose(np.abs(res.u.to_array()), np.abs(ref.u), atol=1e-12)


def test_module_patching_resolves_through_pipeline_globals(monkeypatch):
    """xsvd.pipeline looks block_multiply / thin_qr /
    svd_small up in its module globals at call time, so patched names are
    the ones the shipped orchestration calls."""
    xsvd = _xsvd()
    P = xsvd.pipeline
    seen = []
    for name in ("block_multiply", "thin_qr", "svd_small"):
        orig = getattr(P, name)

        def wrap(*args, _orig=orig, _name=name, **kw):
            seen.append(_name)
            return _orig(*args, **kw)

        monkeypatch.setattr(P, name, wrap)
    pool = xsvd.BlockPool()
    arr = np.random.default_rng(2).standard_normal((120, 60))
    a = xsvd.matrix_from_dense(pool, "A", arr, precision=xsvd.Precision.DOUBLE)
    P.randomized_svd(pool, a, xsvd.RsvdConfig(rank=4, oversample=2, power=1, seed=1))
    assert {"block_multiply", "thin_qr", "svd_small"} <= set(seen)


@pytest.mark.gpu
def test_dispatch_on_device_matches_shipped_driver(monkeypatch):
    """The §1 dispatch with the real device call, on config 1's construction
    (4096 x 2048 f64, k=20 p=10 q=2), against the reference's own shipped
    driver on the same objects (the reference is its own oracle at config
    1)."""
    xsvd = _xsvd()
    from oracle import metrics as M
    from paper_1907_06470_b200.workloads import CONFIGS, workload_dense_np

    w = CONFIGS[1]
    arr = workload_dense_np(w)
    pool_ref = xsvd.BlockPool()
    a_ref = xsvd.matrix_from_dense(pool_ref, "A", arr, precision=xsvd.Precision.DOUBLE)
    cfg = xsvd.RsvdConfig(rank=w.k, oversample=w.p, power=w.q, seed=w.cfg,
                          precision=xsvd.Precision.DOUBLE)
    ref = xsvd.pipeline.randomized_svd(pool_ref, a_ref, cfg)
    calls = _install_dispatch(monkeypatch, xsvd)
    pool = xsvd.BlockPool()
    a = xsvd.matrix_from_dense(pool, "A", arr, precision=xsvd.Precision.DOUBLE)
    res = xsvd.pipeline.randomized_svd(pool, a, cfg)
    assert calls == ["A"]
    assert M.sigma_rel(res.s, ref.s) <= 1e-10
    assert M.sin_angle(res.u.to_array(), ref.u.to_array()) <= 1e-8
    assert M.sin_angle(res.v.to_array(), ref.v.to_array()) <= 1e-8
