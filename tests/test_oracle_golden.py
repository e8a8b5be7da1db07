"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py). CPU only.

Bitwise where the restatement follows the reference's operation sequence
on the same numpy build; 1e-15-level where a `fast` (LAPACK) variant is used.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import kernels as K
from oracle import metrics as M
from oracle import pipeline as P
from oracle import rng as R


def test_rng_bitwise():
    g = golden("rng")
    i = 0
    while f"band{i}" in g:
        seed, r0, r1, n = (int(x) for x in g[f"case{i}"])
        assert np.array_equal(R.gaussian_band(seed, r0, r1, n), g[f"band{i}"]), i
        i += 1
    seed, row, count = (int(x) for x in g["bits_case"])
    assert np.array_equal(R.uniform_bits(seed, row, count), g["bits"])


def test_rng_band_equals_rows():
    whole = R.gaussian_band(5, 0, 40, 64)
    split = np.vstack([R.gaussian_band(5, 0, 13, 64), R.gaussian_band(5, 13, 40, 64)])
    assert np.array_equal(whole, split)


def test_multiply_bitwise():
    g = golden("multiply")
    f64 = np.float64
    assert np.array_equal(K.block_multiply(g["x"], g["y"], f64, f64), g["nn"])
    assert np.array_equal(K.block_multiply(g["x"].T, g["w"], f64, f64), g["tn"])
    x32, y32 = g["x"].astype(np.float32), g["y"].astype(np.float32)
    assert np.array_equal(K.block_multiply(x32, y32, np.float32, np.float32), g["nn32"])
    coo = P.Coo(g["sp_rows"], g["sp_cols"], g["sp_vals"], tuple(g["sp_shape"]))
    assert np.array_equal(P._mul(coo, g["z"], "double", False), g["spmm"])
    assert np.array_equal(P._mul(coo.T, g["q"], "double", False), g["spmm_t"])
    assert np.array_equal(P._mul(g["q"].T, coo, "double", False), g["dense_sp"])
    # fast variants agree to rounding
    assert np.max(np.abs(P._mul(coo, g["z"], "double", True) - g["spmm"])) <= 1e-13
    assert np.max(np.abs(P._mul(g["q"].T, coo, "double", True) - g["dense_sp"])) <= 1e-13


@pytest.mark.parametrize("name", ["tall", "c345", "eye", "zero", "deficient", "tall32"])
def test_qr_matches_reference(name):
    g = golden("qr")
    a = g[f"{name}_a"]
    sdt = a.dtype.type
    cdt = np.float32 if a.dtype == np.float32 else np.float64
    q, r, d = K.thin_qr(a, sdt, cdt)
    assert np.array_equal(q, g[f"{name}_q"])
    assert np.array_equal(r, g[f"{name}_r"])
    assert tuple(d) == tuple(g[f"{name}_def"])
    if name in ("tall", "c345", "eye", "tall32"):
        qf, rf, df = K.thin_qr_fast(a, sdt, cdt)
        tol = 1e-13 if cdt is np.float64 else 1e-6
        assert np.max(np.abs(qf.astype(np.float64) - g[f"{name}_q"])) <= tol
        assert tuple(df) == tuple(g[f"{name}_def"])


@pytest.mark.parametrize("name", ["wide", "diag", "perm", "r30", "deficient"])
def test_svd_small_matches_reference(name):
    g = golden("svd")
    u, s, v = K.svd_small(g[f"{name}_b"])
    assert np.array_equal(s, g[f"{name}_s"])
    assert np.array_equal(u, g[f"{name}_u"])
    assert np.array_equal(v, g[f"{name}_v"])
    uf, sf, vf = K.svd_small_fast(g[f"{name}_b"])
    assert np.max(np.abs(sf - g[f"{name}_s"])) <= 1e-13 * max(1.0, g[f"{name}_s"][0])


def _case(g, name):
    m, n, k, p, q, seed, dbl = (int(x) for x in g[f"{name}_cfg"])
    prec = "double" if dbl else "single"
    if f"{name}_a" in g:
        a = g[f"{name}_a"]
    else:
        a = P.Coo(g[f"{name}_rows"], g[f"{name}_cols"], g[f"{name}_vals"], tuple(g[f"{name}_shape"]))
    return a, k, p, q, seed, prec


@pytest.mark.parametrize("name", ["d_small", "d_q0", "d_wide", "s_small", "sp_small"])
@pytest.mark.parametrize("variant", ["shipped", "reorth"])
def test_rsvd_matches_reference(name, variant):
    g = golden("rsvd")
    a, k, p, q, seed, prec = _case(g, name)
    fn = P.randomized_svd if variant == "shipped" else P.rsvd_reorth
    res = fn(a, k, p, q, seed, prec)
    assert np.array_equal(res.s, g[f"{name}_{variant}_s"])
    assert np.array_equal(res.u, g[f"{name}_{variant}_u"])
    assert np.array_equal(res.v, g[f"{name}_{variant}_v"])
    # the LAPACK-backed fast oracle agrees within the parity tolerances
    fast = fn(a, k, p, q, seed, prec, fast=True)
    tol_s, tol_a = (1e-10, 1e-8) if prec == "double" else (1e-4, 1e-3)
    if variant == "shipped":
        # the shipped driver runs 2q+1 raw products before its only QR
        # (src/pipeline.py:321-371), which amplifies rounding differences
        # (SURVEY F4/F5); only the bitwise restatement is held to 1e-8
        # and in single precision it is not a usable oracle at all
        if prec == "single":
            return
        tol_s, tol_a = tol_s * 100, tol_a * 100
    assert M.sigma_rel(fast.s, res.s) <= tol_s
    assert M.sin_angle(fast.u, res.u) <= tol_a
    assert M.sin_angle(fast.v, res.v) <= tol_a


def test_cfg1_full_size_pinned():
    """Config 1 at full size (4096x2048): oracle (fast) vs the reference's
    shipped driver and xsvd-reorth outputs."""
    from paper_1907_06470_b200.workloads import CONFIGS, workload_dense_np

    g = golden("cfg1")
    w = CONFIGS[1]
    a = workload_dense_np(w)
    assert abs(float(np.sum(a)) - g["checksum"][0]) <= 1e-9 * max(1.0, abs(g["checksum"][0]))
    for variant, fn in (("shipped", P.randomized_svd), ("reorth", P.rsvd_reorth)):
        res = fn(a, w.k, w.p, w.q, w.cfg, "double", fast=True)
        assert M.sigma_rel(res.s, g[f"{variant}_s"]) <= 1e-10
        assert M.sin_angle(res.u, g[f"{variant}_u"]) <= 1e-8
        assert M.sin_angle(res.v, g[f"{variant}_v"]) <= 1e-8
    # at cfg1 the shipped driver IS a valid oracle for the re-orth path
    assert M.sigma_rel(g["shipped_s"], g["reorth_s"]) <= 1e-10
    assert M.sin_angle(g["shipped_u"], g["reorth_u"]) <= 1e-8


def test_sine_angle_metric():
    rng = np.random.default_rng(0)
    x = np.linalg.qr(rng.standard_normal((50, 4)))[0]
    assert M.sin_angle(x, x @ np.diag([1, -1, 2, 3.0])) <= 1e-14
    y = x.copy()
    y[:, 0] = np.linalg.qr(rng.standard_normal((50, 1)))[0][:, 0]
    assert M.sin_angle(x, y) > 0.1


def _autoq_case(g, name):
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    m, n, k, p, q_max, seed = (int(x) for x in g[f"{name}_cfg"])
    spec = str(g[f"{name}_spec"])
    scale, tau = (float(x) for x in g[f"{name}_scale_tau"])
    sa, sn = (int(x) for x in g[f"{name}_a_seeds"])
    a = np.zeros((m, n)) if spec == "zero" else scale * dense_lowrank_np(m, n, spec, 1e-8, sa, sn)
    return a, k, p, q_max, tau, seed


AUTOQ_CASES = ["pow", "geom", "small_scale", "qmax2", "qmax0", "zero"]


@pytest.mark.parametrize("name", AUTOQ_CASES)
def test_power_auto_golden(name):
    """power="auto" restated (oracle.pipeline.sketch_power_auto) against the
    reference's own _sketch_and_power loop: same chosen q, same nu sequence."""
    g = golden("autoq")
    a, k, p, q_max, tau, seed = _autoq_case(g, name)
    chosen, nus = P.sketch_power_auto(a, k, p, seed, q_max=q_max, tau=tau)
    assert chosen == int(g[f"{name}_chosen"])
    ref = g[f"{name}_nus"]
    assert len(nus) == len(ref)
    assert np.allclose(nus, ref, rtol=1e-12, atol=0.0)


GRAM_CASES = ["diag", "rank8", "rank5_q0", "geom"]


@pytest.mark.parametrize("name", GRAM_CASES)
def test_gram_path_golden(name):
    """gram_path restated (oracle.pipeline.rsvd_reorth_gram) against the
    reference's randomized_svd(gram_path=True) on exact-rank / well-resolved
    inputs, where the shipped and re-orthonormalised range finders agree."""
    g = golden("gram")
    k, p, q, seed = (int(x) for x in g[f"{name}_cfg"])
    r = P.rsvd_reorth_gram(g[f"{name}_a"], k, p, q, seed)
    ref_s = g[f"{name}_s"]
    assert np.max(np.abs(r.s - ref_s)) / ref_s[0] <= 1e-12
    assert M.sin_angle(r.u, g[f"{name}_u"]) <= 1e-12
    assert M.sin_angle(r.v, g[f"{name}_v"]) <= 1e-12
