"""float32 (Precision.SINGLE) inputs and large sketch widths (l = 220, 550:
the cooperative multi-CTA Jacobi and the global-memory Cholesky), through the
C ABI, against the CPU oracle and the reference golden vectors.

Tolerances (north star): float32 sigma relative <= 1e-4, sine angle <= 1e-3;
float64 1e-10 / 1e-8.
"""

import os

import numpy as np
import pytest

from conftest import golden
from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu

SIG32, ANG32 = 1e-4, 1e-3
SIG64, ANG64 = 1e-10, 1e-8


@pytest.mark.parametrize("m,n,k", [(300, 30, 520), (1000, 120, 3000), (777, 224, 999),
                                   (4096, 552, 300)])
@pytest.mark.parametrize("trans", [False, True])
def test_gemm_f32(lib, m, n, k, trans):
    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((k, m) if trans else (m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    got = lib.gemm(a, b, trans_a=trans)
    assert got.dtype == np.float32
    ref = (a.T if trans else a).astype(np.float64) @ b.astype(np.float64)
    # float32 products run as 3xTF32 on tcgen05 with round-to-nearest f32
    # folding of each 64-deep TMEM group (measured 1.5e-6..5e-6 on these
    # shapes; cuBLAS SGEMM 1e-6..8e-5 at K = 520..262144, tools/diag_tgemm3.py).
    # The DMMA path (XB_F32_GEMM=dmma) accumulates in f64: one f32 rounding.
    tol = 1e-6 if os.environ.get("XB_F32_GEMM") == "dmma" else 1e-5
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), np.sqrt(k))) <= tol


@pytest.mark.parametrize("trans", [False, True])
def test_gemm_f32_long_k(lib, trans):
    """K = 131072: the TMEM accumulator is folded into f32 registers every
    64 of K, so the error must not grow with the chain (a single TMEM chain
    measured ~30x worse than this bound)."""
    import torch

    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    n = 200
    if trans:  # Z = A^T X with A stored (131072 x 2048): the reduction runs over the long side
        m, kdim = 2048, 131072
        a = torch.randn(kdim, m, device="cuda", generator=gen)
        lda, ref_a = m, a.double().T
    else:  # Y = A X with A stored (2048 x 131072)
        m, kdim = 2048, 131072
        a = torch.randn(m, kdim, device="cuda", generator=gen)
        lda, ref_a = kdim, a.double()
    x = torch.randn(kdim, n, device="cuda", generator=gen)
    c = torch.empty(m, n, device="cuda")
    lib.gemm_dev(np.float32, trans, m, n, kdim, a.data_ptr(), lda, x.data_ptr(), n, c.data_ptr(), n)
    ref = ref_a @ x.double()
    kk = kdim
    torch.cuda.synchronize()
    err = ((c.double() - ref).abs() / torch.clamp(ref.abs(), min=kk ** 0.5)).max().item()
    assert err <= 1e-5


def test_gemm_f32_golden(lib, gold):
    g = gold("multiply")
    got = lib.gemm(g["x"].astype(np.float32), g["y"].astype(np.float32))
    assert np.max(np.abs(got - g["nn32"])) / np.max(np.abs(g["nn32"])) <= 1e-5


def test_thin_qr_f32_golden(lib, gold):
    g = gold("qr")
    q, r, d = lib.thin_qr(g["tall32_a"])
    assert q.dtype == np.float32
    assert np.max(np.abs(q - g["tall32_q"])) <= 1e-5
    assert np.max(np.abs(r - g["tall32_r"])) <= 1e-9 * np.max(np.abs(g["tall32_r"]))
    assert d == ()


def test_rsvd_f32_golden(lib, gold):
    g = gold("rsvd")
    a = g["s_small_a"]
    assert a.dtype == np.float32
    m, n, k, p, q, seed, _ = (int(x) for x in g["s_small_cfg"])
    u, s, v, deficient, _ = lib.rsvd_dense(a, k, p, q, seed)
    assert u.dtype == np.float32 and v.dtype == np.float32
    assert M.sigma_rel(s, g["s_small_reorth_s"]) <= SIG32
    assert M.sin_angle(u, g["s_small_reorth_u"]) <= ANG32
    assert M.sin_angle(v, g["s_small_reorth_v"]) <= ANG32


@pytest.mark.parametrize("m,n,k,p,q", [(1000, 800, 200, 20, 1), (1200, 900, 500, 50, 1)])
def test_large_sketch_f64(lib, m, n, k, p, q):
    """l = 220 and l = 550: the cooperative Jacobi and the L2-resident Cholesky."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(m, n, "inv", 1e-6, 77, 78)
    u, s, v, _, _ = lib.rsvd_dense(a, k, p, q, 3)
    ref = OP.rsvd_reorth(a, k, p, q, 3, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= SIG64
    assert M.sin_angle(u, ref.u) <= ANG64
    assert M.sin_angle(v, ref.v) <= ANG64


def test_svd_small_large_l(lib):
    """svd_small with r = 550 (cooperative Jacobi) vs LAPACK."""
    rng = np.random.default_rng(8)
    b = rng.standard_normal((550, 2000)) * np.logspace(0, -4, 550)[:, None]
    u, s, v = lib.svd_small(b)
    sr = np.linalg.svd(b, compute_uv=False)
    assert np.max(np.abs(s - sr) / sr) <= 1e-10
    assert np.max(np.abs(u @ np.diag(s) @ v.T - b)) <= 1e-12 * np.max(np.abs(b))
    assert M.ortho_defect(u) <= 1e-12 and M.ortho_defect(v) <= 1e-12


def test_cfg4_like_f32(lib):
    """Config 4's construction (rank-500 signal, s_i = exp(-i/50), noise 1e-3,
    float32) at 16384 x 4096, k=200 p=20 q=2."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(16384, 4096, "exp-50", 1e-3, 1004, 2004, 500, np.float32)
    u, s, v, _, _ = lib.rsvd_dense(a, 200, 20, 2, 4)
    ref = OP.rsvd_reorth(a, 200, 20, 2, 4, "single", fast=True)
    assert M.sigma_rel(s, ref.s) <= SIG32
    assert M.sin_angle(u, ref.u) <= ANG32
    assert M.sin_angle(v, ref.v) <= ANG32


def test_cfg5_like_f32(lib):
    """Config 5's construction (wide, rank-1000 signal s_i = 1/i, noise 1e-4,
    float32) at 2048 x 16384, k=500 p=50 q=3."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(2048, 16384, "inv", 1e-4, 1005, 2005, 1000, np.float32)
    u, s, v, _, _ = lib.rsvd_dense(a, 500, 50, 3, 5)
    ref = OP.rsvd_reorth(a, 500, 50, 3, 5, "single", fast=True)
    assert M.sigma_rel(s, ref.s) <= SIG32
    assert M.sin_angle(u, ref.u) <= ANG32
    assert M.sin_angle(v, ref.v) <= ANG32


def test_drop_in_single_precision(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(9)
    arr = rng.standard_normal((500, 300)).astype(np.float32)
    pool = X.BlockPool()
    a = X.matrix_from_dense(pool, "A", arr, precision=X.Precision.SINGLE)
    res = X.randomized_svd(pool, a, X.RsvdConfig(rank=10, oversample=5, power=2, seed=4,
                                                 precision=X.Precision.SINGLE))
    ref = OP.rsvd_reorth(arr, 10, 5, 2, 4, "single", fast=True)
    assert res.u.to_array().dtype == np.float32
    assert M.sigma_rel(res.s, ref.s) <= SIG32
    assert M.sin_angle(res.u.to_array(), ref.u) <= ANG32
