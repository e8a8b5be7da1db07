"""FP64 products on the int8 tensor cores (ozgemm.cu, Ozaki slices) against
torch f64, through the C ABI's gemm entry with the diagnostics switch
XB_GEMM_OZ=1 (set in a subprocess: the switch is read once per process).
The engine uses this path for dense f64 A with m n >= 2^24; the rSVD-level
parity at that size is tests/test_gpu_parity.py::test_rsvd_vs_oracle_medium."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, %(root)r)
from paper_1907_06470_b200 import _lib
ctx = _lib.load(0)
g = torch.Generator(device="cuda")
g.manual_seed(3)
worst = 0.0
for M, N, K, trans, scale in [(128, 64, 32, False, 1.0), (333, 70, 1000, True, 1e-3),
                              (4096, 120, 20000, False, 1e5), (3000, 100, 40000, True, 1.0),
                              (1000, 552, 3000, False, 1.0)]:
    a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float64)
    # rows of op(A) with wildly different scales exercise the per-row exponents
    sc = torch.logspace(-6, 6, M, device="cuda", dtype=torch.float64) * scale
    a = a * (sc[None, :] if trans else sc[:, None])
    b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float64)
    c = torch.empty(M, N, device="cuda", dtype=torch.float64)
    ctx.gemm_dev(np.float64, trans, M, N, K, a.data_ptr(), a.shape[1], b.data_ptr(), N,
                 c.data_ptr(), N)
    torch.cuda.synchronize()
    op = a.T if trans else a
    ref = op @ b
    den = op.abs() @ b.abs()
    worst = max(worst, float(((c - ref).abs() / den).max()))
print(worst)
"""


def test_ozaki_gemm_accuracy():
    env = dict(os.environ, XB_GEMM_OZ="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.strip().splitlines()[-1])
    # 47 significant bits per operand (S = 6 digit slices): elementwise error
    # relative to |A| |B| measured ~1e-14 (f64 GEMM: ~1e-16)
    assert worst <= 1e-13, worst


def test_wide_dynamic_range_rows_take_a_seventh_slice(lib):
    """Rows whose max towers over their RMS (here ~128x: one entry per row
    scaled by 1e4, n = 16384) would lose accuracy against the RMS scale in
    47-bit fixed-point slices. The engine's range vote gives such an A one
    more digit slice (28 slice pairs instead of 21) instead of leaving the
    int8 pipe, and the factorisation still meets the f64 targets."""
    import numpy as np

    from oracle import metrics as M
    from oracle import pipeline as OP

    rng = np.random.default_rng(11)
    m, n = 2048, 16384
    a = rng.standard_normal((m, 40)) @ rng.standard_normal((40, n))
    a[np.arange(m), rng.integers(0, n, m)] *= 1e4  # one dominant entry per row
    lib.profile(True)
    lib.profile_read()
    u, s, v, _, _ = lib.rsvd_dense(a, 30, 10, 1, 5)
    prof = lib.profile_read()
    lib.profile(False)
    assert prof["kind"] == "ozaki_i8", prof
    # 3 of the 4 products over A run on the slices (the first one overlaps the
    # ingest on DMMA, ops = flops): S (S + 1) / 2 = 28 slice pairs at S = 7,
    # sketch width 40 padded to the 64-column tile
    assert abs(prof["pipe_ops"] / prof["flops"] - (3 * 28 * 64 / 40 + 1) / 4) < 0.5, prof
    ref = OP.rsvd_reorth(a, 30, 10, 1, 5, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10
    assert M.sin_angle(u, ref.u) <= 1e-8
    assert M.sin_angle(v, ref.v) <= 1e-8


def test_moderate_dynamic_range_keeps_six_slices(lib):
    """The same construction at n = 4096: max / RMS <= sqrt(n) = 64, inside
    the 6-slice range (21 slice pairs)."""
    import numpy as np

    from oracle import metrics as M
    from oracle import pipeline as OP

    rng = np.random.default_rng(11)
    m = n = 4096  # m n = 2^24: the int8 path's size threshold
    a = rng.standard_normal((m, 40)) @ rng.standard_normal((40, n))
    a[np.arange(m), rng.integers(0, n, m)] *= 1e4
    lib.profile(True)
    lib.profile_read()
    u, s, v, _, _ = lib.rsvd_dense(a, 30, 10, 1, 5)
    prof = lib.profile_read()
    lib.profile(False)
    assert prof["kind"] == "ozaki_i8", prof
    assert abs(prof["pipe_ops"] / prof["flops"] - (3 * 21 * 64 / 40 + 1) / 4) < 0.5, prof
    ref = OP.rsvd_reorth(a, 30, 10, 1, 5, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10
    assert M.sin_angle(u, ref.u) <= 1e-8
    assert M.sin_angle(v, ref.v) <= 1e-8


SCRIPT_F32 = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, %(root)r)
from paper_1907_06470_b200 import _lib
ctx = _lib.load(0)
g = torch.Generator(device="cuda")
g.manual_seed(4)
worst = 0.0
for M, N, K, trans in [(128, 64, 32, False), (332, 70, 1000, True), (4096, 144, 20000, False),
                       (3000, 200, 40000, True), (1000, 552, 3000, False), (777, 129, 70000, False)]:
    a = torch.randn((K, M) if trans else (M, K), device="cuda", generator=g, dtype=torch.float32)
    sc = torch.logspace(-6, 6, M, device="cuda", dtype=torch.float32)
    a = a * (sc[None, :] if trans else sc[:, None])
    b = torch.randn(K, N, device="cuda", generator=g, dtype=torch.float32)
    c = torch.empty(M, N, device="cuda", dtype=torch.float32)
    ctx.gemm_dev(np.float32, trans, M, N, K, a.data_ptr(), a.shape[1], b.data_ptr(), N,
                 c.data_ptr(), N)
    torch.cuda.synchronize()
    op = (a.T if trans else a).double()
    ref = op @ b.double()
    den = op.abs() @ b.double().abs()
    worst = max(worst, float(((c.double() - ref).abs() / den).max()))
print(worst)
"""


def test_ozaki_f32_gemm_accuracy():
    """float32 A on the int8 pipe (ozf_kernel, 22-bit digits of A made in the
    kernel, 23-bit digits of B) through the diagnostics switch XB_GEMM_OZF=1,
    rows spanning 12 decades of scale."""
    env = dict(os.environ, XB_GEMM_OZF="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT_F32 % {"root": ROOT}], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.strip().splitlines()[-1])
    # elementwise error relative to |A| |B|: 2^-23 of the row scale per A
    # element plus the f32 output rounding (~6e-8); measured <= 2e-6
    assert worst <= 1e-5, worst


def test_f32_wide_dynamic_range_stays_on_tf32(lib):
    """A float32 matrix with a dominant entry per row keeps the 3xTF32 kernel
    (range guard) and still meets the f32 targets."""
    import numpy as np

    from oracle import metrics as M
    from oracle import pipeline as OP

    rng = np.random.default_rng(12)
    m = n = 4096
    a = (rng.standard_normal((m, 30)) @ rng.standard_normal((30, n))).astype(np.float32)
    a[np.arange(m), rng.integers(0, n, m)] *= 1e4
    u, s, v, _, _ = lib.rsvd_dense(a, 20, 10, 1, 5)
    ref = OP.rsvd_reorth(a, 20, 10, 1, 5, "single", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-4
    assert M.sin_angle(u, ref.u) <= 1e-3
