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


def test_wide_dynamic_range_rows_stay_on_dmma(lib):
    """Rows whose max towers over their RMS would lose relative accuracy in
    fixed-point slices: the engine's range guard keeps such an A on DMMA, and
    the factorisation still meets the f64 targets."""
    import numpy as np

    from oracle import metrics as M
    from oracle import pipeline as OP

    rng = np.random.default_rng(11)
    m = n = 4096  # m n = 2^24: the int8 path's size threshold
    a = rng.standard_normal((m, 40)) @ rng.standard_normal((40, n))
    a[np.arange(m), rng.integers(0, n, m)] *= 1e4  # one dominant entry per row
    u, s, v, _, _ = lib.rsvd_dense(a, 30, 10, 1, 5)
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
