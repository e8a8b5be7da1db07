"""CPU-only checks of the boundary: the C-ABI library loads, exports every
symbol include/xsvd_b200.h declares, the Python bindings cover them, and the
host-side mirror of the reference interface behaves like the reference
(validation, errors, pool semantics). No compute calls (no GPU here)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "xsvd_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("xb_create", "xb_destroy", "xb_rsvd_dense", "xb_rsvd_dense_dev", "xb_gemm",
                 "xb_thin_qr", "xb_svd_small", "xb_gaussian", "xb_last_error"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    import __graft_entry__

    __graft_entry__.build()
    from paper_1907_06470_b200 import _lib

    lib = _lib.lib_handle()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_symbols())
    assert lib.xb_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_1907_06470_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    """The product path must fail loudly, not compute on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1907_06470_b200 as X

    pool = X.BlockPool()
    a = X.matrix_from_dense(pool, "A", np.eye(4), precision=X.Precision.DOUBLE)
    with pytest.raises(X.XsvdError):
        X.randomized_svd(pool, a, X.RsvdConfig(rank=2, power=0))


def test_config_validation_mirrors_reference():
    from paper_1907_06470_b200 import RsvdConfig

    with pytest.raises(ValueError):
        RsvdConfig(rank=0)
    with pytest.raises(ValueError):
        RsvdConfig(rank=1, power=6)
    with pytest.raises(ValueError):
        RsvdConfig(rank=1, power="fixed")
    with pytest.raises(ValueError):
        RsvdConfig(rank=1, oversample=-1)
    c = RsvdConfig(rank=3, power=2, seed=5)
    assert len(c.digest()) == 64


def test_shape_error_before_any_device_work():
    import paper_1907_06470_b200 as X

    pool = X.BlockPool()
    a = X.matrix_from_dense(pool, "A", np.zeros((10, 8)), precision=X.Precision.DOUBLE)
    with pytest.raises(X.ShapeError):
        X.randomized_svd(pool, a, X.RsvdConfig(rank=8, oversample=1, power=0))


def test_status_mapping():
    from paper_1907_06470_b200 import errors as E

    for status, cls in ((1, E.ShapeError), (2, ValueError), (3, E.BudgetError),
                        (4, E.ConvergenceError), (5, E.XsvdError), (7, E.XsvdError)):
        with pytest.raises(cls):
            E.raise_for_status(status, "x")


def test_pool_mirror_round_trip():
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(0)
    arr = rng.standard_normal((9, 7))
    pool = X.BlockPool()
    m = X.matrix_from_dense(pool, "m", arr, precision=X.Precision.DOUBLE, grid=(3, 2))
    assert np.array_equal(m.to_array(), arr)
    assert np.array_equal(m.T.to_array(), arr.T)
    assert m.T.shape == (7, 9)
    sp = X.matrix_from_coo(pool, "s", 4, 5, [0, 0, 3], [1, 1, 4], [1.0, 2.0, 5.0],
                           precision=X.Precision.DOUBLE)
    dense = sp.to_array()
    assert dense[0, 1] == 3.0 and dense[3, 4] == 5.0 and sp.desc.nnz == 2


def test_results_register_in_a_reference_pool():
    """Outputs go to the CALLER's pool; with the reference importable here,
    register into xsvd's own BlockPool through its own matrix_from_dense."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import xsvd
    except ImportError:
        pytest.skip("reference not importable")
    from paper_1907_06470_b200.pool import register_dense

    pool = xsvd.BlockPool()
    m = register_dense(pool, "U", np.ones((3, 2)), "double")
    assert isinstance(m, xsvd.StoredMatrix)
    assert np.array_equal(m.to_array(), np.ones((3, 2)))


def test_workload_shapes():
    from paper_1907_06470_b200.workloads import CONFIGS, spectrum

    assert CONFIGS[2].m * CONFIGS[2].n * 8 == 8 * 2**30
    assert CONFIGS[1].l == 30 and CONFIGS[2].l == 120 and CONFIGS[5].l == 550
    s = spectrum("pow-1.5", 4)
    assert s[0] == 1.0 and abs(s[3] - 4 ** -1.5) < 1e-16


def test_coo_sorted_check_runs_without_a_device():
    """xb_coo_sorted (host threads, no CUDA call): the SparseBlock invariant
    of core.py:245-284 — strictly increasing (row, col)."""
    import ctypes as C

    from paper_1907_06470_b200 import _lib

    lib = _lib.lib_handle()
    rng = np.random.default_rng(0)
    n = 3_000_000
    rows = np.sort(rng.integers(0, 50_000, n)).astype(np.int64)
    cols = np.zeros(n, dtype=np.int64)
    # strictly increasing columns inside every row
    start = np.flatnonzero(np.r_[True, rows[1:] != rows[:-1]])
    cols = np.arange(n, dtype=np.int64) - np.repeat(start, np.diff(np.r_[start, n]))
    ok = C.c_int(-1)
    assert lib.xb_coo_sorted(rows.ctypes.data, cols.ctypes.data, n, C.byref(ok)) == 0
    assert ok.value == 1
    for pos in (1, n // 2, n - 1):
        c2 = cols.copy()
        r2 = rows.copy()
        r2[pos], c2[pos] = r2[pos - 1], c2[pos - 1]  # a duplicate entry
        assert lib.xb_coo_sorted(r2.ctypes.data, c2.ctypes.data, n, C.byref(ok)) == 0
        assert ok.value == 0
    r, c, v = _lib.Context._coo(rows[::-1], cols[::-1], np.ones(n))
    assert np.array_equal(r, rows) and np.array_equal(c, cols)
