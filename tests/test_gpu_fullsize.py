"""Parity at the BENCHMARKED sizes (`-m gpu`): the configurations bench.py
times, factorised through the C ABI with host buffers (the path a reference
caller takes: pageable numpy A in, host U/s/V out) and compared with the
CPU oracle's xsvd-reorth on the same seeded A and Omega.

  cfg2  65536 x 16384 float64, k=100 p=20 q=2   (the default bench line)
  K-split 65536 x 2048 float64                   (A^T Q reduces over K = 65536
                                                  rows: 4 int32 splits over the
                                                  column-slice set inside a
                                                  factorisation)
  cfg3  1e6 x 2e5 CSR, 2e7 nnz, k=100 p=20 q=3   (the whole config)
  cfg5  16384 x 262144 float32 column slice, k=500 p=50 q=3 (1/4 of the
        config's columns: the full 64 GB A plus a host f32 oracle does not fit
        the GPU-test time budget; the kernels, tile shapes and l are the
        config's own)

Each test also asserts which product kernel ran (the profiling counters'
kind): the int8-slice (Ozaki) GEMM for f64, the in-GEMM-sliced f32 GEMM for
cfg5, the CSR SpMM for cfg3 — so a silent fallback fails the test.

Tolerances (north star, BASELINE.json): sigma relative <= 1e-10 (f64) /
1e-4 (f32); largest principal angle (sine form) of U_k, V_k <= 1e-8 (f64) /
1e-3 (f32).
"""

import gc

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SIG64, ANG64 = 1e-10, 1e-8
SIG32, ANG32 = 1e-4, 1e-3


def _torch_dense(m, n, kind, noise, cfg, signal_rank=None, f32=False):
    """The config's seeded construction, built on the GPU (torch) and moved
    to pageable host memory; the device copy is released."""
    import torch

    from paper_1907_06470_b200.workloads import dense_lowrank_torch

    a = dense_lowrank_torch(m, n, kind, noise, cfg, signal_rank,
                            dtype=torch.float32 if f32 else torch.float64, device="cuda")
    host = a.cpu().numpy()
    del a
    torch.cuda.empty_cache()
    return host


def _check(got, ref, sig, ang):
    u, s, v = got
    es = M.sigma_rel(s, ref.s)
    eu = M.sin_angle(u, ref.u)
    ev = M.sin_angle(v, ref.v)
    print(f"sigma rel {es:.3e}  angle U {eu:.3e}  V {ev:.3e}")
    assert es <= sig, es
    assert eu <= ang, eu
    assert ev <= ang, ev


def _factorise(lib, a, k, p, q, seed):
    lib.profile(True)
    lib.profile_read()
    u, s, v, deficient, stages = lib.rsvd_dense(a, k, p, q, seed)
    prof = lib.profile_read()
    lib.profile(False)
    return (u, s, v), deficient, stages, prof


def test_cfg2_full_size(lib):
    """Config 2 exactly as benchmarked: 65536 x 16384 f64, s_i = i^-1.5,
    noise 1e-8, k=100 p=20 q=2, Omega seed 2."""
    from paper_1907_06470_b200.workloads import CONFIGS

    w = CONFIGS[2]
    a = _torch_dense(w.m, w.n, w.spectrum, w.noise, w.cfg)
    got, deficient, stages, prof = _factorise(lib, a, w.k, w.p, w.q, w.cfg)
    # the int8 tensor-core products ran (the first product is computed per
    # ingest chunk as A lands, on DMMA; the other 2q + 1 on the slices)
    assert prof["kind"] == "ozaki_i8", prof
    ref = OP.rsvd_reorth(a, w.k, w.p, w.q, w.cfg, "double", fast=True)
    del a
    gc.collect()
    _check(got, ref, SIG64, ANG64)
    assert deficient == ref.deficient_columns == ()
    assert stages[2] > 0 and stages[0] > 0  # sketch time, overlapped ingest


def test_tn_ksplit_inside_factorisation(lib):
    """65536 x 2048 f64: every A^T Q product reduces over K = 65536 rows, so
    the int32-exact chains split into 4 K ranges summed in f64 in order."""
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(65536, 2048, "pow-1.5", 1e-8, 1002, 2002)
    got, _, _, prof = _factorise(lib, a, 100, 20, 2, 2)
    assert prof["kind"] == "ozaki_i8", prof
    ref = OP.rsvd_reorth(a, 100, 20, 2, 2, "double", fast=True)
    _check(got, ref, SIG64, ANG64)


def test_cfg3_full_size(lib):
    """Config 3 exactly as benchmarked: 1e6 x 2e5 CSR, 20 distinct uniform
    columns per row (nnz 2e7), N(0,1) values, k=100 p=20 q=3, Omega seed 3;
    oracle products through scipy CSR."""
    from paper_1907_06470_b200.workloads import CONFIGS, sparse_uniform_np

    w = CONFIGS[3]
    rowptr, col, val = sparse_uniform_np(w.m, w.n, 20, 3000 + w.cfg)
    rows = np.repeat(np.arange(w.m, dtype=np.int64), np.diff(rowptr))
    cols = col.astype(np.int64)
    lib.profile(True)
    lib.profile_read()
    u, s, v, deficient, _ = lib.rsvd_coo(rows, cols, val, (w.m, w.n), w.k, w.p, w.q, w.cfg)
    prof = lib.profile_read()
    lib.profile(False)
    assert prof["kind"] == "spmm", prof
    ref = OP.rsvd_reorth(OP.Coo(rows, cols, val, (w.m, w.n)), w.k, w.p, w.q, w.cfg, "double",
                         fast=True)
    del rows, cols, val, rowptr, col
    gc.collect()
    _check((u, s, v), ref, SIG64, ANG64)
    assert deficient == ref.deficient_columns


def test_cfg5_column_slice(lib):
    """Config 5's construction (rank-1000 signal s_i = 1/i, noise 1e-4,
    float32) at 16384 x 262144 (a quarter of its columns), k=500 p=50 q=3:
    the float32 products on the int8 pipe with the config's l = 550."""
    a = _torch_dense(16384, 262144, "inv", 1e-4, 5, 1000, f32=True)
    got, _, _, prof = _factorise(lib, a, 500, 50, 3, 5)
    assert prof["kind"] == "ozaki_f32_i8", prof
    ref = OP.rsvd_reorth(a, 500, 50, 3, 5, "single", fast=True)
    del a
    gc.collect()
    _check(got, ref, SIG32, ANG32)
