"""Host ingest of pageable arrays (`-m gpu`): the staging ring of engine.cu
(`HostStager`: worker threads copy the caller's rows into pinned slots, each
slot's DMA behind the fill) must deliver exactly the bytes a pinned source
delivers — contiguous and strided rows, float64 and float32, in-HBM ingest
and the out-of-core streamer.

The reference hands `randomized_svd` plain numpy arrays (pool.py:397-418
`read_cell_dense`); page-locking them per call was measured at 2.4x the copy
itself (profiles/r02_stage_probe.md)."""

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu


def _lowrank(rng, m, n, r, dtype):
    a = (rng.standard_normal((m, r)) * np.logspace(0, -2, r)) @ rng.standard_normal((r, n))
    a += 1e-6 * rng.standard_normal((m, n))
    return a.astype(dtype)


def _pinned_copy(a):
    import torch

    t = torch.empty(a.shape, dtype=torch.float64 if a.dtype == np.float64 else torch.float32,
                    pin_memory=True)
    v = t.numpy()
    v[...] = a
    return t, v


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_staged_equals_pinned_contiguous(lib, dtype):
    """>= 32 MB pageable A through the ring vs the same bytes from pinned
    memory: bitwise identical factors (the device sees identical input)."""
    rng = np.random.default_rng(21)
    m, n = 6144, 1536 if dtype == np.float64 else 3072  # 75 MB
    a = _lowrank(rng, m, n, 40, dtype)
    keep, ap = _pinned_copy(a)
    u1, s1, v1, _, _ = lib.rsvd_dense(a, 24, 8, 1, 3)
    u2, s2, v2, _, _ = lib.rsvd_dense(ap, 24, 8, 1, 3)
    assert np.array_equal(s1, s2) and np.array_equal(u1, u2) and np.array_equal(v1, v2)
    del keep


def test_staged_strided_rows_against_oracle(lib):
    """A is a column window of a wider pageable array (lda > n): the ring
    copies row by row; checked against the oracle and the pinned path."""
    rng = np.random.default_rng(22)
    m, n, pad = 5120, 1100, 57
    wide = np.zeros((m, n + pad))
    wide[:, :n] = _lowrank(rng, m, n, 30, np.float64)
    wide[:, n:] = 7.0  # must never reach the device
    a = wide[:, :n]
    assert a.strides[0] == (n + pad) * 8 and a.nbytes >= 32 << 20
    u, s, v, _, _ = lib.rsvd_dense(a, 20, 8, 2, 4)
    ref = OP.rsvd_reorth(np.ascontiguousarray(a), 20, 8, 2, 4, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= 1e-10
    assert M.sin_angle(u, ref.u) <= 1e-8
    assert M.sin_angle(v, ref.v) <= 1e-8
    keep, ap = _pinned_copy(np.ascontiguousarray(a))
    u2, s2, v2, _, _ = lib.rsvd_dense(ap, 20, 8, 2, 4)
    assert np.array_equal(s, s2) and np.array_equal(u, u2) and np.array_equal(v, v2)
    del keep


def test_streamer_staged_equals_pinned(lib):
    """The out-of-core streamer (forced, small tiles) reads a pageable A
    through the ring on every pass: same factors as from pinned memory."""
    rng = np.random.default_rng(23)
    m, n = 8192, 1024  # 64 MB f64
    a = _lowrank(rng, m, n, 30, np.float64)
    keep, ap = _pinned_copy(a)
    u1, s1, v1, _, _ = lib.rsvd_dense_streamed(a, 16, 8, 2, 5, tile_rows=1024)
    u2, s2, v2, _, _ = lib.rsvd_dense_streamed(ap, 16, 8, 2, 5, tile_rows=1024)
    assert np.array_equal(s1, s2) and np.array_equal(u1, u2) and np.array_equal(v1, v2)
    ref = OP.rsvd_reorth(a, 16, 8, 2, 5, "double", fast=True)
    assert M.sigma_rel(s1, ref.s) <= 1e-10
    del keep
