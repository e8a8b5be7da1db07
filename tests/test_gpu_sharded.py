"""The NCCL row-sharded entry point on one GPU (world = 1).

Only one GPU is available to the tests, and two NCCL ranks on one GPU would
wait on each other, so the exchange pattern with world = 2 is checked on CPU
(tests/test_distributed_cpu.py). Here the real NCCL communicator (world 1)
runs every all-reduce of the sharded schedule through the C ABI; with one
rank the sums are identities, so the results must equal the unsharded path
bit for bit.
"""

import os
import socket

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture(scope="module")
def world1(lib):
    import torch.distributed as dist

    from paper_1907_06470_b200.distributed import init_comm

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    init_comm(lib)
    yield lib
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sharded_world1_equals_unsharded(world1, dtype):
    import torch

    from paper_1907_06470_b200.distributed import randomized_svd_sharded
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    npdt = np.float64 if dtype == "float64" else np.float32
    a = dense_lowrank_np(3000, 1200, "pow-1.5", 1e-8, 31, 32).astype(npdt)
    at = torch.from_numpy(a).cuda()
    u, s, v = randomized_svd_sharded(world1, at, 3000, 40, 10, 2, 7)
    # the unsharded device-resident path (same kernels, same split plans)
    u0 = torch.empty_like(u)
    v0 = torch.empty_like(v)
    s0 = torch.empty_like(s)
    world1.rsvd_dense_dev(npdt, 3000, 1200, at.data_ptr(), 1200, 40, 10, 2, 7, u0.data_ptr(),
                          s0.data_ptr(), v0.data_ptr())
    assert torch.equal(s, s0)
    assert torch.equal(u, u0)
    assert torch.equal(v, v0)
    # and the host-buffer path agrees to rounding (its sketch runs in row chunks)
    u1, s1, v1, _, _ = world1.rsvd_dense(a, 40, 10, 2, 7)
    tol = 1e-10 if dtype == "float64" else 1e-4
    assert M.sigma_rel(s.cpu().numpy(), s1) <= tol


def test_sharded_rank_deficient_sketch_uses_tsqr(world1):
    """rank(A) = 8 < l = 20 on the sharded path: the all-reduced Gram's
    Cholesky breaks down on every rank and the sharded TSQR (local tree, R
    all-gather, replicated root) carries the factorisation; identical to the
    unsharded engine at world 1 and to the oracle's leading sigma."""
    import torch

    from paper_1907_06470_b200.distributed import randomized_svd_sharded

    rng = np.random.default_rng(3)
    a = rng.standard_normal((500, 8)) @ rng.standard_normal((8, 300))  # rank 8 < l = 20
    u, s, v = randomized_svd_sharded(world1, torch.from_numpy(a).cuda(), 500, 15, 5, 1, 1)
    ref = OP.rsvd_reorth(a, 15, 5, 1, 1, "double", fast=True)
    s = s.cpu().numpy()
    assert np.max(np.abs(s[:8] - ref.s[:8]) / ref.s[:8]) <= 1e-10
    assert np.max(np.abs(s[8:])) <= 1e-10 * s[0]
    assert M.ortho_defect(u.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_colsharded_world1_equals_unsharded(world1, dtype):
    """Config 5's column layout through NCCL (world 1): identical to the
    unsharded engine (all-reduces are identities, same kernels)."""
    import torch

    from paper_1907_06470_b200.distributed import randomized_svd_colsharded
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    npdt = np.float64 if dtype == "float64" else np.float32
    a = dense_lowrank_np(1100, 3200, "pow-1.5", 1e-8, 41, 42).astype(npdt)
    at = torch.from_numpy(a).cuda()
    u, s, v = randomized_svd_colsharded(world1, at, 3200, 0, 40, 10, 2, 7)
    u0 = torch.empty_like(u)
    v0 = torch.empty_like(v)
    s0 = torch.empty_like(s)
    world1.rsvd_dense_dev(npdt, 1100, 3200, at.data_ptr(), 3200, 40, 10, 2, 7, u0.data_ptr(),
                          s0.data_ptr(), v0.data_ptr())
    assert torch.equal(s, s0)
    assert torch.equal(u, u0)
    assert torch.equal(v, v0)


def test_colsharded_block_offsets_omega(world1):
    """A column block at col0 > 0 uses Omega's rows col0.. (keyed by index):
    the world-1 call on A[:, c0:] equals the oracle run with that Omega block."""
    import torch

    from oracle import pipeline as OP
    from oracle import rng as R
    from paper_1907_06470_b200.distributed import randomized_svd_colsharded
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    m, n, c0, k, p, q, seed = 600, 2000, 700, 20, 10, 1, 3
    a = dense_lowrank_np(m, n, "pow-1.5", 1e-8, 51, 52)
    blk = np.ascontiguousarray(a[:, c0:])
    # world 1 sees only its block: n_global = c0 + block width keeps Omega's rows c0..n-1
    u, s, v = randomized_svd_colsharded(world1, torch.from_numpy(blk).cuda(), n, c0, k, p, q,
                                        seed)
    om = R.gaussian_band(seed, 0, n, k + p)[c0:]
    ref = OP.rsvd_reorth(blk, k, p, q, seed, "double", fast=True, om=om)
    assert M.sigma_rel(s.cpu().numpy(), ref.s) <= 1e-10
    assert M.sin_angle(u.cpu().numpy(), ref.u) <= 1e-8
    assert M.sin_angle(v.cpu().numpy(), ref.v) <= 1e-8
