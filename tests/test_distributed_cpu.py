"""Multi-rank host logic on CPU (gloo, world_size 2).

The CUDA engine's sharded path (xb_rsvd_dense_sharded_dev) cannot run two
ranks on this CPU box, and two NCCL ranks on one GPU would wait on each
other (forbidden on the GPU box). So this test checks, with real gloo
processes: (1) the row partition, (2) the unique-id broadcast plumbing, and
(3) that the engine's exchange pattern — Grams of the row-sharded sketch
summed over ranks, A_g^T Q_g partials summed, n-side QRs and the small SVD
replicated — reproduces the single-process oracle. The numpy model below
mirrors rsvd_impl in csrc/engine.cu step for step (test infrastructure).
"""

import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP
from oracle import rng as R


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cholqr(y, allreduce, passes):
    rr = np.eye(y.shape[1])
    for _ in range(passes):
        g = y.T @ y
        if allreduce is not None:
            g = allreduce(g)
        r = np.linalg.cholesky(g).T
        y = np.linalg.solve(r.T, y.T).T
        rr = r @ rr
    return y, rr


def sharded_model(a_local, n, k, p, q, seed, allreduce):
    """The engine's row-sharded schedule (engine.cu rsvd_impl, sharded=true)."""
    l = k + p
    om = R.gaussian_band(seed, 0, n, l)
    y = a_local @ om
    qm, _ = _cholqr(y, allreduce, 1 if q else 2)
    for it in range(q):
        z = allreduce(a_local.T @ qm)
        qz, _ = _cholqr(z, None, 1)
        y = a_local @ qz
        qm, _ = _cholqr(y, allreduce, 2 if it == q - 1 else 1)
    bt = allreduce(a_local.T @ qm)
    qb, rb = _cholqr(bt, None, 2)
    ub, s, wt = np.linalg.svd(rb.T)
    w = wt.T
    for j in range(l):  # sign rule, kernels.py:556-561
        i = int(np.argmax(np.abs(ub[:, j])))
        if ub[i, j] < 0:
            ub[:, j] *= -1
            w[:, j] *= -1
    return qm @ ub[:, :k], s[:k], qb @ w[:, :k]


def colsharded_model(a_local, col0, n_global, k, p, q, seed, allreduce):
    """The engine's column-sharded schedule (engine.cu rsvd_impl, col_shard):
    Y partials all-reduced, m-side QRs replicated, n-side Grams all-reduced,
    A_g^T Q local; U replicated, V for this rank's columns."""
    l = k + p
    n_local = a_local.shape[1]
    om = R.gaussian_band(seed, 0, n_global, l)[col0:col0 + n_local]
    y = allreduce(a_local @ om)
    qm, _ = _cholqr(y, None, 1 if q else 2)
    for it in range(q):
        z = a_local.T @ qm
        qz, _ = _cholqr(z, allreduce, 1)
        y = allreduce(a_local @ qz)
        qm, _ = _cholqr(y, None, 2 if it == q - 1 else 1)
    bt = a_local.T @ qm
    qb, rb = _cholqr(bt, allreduce, 2)
    ub, s, wt = np.linalg.svd(rb.T)
    w = wt.T
    for j in range(l):  # sign rule, kernels.py:556-561
        i = int(np.argmax(np.abs(ub[:, j])))
        if ub[i, j] < 0:
            ub[:, j] *= -1
            w[:, j] *= -1
    return qm @ ub[:, :k], s[:k], qb @ w[:, :k]


def _worker(rank, world, port, out_dir, m, n, k, p, q, seed, layout="rows"):
    import torch
    import torch.distributed as dist

    from paper_1907_06470_b200.distributed import broadcast_bytes, row_shards
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = broadcast_bytes(bytes(range(128)) if rank == 0 else None)
        assert uid == bytes(range(128))
        a = dense_lowrank_np(m, n, "pow-1.5", 1e-8, 91, 92)

        def allreduce(x):
            t = torch.from_numpy(np.ascontiguousarray(x))
            dist.all_reduce(t)
            return t.numpy()

        if layout == "rows":
            r0, r1 = row_shards(m, world)[rank]
            u, s, v = sharded_model(a[r0:r1], n, k, p, q, seed, allreduce)
        else:
            from paper_1907_06470_b200.distributed import col_shards

            r0, r1 = col_shards(n, world)[rank]
            u, s, v = colsharded_model(a[:, r0:r1], r0, n, k, p, q, seed, allreduce)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=u, s=s, v=v, r0=r0, r1=r1)
    finally:
        dist.destroy_process_group()


def test_row_shards():
    from paper_1907_06470_b200.distributed import row_shards

    assert row_shards(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert row_shards(65536, 8)[-1] == (57344, 65536)
    with pytest.raises(ValueError):
        row_shards(2, 3)


def test_sharded_schedule_matches_oracle_gloo():
    import torch.multiprocessing as mp

    m, n, k, p, q, seed, world = 900, 300, 20, 10, 2, 4, 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, m, n, k, p, q, seed), nprocs=world,
                 join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    u = np.vstack([pt["u"] for pt in parts])
    # replicated outputs are bitwise identical across ranks
    assert np.array_equal(parts[0]["s"], parts[1]["s"])
    assert np.array_equal(parts[0]["v"], parts[1]["v"])
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(m, n, "pow-1.5", 1e-8, 91, 92)
    ref = OP.rsvd_reorth(a, k, p, q, seed, "double", fast=True)
    assert M.sigma_rel(parts[0]["s"], ref.s) <= 1e-10
    assert M.sin_angle(u, ref.u) <= 1e-8
    assert M.sin_angle(parts[0]["v"], ref.v) <= 1e-8


def test_colsharded_schedule_matches_oracle_gloo():
    """Config 5's layout: columns of a wide A split over 2 gloo ranks."""
    import torch.multiprocessing as mp

    m, n, k, p, q, seed, world = 300, 900, 20, 10, 2, 4, 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, m, n, k, p, q, seed, "cols"),
                 nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(world)]
    v = np.vstack([pt["v"] for pt in parts])
    assert np.array_equal(parts[0]["s"], parts[1]["s"])
    assert np.array_equal(parts[0]["u"], parts[1]["u"])
    from paper_1907_06470_b200.workloads import dense_lowrank_np

    a = dense_lowrank_np(m, n, "pow-1.5", 1e-8, 91, 92)
    ref = OP.rsvd_reorth(a, k, p, q, seed, "double", fast=True)
    assert M.sigma_rel(parts[0]["s"], ref.s) <= 1e-10
    assert M.sin_angle(parts[0]["u"], ref.u) <= 1e-8
    assert M.sin_angle(v, ref.v) <= 1e-8
