"""Sharding of A over GPUs, one process per GPU.

The reference has no distributed path; these are the north star's
multi-GPU layouts:

* row blocks (tall A, configs 2-4): rank g holds rows R_g of A
  (m_global x n). Y_g = A_g Omega and Y_g = A_g Z need no communication; the
  n x l partials of A^T Q and the l x l Grams of the row-sharded sketch are
  summed by NCCL all-reduce inside the library (xb_rsvd_dense_sharded_dev).
* column blocks (wide A, config 5): rank g holds columns C_g of A
  (m x n_global) and the matching rows of Omega. The m x l partials of
  A_g X_g are all-reduced, A_g^T Q is local, and the l x l Grams of the
  row-sharded n-side sketches are all-reduced (xb_rsvd_dense_colsharded_dev).

torch.distributed is only the plumbing that carries the NCCL unique id.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def row_shards(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced row blocks (the reference's equal-cut rule,
    core.py:90-98): the first m % world blocks get one extra row."""
    if world < 1 or m < world:
        raise ValueError(f"cannot split {m} rows over {world} ranks")
    q, rem = divmod(m, world)
    cuts = [0]
    for g in range(world):
        cuts.append(cuts[-1] + q + (1 if g < rem else 0))
    return [(cuts[g], cuts[g + 1]) for g in range(world)]


def col_shards(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced column blocks (same cut rule as row_shards)."""
    return row_shards(n, world)


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from `src` over torch.distributed."""
    import torch.distributed as dist

    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def init_comm(ctx: "_lib.Context", group=None) -> None:
    """Create the library's NCCL communicator over the torch.distributed world."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = ctx.comm_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid, 0, group)
    ctx.comm_init(uid, world, rank)


def init_host_comm(ctx: "_lib.Context", group=None) -> None:
    """Create the library's communicator on top of torch.distributed itself
    (any backend, e.g. gloo): every exchange is a host all-reduce /
    all-gather of the operand (xb_comm_init_host). Ranks meet only on the
    host, so several processes may share one GPU — how the sharded engine is
    tested on a single-GPU box. Production runs use init_comm (NCCL)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def collective(op: int, buf: np.ndarray) -> None:
        t = torch.from_numpy(buf)
        if op == _lib.COLL_ALLREDUCE_SUM:
            dist.all_reduce(t, group=group)
        else:
            parts = list(t.chunk(world))
            mine = parts[rank].clone()
            dist.all_gather(parts, mine, group=group)

    ctx.comm_init_host(world, rank, collective)


def csr_row_shard(rowptr: np.ndarray, col: np.ndarray, val: np.ndarray, r0: int, r1: int):
    """Rows [r0, r1) of a CSR matrix as a CSR of their own (rowptr rebased)."""
    a, b = int(rowptr[r0]), int(rowptr[r1])
    return (np.ascontiguousarray(rowptr[r0:r1 + 1] - a, dtype=np.int64),
            np.ascontiguousarray(col[a:b], dtype=np.int32), np.ascontiguousarray(val[a:b]))


def randomized_svd_csr_sharded(ctx, rowptr, col, val, m_global: int, n: int, k: int, p: int,
                               q: int, seed: int):
    """Factorise the row-sharded sparse A: this rank's rows as device CSR
    (torch tensors: rowptr int64 rebased to the rank's first row, col int32,
    val float64). Returns (U_local, s, V) as torch tensors."""
    import torch

    m_local = rowptr.numel() - 1
    dev = val.device
    u = torch.empty((m_local, k), dtype=torch.float64, device=dev)
    v = torch.empty((n, k), dtype=torch.float64, device=dev)
    s = torch.empty((k,), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ctx.rsvd_csr_sharded_dev(m_global, n, m_local, val.numel(), rowptr.data_ptr(), col.data_ptr(),
                             val.data_ptr(), k, p, q, seed, u.data_ptr(), s.data_ptr(),
                             v.data_ptr())
    return u, s, v


def randomized_svd_sharded(ctx, a_local, m_global: int, k: int, p: int, q: int, seed: int):
    """Factorise the row-sharded A (this rank's rows as a CUDA torch tensor).

    Returns (U_local, s, V) as torch tensors: U for this rank's rows, s and V
    replicated (bitwise identical on every rank)."""
    import torch

    m_local, n = a_local.shape
    dt = np.float64 if a_local.dtype == torch.float64 else np.float32
    u = torch.empty((m_local, k), dtype=a_local.dtype, device=a_local.device)
    v = torch.empty((n, k), dtype=a_local.dtype, device=a_local.device)
    s = torch.empty((k,), dtype=torch.float64, device=a_local.device)
    a_local = a_local.contiguous()
    torch.cuda.synchronize(a_local.device)
    ctx.rsvd_dense_sharded_dev(dt, m_global, n, m_local, a_local.data_ptr(), n, k, p, q, seed,
                               u.data_ptr(), s.data_ptr(), v.data_ptr())
    return u, s, v


def randomized_svd_colsharded(ctx, a_local, n_global: int, col0: int, k: int, p: int, q: int,
                              seed: int):
    """Factorise the column-sharded A (this rank's columns [col0, col0 + n_local)
    as a CUDA torch tensor, m x n_local).

    Returns (U, s, V_local) as torch tensors: U and s replicated (bitwise
    identical on every rank), V for this rank's columns."""
    import torch

    m, n_local = a_local.shape
    dt = np.float64 if a_local.dtype == torch.float64 else np.float32
    u = torch.empty((m, k), dtype=a_local.dtype, device=a_local.device)
    v = torch.empty((n_local, k), dtype=a_local.dtype, device=a_local.device)
    s = torch.empty((k,), dtype=torch.float64, device=a_local.device)
    a_local = a_local.contiguous()
    torch.cuda.synchronize(a_local.device)
    ctx.rsvd_dense_colsharded_dev(dt, m, n_global, n_local, col0, a_local.data_ptr(), n_local,
                                  k, p, q, seed, u.data_ptr(), s.data_ptr(), v.data_ptr())
    return u, s, v
