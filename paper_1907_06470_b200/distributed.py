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
