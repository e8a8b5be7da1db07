"""World-size-2 worker for tests/test_gpu_multirank.py (not a test module).

Two processes share cuda:0 and meet through torch.distributed (gloo on
127.0.0.1). The library's communicator is the host-callback backend
(distributed.init_host_comm), so each rank runs the REAL sharded engine —
xb_rsvd_dense_sharded_dev, xb_rsvd_dense_colsharded_dev and
xb_rsvd_csr_sharded_dev, including the sharded TSQR's R all-gather — and the
ranks exchange partial products on the host. Rank 0 gathers the factors and
writes them to an npz for the parent test to check against the oracle.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def cases():
    from paper_1907_06470_b200.workloads import dense_lowrank_np, sparse_uniform_np

    out = {}
    out["rows_f64"] = ("rows", dense_lowrank_np(6000, 1500, "pow-1.5", 1e-8, 71, 72), 40, 10, 2, 3)
    # m_local * n = 2^24 per rank: the int8-slice (Ozaki) products on each rank
    out["rows_oz"] = ("rows", dense_lowrank_np(16384, 2048, "pow-1.5", 1e-8, 73, 74, 256), 100, 20,
                      2, 2)
    out["cols_f64"] = ("cols", dense_lowrank_np(1200, 5000, "inv", 1e-6, 75, 76, 400), 60, 10, 2, 5)
    out["cols_f32"] = ("cols", dense_lowrank_np(1200, 5000, "inv", 1e-4, 77, 78, 400, np.float32),
                       60, 10, 2, 5)
    rng = np.random.default_rng(79)
    out["rows_deficient"] = ("rows", rng.standard_normal((3000, 12)) @ rng.standard_normal((12, 800)),
                             20, 10, 1, 1)
    rowptr, col, val = sparse_uniform_np(20000, 3000, 20, 80)
    out["csr"] = ("csr", (rowptr, col, val, (20000, 3000)), 50, 10, 3, 3)
    return out


def run(rank: int, world: int, port: int, path: str) -> None:
    import torch
    import torch.distributed as dist

    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200 import distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    ctx = _lib.load(0)
    D.init_host_comm(ctx)
    results = {}
    for name, (layout, a, k, p, q, seed) in cases().items():
        if layout == "rows":
            m, n = a.shape
            r0, r1 = D.row_shards(m, world)[rank]
            u, s, v = D.randomized_svd_sharded(ctx, torch.from_numpy(a[r0:r1]).cuda(), m, k, p, q,
                                               seed)
            parts = [None] * world
            dist.all_gather_object(parts, u.cpu().numpy())
            results[name + "_u"] = np.vstack(parts)
            results[name + "_v"] = v.cpu().numpy()
        elif layout == "cols":
            m, n = a.shape
            c0, c1 = D.col_shards(n, world)[rank]
            u, s, v = D.randomized_svd_colsharded(
                ctx, torch.from_numpy(np.ascontiguousarray(a[:, c0:c1])).cuda(), n, c0, k, p, q,
                seed)
            parts = [None] * world
            dist.all_gather_object(parts, v.cpu().numpy())
            results[name + "_u"] = u.cpu().numpy()
            results[name + "_v"] = np.vstack(parts)
        else:
            rowptr, col, val, (m, n) = a
            r0, r1 = D.row_shards(m, world)[rank]
            lp, lc, lv = D.csr_row_shard(rowptr, col, val, r0, r1)
            u, s, v = D.randomized_svd_csr_sharded(ctx, torch.from_numpy(lp).cuda(),
                                                   torch.from_numpy(lc).cuda(),
                                                   torch.from_numpy(lv).cuda(), m, n, k, p, q,
                                                   seed)
            parts = [None] * world
            dist.all_gather_object(parts, u.cpu().numpy())
            results[name + "_u"] = np.vstack(parts)
            results[name + "_v"] = v.cpu().numpy()
        sv = s.cpu().numpy()
        allsv = [None] * world
        dist.all_gather_object(allsv, sv)
        results[name + "_s"] = sv
        # replicated factors must be bitwise identical on every rank
        results[name + "_s_same"] = np.array(all(np.array_equal(allsv[0], x) for x in allsv))
    if rank == 0:
        np.savez(path, **results)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
