"""The sharded engine at world size 2 on one GPU (`-m gpu`).

Two processes run tests/_multirank_worker.py on cuda:0 and exchange the
sharded factorisation's sums and gathers through the host-callback
communicator over torch.distributed gloo — the real
xb_rsvd_dense_sharded_dev (row blocks, incl. the int8-slice products and a
rank-deficient sketch through the sharded TSQR with its R all-gather),
xb_rsvd_dense_colsharded_dev (column blocks, f64 and f32) and
xb_rsvd_csr_sharded_dev (row-sharded CSR). The assembled factors are
checked against the oracle's xsvd-reorth on the whole A, and
the replicated singular values must be bitwise identical on both ranks.
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SIG64, ANG64 = 1e-10, 1e-8
SIG32, ANG32 = 1e-4, 1e-3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def world2(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("mr") / "out.npz")
    port = _free_port()
    env = dict(os.environ, PYTHONPATH=os.path.dirname(HERE))
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_multirank_worker.py"),
                               str(r), "2", str(port), path], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            out, _ = p.communicate()
        outs.append(out)
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    return np.load(path)


@pytest.mark.parametrize("name", ["rows_f64", "rows_oz", "cols_f64", "cols_f32", "csr"])
def test_world2_matches_oracle(world2, name):
    import _multirank_worker as W

    layout, a, k, p, q, seed = W.cases()[name]
    if layout == "csr":
        rowptr, col, val, shape = a
        rows = np.repeat(np.arange(shape[0]), np.diff(rowptr))
        a = OP.Coo(rows, col.astype(np.int64), val, shape)
    f32 = layout != "csr" and a.dtype == np.float32
    ref = OP.rsvd_reorth(a, k, p, q, seed, "single" if f32 else "double", fast=True)
    sig, ang = (SIG32, ANG32) if f32 else (SIG64, ANG64)
    u, s, v = world2[name + "_u"], world2[name + "_s"], world2[name + "_v"]
    assert bool(world2[name + "_s_same"])
    assert M.sigma_rel(s, ref.s) <= sig
    assert M.sin_angle(u, ref.u) <= ang
    assert M.sin_angle(v, ref.v) <= ang


def test_world2_rank_deficient_sharded_tsqr(world2):
    """rank(A) = 12 < l = 30 on row shards: every rank's all-reduced Gram
    fails its Cholesky, the sharded TSQR (local trees, R all-gather,
    replicated root) orthonormalises; leading sigma match the oracle."""
    import _multirank_worker as W

    _, a, k, p, q, seed = W.cases()["rows_deficient"]
    ref = OP.rsvd_reorth(a, k, p, q, seed, "double", fast=True)
    s, u = world2["rows_deficient_s"], world2["rows_deficient_u"]
    assert bool(world2["rows_deficient_s_same"])
    assert np.max(np.abs(s[:12] - ref.s[:12]) / ref.s[:12]) <= 1e-10
    assert np.max(np.abs(s[12:])) <= 1e-10 * s[0]
    assert M.sin_angle(u[:, :12], ref.u[:, :12]) <= 1e-8
    assert M.ortho_defect(u) <= 1e-12
