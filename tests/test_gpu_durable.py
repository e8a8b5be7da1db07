"""Durable plans on the device path: run_command / resume
through the GPU factorisation, with exports checked against a whole
`run_command("rsvd")` plan the REAL reference wrote on the same seeded
Matrix Market file (tests/golden/store.npz). Mirrors the reference's
crash/resume tests (XSVD_ABORT_AFTER_STEPS -> exit 70, then resume)."""

import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
from store_inputs import mtx_text  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "store.npz"))


def _mtx(tmp_path):
    seed, m, n = (int(x) for x in GOLD["plan_mtx_seed"])
    path = tmp_path / "a.mtx"
    path.write_text(mtx_text(seed, m, n))
    return str(path)


def _config(workdir):
    import paper_1907_06470_b200 as X

    return X.RsvdConfig(rank=4, oversample=3, power=1, seed=11, precision=X.Precision.DOUBLE,
                        workdir=str(workdir))


def _sine_angle(a, b):
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    return np.linalg.norm(qb - qa @ (qa.T @ qb), 2)


def _check_exports(outdir, tmp_path):
    """Header and descriptor bytes as the reference's; values within the
    north-star tolerances (sigma 1e-10 relative, angle 1e-8)."""
    import paper_1907_06470_b200 as X

    ref_s = np.array([float(x) for x in bytes(GOLD["plan_S_txt"]).decode().split()])
    got_s = np.array([float(x) for x in open(os.path.join(outdir, "S.txt")).read().split()])
    assert got_s.shape == ref_s.shape
    assert np.max(np.abs(got_s - ref_s) / ref_s) <= 1e-10
    for name in ("U", "S", "V"):
        raw = open(os.path.join(outdir, f"{name}.blk"), "rb").read()
        ref = bytes(GOLD[f"plan_{name}_blk"])
        head = ref.index(b"\n", 9) + 1
        assert raw[:head] == ref[:head]  # magic + descriptor line
        assert len(raw) == len(ref)
        # tile length prefix + 64-byte header, checksum (last 8 bytes) aside
        assert raw[head:head + 8 + 56] == ref[head:head + 8 + 56]
        (tmp_path / "ref.blk").write_bytes(ref)
        want = X.read_block_file(str(tmp_path / "ref.blk"), X.BlockPool()).to_array()
        got = X.read_block_file(os.path.join(outdir, f"{name}.blk"), X.BlockPool()).to_array()
        if name == "S":
            np.testing.assert_allclose(got, want, rtol=1e-10)
        else:
            assert _sine_angle(got, want) <= 1e-8


def test_run_command_rsvd_exports_match_reference(lib, tmp_path):
    import paper_1907_06470_b200 as X

    outdir = tmp_path / "out"
    res, pool, runner = X.run_command("rsvd", _mtx(tmp_path), str(outdir),
                                      _config(tmp_path / "work"))
    assert runner.ran == 5  # parse, rsvd-device, export-u, export-s, export-v
    _check_exports(str(outdir), tmp_path)
    recs = X.BlockStore(str(tmp_path / "work")).scan_plan()
    assert [r.op for r in recs.values()] == ["parse", "rsvd-device", "export-u", "export-s",
                                             "export-v"]
    assert all(r.status == "done" for r in recs.values())
    assert recs[1].meta["chosen_q"] == 1 and res.chosen_q == 1


def _run_aborted(tmp_path, after):
    script = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1907_06470_b200 as X\n"
        "cfg = X.RsvdConfig(rank=4, oversample=3, power=1, seed=11, "
        "precision=X.Precision.DOUBLE, workdir=%r)\n"
        "X.run_command('rsvd', %r, %r, cfg)\n"
    ) % (ROOT, str(tmp_path / "work"), _mtx(tmp_path), str(tmp_path / "out"))
    env = dict(os.environ, XSVD_ABORT_AFTER_STEPS=str(after))
    proc = subprocess.run([sys.executable, "-c", script], env=env, cwd=ROOT, timeout=600)
    assert proc.returncode == 70


@pytest.mark.parametrize("after,reran", [(1, 4), (2, 3), (4, 1)])
def test_resume_after_kill(lib, tmp_path, after, reran):
    """Killed between two steps, the plan resumes and runs only what was not
    durably done; exports still match the reference's plan."""
    import paper_1907_06470_b200 as X

    _run_aborted(tmp_path, after)
    res, pool, runner = X.resume(str(tmp_path / "work"))
    assert runner.ran == reran
    _check_exports(str(tmp_path / "out"), tmp_path)
    assert res.chosen_q == 1 and res.s.shape == (4,)


def test_run_command_svd(lib, tmp_path):
    import paper_1907_06470_b200 as X

    seed, m, n = (int(x) for x in GOLD["plan_mtx_seed"])
    outdir = tmp_path / "out"
    res, _, runner = X.run_command("svd", _mtx(tmp_path), str(outdir), _config(tmp_path / "w"))
    a = X.read_block_file(str(outdir / "U.blk"), X.BlockPool()).to_array()
    assert a.shape == (m, min(m, n))
    s = np.array([float(x) for x in (outdir / "S.txt").read_text().split()])
    dense = np.zeros((m, n))
    for line in mtx_text(seed, m, n).splitlines()[2:]:
        i, j, v = line.split()
        dense[int(i) - 1, int(j) - 1] = float(v)
    ref = np.linalg.svd(dense, compute_uv=False)
    assert np.max(np.abs(s - ref)) / ref[0] <= 1e-10


def test_direct_call_on_store_pool_resumes_after_kill(lib, tmp_path):
    """randomized_svd(pool-with-store, A, config) without a runner journals
    its own plan: step 0 ("ingest") makes A durable, so a process killed
    right after it resumes from the workdir alone (pipeline.py:466-485, 924)."""
    import paper_1907_06470_b200 as X

    work = str(tmp_path / "work")
    script = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "import paper_1907_06470_b200 as X\n"
        "cfg = X.RsvdConfig(rank=6, oversample=4, power=1, seed=5, workdir=%r)\n"
        "pool = X.BlockPool(X.BlockStore(%r))\n"
        "arr = np.random.default_rng(2).standard_normal((300, 120))\n"
        "a = X.matrix_from_dense(pool, 'A', arr, precision=X.Precision.DOUBLE)\n"
        "X.randomized_svd(pool, a, cfg)\n"
    ) % (ROOT, work, work)
    env = dict(os.environ, XSVD_ABORT_AFTER_STEPS="1")
    proc = subprocess.run([sys.executable, "-c", script], env=env, cwd=ROOT, timeout=600)
    assert proc.returncode == 70  # killed after the ingest step
    recs = X.BlockStore(work).scan_plan()
    assert [(r.op, r.status) for r in recs.values()] == [("ingest", "done")]
    res, _, runner = X.resume(work)
    assert runner.ran == 1  # only the device step reran
    arr = np.random.default_rng(2).standard_normal((300, 120))
    ref = np.linalg.svd(arr, compute_uv=False)[:6]
    assert res.s.shape == (6,)
    assert np.max(np.abs(res.s - ref) / ref) <= 0.2  # rSVD with q = 1 on a flat spectrum
    from oracle import pipeline as OP

    want = OP.rsvd_reorth(arr, 6, 4, 1, 5, "double", fast=True)
    assert np.max(np.abs(res.s - want.s) / want.s) <= 1e-10
