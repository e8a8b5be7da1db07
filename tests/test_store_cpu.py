"""Durable-plan formats and PlanRunner semantics on the CPU (no device).

Block files and encoded tiles are pinned byte-for-byte against exports the
REAL reference wrote (tests/golden/make_golden_store.py -> store.npz);
store/record/resume behaviour follows the reference's tests of
src/store.py and src/pipeline.py:163-253, 880-934.
"""

import json
import os

import numpy as np
import pytest

from paper_1907_06470_b200 import (BlockCorruptError, BlockPool, BlockStore, ConfigMismatchError,
                                   FormatError, PlanNotFoundError, PlanRunner, Precision,
                                   RsvdConfig, StageClock, matrix_from_coo, matrix_from_dense,
                                   read_block_file, resume, write_block_file)
from paper_1907_06470_b200.store import decode_block, encode_block

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "store.npz"))


def _gold_mats(pool):
    return {
        "d64": matrix_from_dense(pool, "U", GOLD["dense64"], precision=Precision.DOUBLE),
        "d32": matrix_from_dense(pool, "V", GOLD["dense32"], precision=Precision.SINGLE),
        "sp": matrix_from_coo(pool, "A", 50, 70, GOLD["sp_r"], GOLD["sp_c"], GOLD["sp_v"],
                              precision=Precision.DOUBLE),
    }


@pytest.mark.parametrize("key", ["d64", "d32", "sp"])
def test_block_file_bytes_match_reference(tmp_path, key):
    mat = _gold_mats(BlockPool())[key]
    assert encode_block(mat.desc.matrix_id, mat.tile(0, 0)) == bytes(GOLD[f"enc_{key}"])
    path = tmp_path / f"{key}.blk"
    write_block_file(str(path), mat)
    assert path.read_bytes() == bytes(GOLD[f"blk_{key}"])


@pytest.mark.parametrize("key", ["d64", "d32", "sp"])
def test_read_reference_block_file(tmp_path, key):
    path = tmp_path / "ref.blk"
    path.write_bytes(bytes(GOLD[f"blk_{key}"]))
    want = _gold_mats(BlockPool())[key]
    got = read_block_file(str(path), BlockPool(), "X")
    assert got.desc.matrix_id == "X" and got.shape == want.shape
    assert got.desc.partition == want.desc.partition
    np.testing.assert_array_equal(got.to_array(), want.to_array())


def test_reference_plan_exports_read_back(tmp_path):
    """U/S/V exports of a whole reference run_command('rsvd') plan load here,
    and re-exporting them reproduces the reference's bytes."""
    for name in ("U", "S", "V"):
        ref = bytes(GOLD[f"plan_{name}_blk"])
        (tmp_path / "in.blk").write_bytes(ref)
        mat = read_block_file(str(tmp_path / "in.blk"), BlockPool())
        write_block_file(str(tmp_path / "out.blk"), mat)
        assert (tmp_path / "out.blk").read_bytes() == ref
    s = read_block_file(str(tmp_path / "in.blk"), BlockPool())  # V, any matrix
    assert s.desc.precision is Precision.DOUBLE


def test_descriptor_file_matches_reference(tmp_path):
    want = json.loads(bytes(GOLD["plan_U_json"]).decode())
    store = BlockStore(str(tmp_path))
    pool = BlockPool(store)
    matrix_from_dense(pool, "U", np.zeros((want["rows"], want["cols"])), precision=Precision.DOUBLE)
    raw = (tmp_path / "matrices" / "U.json").read_bytes()
    assert raw == bytes(GOLD["plan_U_json"])


def test_corrupt_and_truncated_blocks(tmp_path):
    mat = _gold_mats(BlockPool())["d64"]
    raw = bytearray(encode_block("U", mat.tile(0, 0)))
    raw[100] ^= 1
    with pytest.raises(BlockCorruptError, match="checksum"):
        decode_block(bytes(raw))
    with pytest.raises(BlockCorruptError, match="shorter"):
        decode_block(bytes(raw[:10]))
    path = tmp_path / "t.blk"
    path.write_bytes(bytes(GOLD["blk_d64"])[:-5])
    with pytest.raises(FormatError, match="truncated"):
        read_block_file(str(path), BlockPool())
    path.write_bytes(b"NOTABLK!\n")
    with pytest.raises(FormatError, match="not a block-file"):
        read_block_file(str(path), BlockPool())


def test_pool_flush_and_reload(tmp_path):
    store = BlockStore(str(tmp_path))
    pool = BlockPool(store)
    arr = np.arange(12.0).reshape(4, 3)
    matrix_from_dense(pool, "M", arr, precision=Precision.DOUBLE, grid=(2, 1))
    assert not store.has_block("M", 0, 0)
    pool.flush_matrix("M", evict=True)
    assert store.has_block("M", 0, 0) and store.has_block("M", 1, 0)
    pool2 = BlockPool(store)
    desc = pool2.register(store.load_descriptor("M"))
    from paper_1907_06470_b200 import StoredMatrix

    np.testing.assert_array_equal(StoredMatrix(desc, pool2).to_array(), arr)


def _runner(tmp_path, completed=None, plan="p1"):
    store = BlockStore(str(tmp_path))
    pool = BlockPool(store)
    return PlanRunner(store, pool, plan, StageClock(), completed=completed), store, pool


def test_plan_runner_records_and_replay(tmp_path):
    runner, store, pool = _runner(tmp_path)
    calls = []

    def make(name, value):
        def fn():
            calls.append(name)
            matrix_from_dense(pool, name, np.full((2, 2), value), precision=Precision.DOUBLE)
            return {"value": value}
        return fn

    runner.step("a", stage="SVD0", fn=make("X", 1.0), outputs=["X"])
    runner.step("b", stage="SVD0", fn=make("Y", 2.0), outputs=["Y"])
    recs = store.scan_plan()
    assert [r.status for r in recs.values()] == ["done", "done"]
    assert recs[1].meta == {"value": 2.0} and recs[0].outputs == ["X"]

    # replay: done steps return their meta without running; outputs load from the store
    done = {k: r for k, r in store.scan_plan().items() if r.status == "done"}
    r2, _, _ = _runner(tmp_path, completed=done)
    assert r2.step("a", stage="SVD0", fn=make("X", 9.0), outputs=["X"]) == {"value": 1.0}
    # a different op at the same slot reruns
    assert r2.step("other", stage="SVD0", fn=make("Y", 3.0), outputs=["Y"]) == {"value": 3.0}
    assert calls == ["X", "Y", "Y"]
    np.testing.assert_array_equal(r2.matrix("X").to_array(), np.full((2, 2), 1.0))


def test_scan_plan_downgrades_damaged_outputs(tmp_path):
    runner, store, pool = _runner(tmp_path)
    runner.step("a", stage="SVD0", outputs=["X"],
                fn=lambda: matrix_from_dense(pool, "X", np.eye(3), precision=Precision.DOUBLE)
                and {})
    assert store.scan_plan()[0].status == "done"
    path = store.block_path("X", 0, 0)
    raw = bytearray(open(path, "rb").read())
    raw[-1] ^= 0xFF
    open(path, "wb").write(bytes(raw))
    assert store.scan_plan()[0].status == "pending"
    with open(os.path.join(store.plan_dir, "step_00001.json"), "w") as f:
        f.write("{not json")
    assert store.scan_plan()[1].status == "pending"


def test_resume_refusals(tmp_path):
    with pytest.raises(PlanNotFoundError):
        resume(str(tmp_path / "nothing"))
    cfg = RsvdConfig(rank=3, oversample=2, power=1, seed=5, workdir=str(tmp_path))
    store = BlockStore(str(tmp_path))
    store.save_plan_config({"command": "rsvd", "input": "x", "output": "y", "threads": 1,
                            "config": cfg.to_json(), "digest": cfg.digest()})
    with pytest.raises(ConfigMismatchError, match="differs"):
        resume(str(tmp_path), RsvdConfig(rank=4, oversample=2, power=1, seed=5))
    saved = store.load_plan_config()
    saved["digest"] = "0" * 64
    store.save_plan_config(saved)
    with pytest.raises(ConfigMismatchError, match="recorded digest"):
        resume(str(tmp_path))
    with open(os.path.join(store.plan_dir, "config.json"), "w") as f:
        f.write("garbage")
    with pytest.raises(PlanNotFoundError, match="unreadable"):
        resume(str(tmp_path))


def test_config_json_round_trip():
    cfg = RsvdConfig(rank=7, oversample=3, power="auto", q_max=4, tau=1e-5, seed=9,
                     precision=Precision.SINGLE, gram_path=True)
    back = RsvdConfig.from_json(cfg.to_json())
    assert back.digest() == cfg.digest()


def test_truncation_fuzz_never_returns_wrong_data(tmp_path):
    """Any prefix of a stored sparse tile is corrupt or absent, never data
    (reference tests/test_store.py:98-110)."""
    from paper_1907_06470_b200 import BlockAbsentError

    store = BlockStore(str(tmp_path))
    mat = _gold_mats(BlockPool())["sp"]
    store.store_block("s", 0, 0, mat.tile(0, 0))
    path = store.block_path("s", 0, 0)
    raw = open(path, "rb").read()
    rng = np.random.default_rng(4)
    for cut in list(rng.integers(0, len(raw), 30)) + [0, 63, 64, len(raw) - 1]:
        open(path, "wb").write(raw[:int(cut)])
        with pytest.raises((BlockCorruptError, BlockAbsentError)):
            store.load_block("s", 0, 0)
    open(path, "wb").write(raw)
    np.testing.assert_array_equal(store.load_block("s", 0, 0).values, mat.tile(0, 0).values)


def test_crash_at_every_barrier_is_conservative(tmp_path):
    """A kill at any write barrier never leaves a done record without intact
    outputs (reference tests/test_store.py:204-243)."""
    from paper_1907_06470_b200 import Density, MatrixDescriptor, StepRecord

    class Crash(Exception):
        pass

    def write_all(store):
        store.save_descriptor(MatrixDescriptor("m", 4, 4, Density.DENSE, Precision.DOUBLE))
        from paper_1907_06470_b200 import DenseBlock

        store.store_block("m", 0, 0, DenseBlock(0, 4, 0, 4, np.eye(4)))
        store.write_step(StepRecord("p", 0, "op", [], ["m"], status="done"))

    seen = []
    probe = BlockStore(str(tmp_path / "probe"))
    probe.fault_hook = lambda name, path: seen.append(name)
    write_all(probe)
    assert {"payload-written", "payload-synced", "payload-visible", "record-written",
            "record-synced", "record-visible"} <= set(seen)
    for i, target in enumerate(seen):
        store = BlockStore(str(tmp_path / f"crash_{i}"))
        count = [0]

        def hook(name, path, i=i):
            if count[0] == i:
                raise Crash()
            count[0] += 1

        store.fault_hook = hook
        with pytest.raises(Crash):
            write_all(store)
        store.fault_hook = None
        recs = store.scan_plan()
        assert 0 not in recs or recs[0].status != "done" or store.verify_block("m", 0, 0)
