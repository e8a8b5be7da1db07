"""rSVD driver: the drop-in for the reference's `randomized_svd`.

  randomized_svd(pool, a, config, *, threads=1, runner=None, clock=None)
      -> RsvdResult(u, s, v, chosen_q, stage_seconds, deficient_columns)
  (reference: src/pipeline.py:442-625; RsvdConfig 78-150; RsvdResult 153-160;
   STAGE_NAMES/StageClock 33-75; gaussian_matrix 259-284)

One call runs the whole factorisation inside libxsvdb200.so
(xb_rsvd_dense): A is streamed host->HBM in row chunks overlapped with the
sketch, then every product, orthonormalisation and the small SVD run on the
device; U, s, V come back and are registered in the CALLER's pool under the
reference's ids "U", "S", "V". The power iteration re-orthonormalises after
every product (the north star; the reference's shipped driver does not,
pipeline.py:321-371 — SURVEY.md F4), so results match the "xsvd-reorth"
oracle. Stage times are device-timed per STAGE_NAMES key.

power="auto" (the reference's default, pipeline.py:295-372) runs on the
device: up to q_max passes, stopped by the reference's rule on
nu_q = ||(A A^T)^q A Omega||_F / sqrt(m l), whose raw-product norms are
carried through the re-orthonormalised iteration as small triangular factors
(engine.cu AutoPower); `auto_select_q` (396-418) is the same loop on a
rank-wide probe. gram_path=True (526-580) projects the power matrix and
factors its Gram on the device too.

Durable plans (pipeline.py:163-253, 722-756, 838-934): with a BlockStore
behind the pool (RsvdConfig.workdir, `run_command`, `resume`), PlanRunner
writes a step record per step and flushes each step's outputs before
marking it done, in the reference's on-disk formats (store.py). The device
factorisation is ONE step ("rsvd-device", outputs U/S/V): it runs in
milliseconds to seconds, so finer records would only add fsyncs. A resumed
plan replays done steps from their records (U/S/V load from the store, the
chosen q from the record's meta) and runs the rest; `_export_steps` writes
U.blk/S.blk/V.blk/S.txt byte-compatible with the reference's exports.
Step ids are our own sequence: a workdir the reference started does not
resume here mid-plan (its op names differ, so its records never match and
every step reruns).
"""

from __future__ import annotations

import hashlib
import json
import os
from contextlib import contextmanager
from dataclasses import dataclass, field
import time

import numpy as np

from . import _lib
from .core import Precision, as_precision
from .errors import ConfigMismatchError, PlanNotFoundError, ShapeError, XsvdError
from .pool import (BlockPool, StoredMatrix, canonical_coo, is_sparse, register_dense,
                   stored_to_array)
from .store import BlockStore, StepRecord, write_block_file

ABORT_ENV = "XSVD_ABORT_AFTER_STEPS"
ABORT_EXIT_CODE = 70


def _abort_after():
    """Test hook: exit between two steps after N of them (pipeline.py:54-60)."""
    raw = os.environ.get(ABORT_ENV)
    return int(raw) if raw else None

STAGE_PARSE = "Text Parsing"
STAGE_GAUSSIAN = "Preparation of O"
STAGE_SKETCH = "O*A^T"
STAGE_ORTHO = "Orthogonalization"
STAGE_PROJECT = "A^T*Q_r"
STAGE_SVD_PREP = "SVD0 Preparation"
STAGE_SVD = "SVD0"
STAGE_POST = "Postprocessing"
STAGE_NAMES = (STAGE_PARSE, STAGE_GAUSSIAN, STAGE_SKETCH, STAGE_ORTHO, STAGE_PROJECT,
               STAGE_SVD_PREP, STAGE_SVD, STAGE_POST)


class StageClock:
    """Accumulator keyed by stage name (pipeline.py:63-75)."""

    def __init__(self):
        self.seconds = {name: 0.0 for name in STAGE_NAMES}

    @contextmanager
    def timing(self, stage: str):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            self.seconds[stage] += time.perf_counter() - t0


@dataclass(frozen=True)
class RsvdConfig:
    """Same fields, defaults and validation as pipeline.py:78-150."""

    rank: int
    power: object = "auto"
    q_max: int = 5
    tau: float = 1e-6
    seed: int = 0
    precision: object = Precision.DOUBLE
    oversample: int = 0
    gram_path: bool = False
    budget: object = None
    workdir: str | None = None

    def __post_init__(self):
        if self.rank < 1:
            raise ValueError(f"rank must be at least 1, got {self.rank}")
        if self.q_max < 0:
            raise ValueError(f"q_max must be nonnegative, got {self.q_max}")
        if isinstance(self.power, str):
            if self.power != "auto":
                raise ValueError(f"power must be 'auto' or an integer, got {self.power!r}")
        elif not 0 <= self.power <= self.q_max:
            raise ValueError(f"power {self.power} outside 0..{self.q_max}")
        if not self.tau > 0:
            raise ValueError(f"tau must be positive, got {self.tau}")
        if self.oversample < 0:
            raise ValueError(f"oversample must be nonnegative, got {self.oversample}")

    def to_json(self) -> dict:
        return {"rank": self.rank, "power": self.power, "q_max": self.q_max, "tau": self.tau,
                "seed": self.seed, "precision": as_precision(self.precision).value,
                "oversample": self.oversample, "gram_path": self.gram_path}

    def digest(self) -> str:
        blob = json.dumps(self.to_json(), sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(blob.encode()).hexdigest()

    @classmethod
    def from_json(cls, d: dict, workdir: str | None = None) -> "RsvdConfig":
        """pipeline.py:134-146 (budget keys, if present, are not used here)."""
        return cls(rank=d["rank"], power=d["power"], q_max=d["q_max"], tau=d["tau"],
                   seed=d["seed"], precision=Precision(d["precision"]),
                   oversample=d["oversample"], gram_path=d["gram_path"], workdir=workdir)


@dataclass
class RsvdResult:
    u: object
    s: np.ndarray
    v: object
    chosen_q: int
    stage_seconds: dict = field(default_factory=dict)
    deficient_columns: tuple = ()


class PlanRunner:
    """Runs plan steps in order, skipping ones already durably done
    (pipeline.py:163-253). Step ids follow call order, so a resumed process
    lines each `step` call up with its prior record; a done step returns its
    recorded meta instead of running."""

    def __init__(self, store, pool, plan_id, clock, *, completed=None, abort_after=None):
        self.store = store
        self.pool = pool
        self.plan_id = plan_id
        self.clock = clock
        self.completed = completed or {}
        self.abort_after = abort_after
        self.next_id = 0
        self.ran = 0

    def step(self, op, *, stage, fn, inputs=(), outputs=(), seed=None, self_clocked=False):
        step_id = self.next_id
        self.next_id += 1
        prior = self.completed.get(step_id)
        if (prior is not None and prior.status == "done" and prior.op == op
                and prior.plan_id == self.plan_id):
            return dict(prior.meta)
        record = StepRecord(self.plan_id, step_id, op, list(inputs), list(outputs), "pending",
                            seed)
        if self.store is not None:
            with self.clock.timing(stage):
                self.store.write_step(record)
        if self_clocked:
            meta = fn() or {}
        else:
            with self.clock.timing(stage):
                meta = fn() or {}
        with self.clock.timing(stage):
            if self.store is not None:
                for matrix_id in outputs:
                    self.pool.flush_matrix(matrix_id)
                record.status = "done"
                record.meta = meta
                self.store.write_step(record)
        self.ran += 1
        if self.abort_after is not None and self.ran >= self.abort_after:
            os._exit(ABORT_EXIT_CODE)  # simulated kill between two steps
        return meta

    def matrix(self, matrix_id):
        """Handle on a step output, produced now or by a prior run."""
        try:
            return StoredMatrix(self.pool.descriptor(matrix_id), self.pool)
        except KeyError:
            if self.store is None:
                raise
            desc = self.pool.register(self.store.load_descriptor(matrix_id))
            return StoredMatrix(desc, self.pool)


def gaussian_matrix(pool, matrix_id, rows, cols, seed, *, precision=Precision.DOUBLE):
    """N(0,1) matrix keyed by (seed, row) (pipeline.py:259-284), generated on
    the device (rng.py restated in csrc/rng.cu)."""
    precision = as_precision(precision)
    dt = np.float64 if precision is Precision.DOUBLE else np.float32
    arr = _lib.load().gaussian(seed, 0, rows, cols, dtype=dt)
    return register_dense(pool, matrix_id, arr.astype(precision.storage_dtype, copy=False),
                          precision)


def _dense_input(a) -> np.ndarray:
    """The caller's A as one row-major host array (zero-copy for an
    unbudgeted single-tile matrix, as SURVEY.md §8a notes)."""
    d = a.desc
    part = d.partition
    if not d.transposed and part.n_row_tiles == 1 and part.n_col_tiles == 1:
        return a.pool.get(d.matrix_id, 0, 0).values
    return np.ascontiguousarray(stored_to_array(a))


def randomized_svd(pool, a, config: RsvdConfig, *, threads: int = 1, runner=None, clock=None):
    """Rank-k randomized factorisation A ~ U diag(s) V^T on the GPU."""
    m, n = a.shape
    r_work = config.rank + config.oversample
    if r_work > min(m, n):
        raise ShapeError(f"rank {config.rank} (+{config.oversample} oversampling) exceeds "
                         f"min{tuple(a.shape)} = {min(m, n)}")
    precision = as_precision(config.precision)
    if precision is Precision.HALF:
        raise XsvdError("half precision (storage-only in the reference) is not built on the GPU path")
    clock = clock or (runner.clock if runner is not None else StageClock())
    store = getattr(pool, "store", None)
    if runner is None and store is not None:
        # a store-backed pool without a runner starts a plan (pipeline.py:466-479)
        runner = PlanRunner(store, pool, config.digest(), clock, abort_after=_abort_after())
        store.save_plan_config({"command": None, "input_matrix": a.matrix_id,
                                "config": config.to_json(), "digest": config.digest()})
    if runner is None:
        u, s, v, deficient, chosen_q = _rsvd_device(a, config, precision, clock)
        register_dense(pool, "S", s.reshape(-1, 1), Precision.DOUBLE)
        umat = register_dense(pool, "U", u, precision)
        vmat = register_dense(pool, "V", v, precision)
        return RsvdResult(u=umat, s=s.astype(np.float64), v=vmat, chosen_q=chosen_q,
                          stage_seconds=dict(clock.seconds), deficient_columns=deficient)

    def device_step():
        u, s, v, deficient, chosen_q = _rsvd_device(a, config, precision, clock)
        register_dense(pool, "S", s.reshape(-1, 1), Precision.DOUBLE)
        register_dense(pool, "U", u, precision)
        register_dense(pool, "V", v, precision)
        return {"chosen_q": int(chosen_q), "deficient": [int(c) for c in deficient]}

    meta = runner.step("rsvd-device", stage=STAGE_SKETCH, inputs=[a.matrix_id],
                       outputs=["U", "S", "V"], seed=config.seed, fn=device_step,
                       self_clocked=True)
    smat = runner.matrix("S")
    return RsvdResult(u=runner.matrix("U"), s=smat.to_array().astype(np.float64).ravel(),
                      v=runner.matrix("V"), chosen_q=int(meta["chosen_q"]),
                      stage_seconds=dict(clock.seconds),
                      deficient_columns=tuple(meta.get("deficient", ())))


def _rsvd_device(a, config, precision, clock):
    """One synchronous xb_rsvd_* call; device stage times go into `clock`."""
    ctx = _lib.load()
    auto = config.power == "auto"
    q = _lib.POWER_AUTO if auto else int(config.power)
    if auto:
        ctx.set_power_auto(config.q_max, config.tau)
    ctx.set_gram_path(config.gram_path)
    try:
        if is_sparse(a):
            if precision is not Precision.DOUBLE:
                raise XsvdError("sparse A is built for float64 only")
            rows, cols, vals = canonical_coo(a)
            if a.desc.transposed:
                rows, cols = cols, rows
            u, s, v, deficient, stages = ctx.rsvd_coo(rows, cols, vals, tuple(a.shape), config.rank,
                                                      config.oversample, q, config.seed)
        else:
            host = _dense_input(a).astype(precision.storage_dtype, copy=False)
            u, s, v, deficient, stages = ctx.rsvd_dense(host, config.rank, config.oversample, q,
                                                        config.seed)
    finally:
        ctx.set_gram_path(False)  # context state must not leak into other calls
    chosen_q = ctx.last_power()[0] if auto else int(config.power)
    for name, sec in zip(STAGE_NAMES, stages):
        clock.seconds[name] += float(sec)
    return u, s, v, tuple(deficient), chosen_q


def auto_select_q(pool, a, rank, *, q_max: int = 5, tau: float = 1e-6, seed: int = 0,
                  threads: int = 1, precision=None) -> int:
    """Pick the power exponent (pipeline.py:396-418): the power="auto" loop
    on a rank-wide probe Omega = gaussian_band(seed, 0, n, rank). Runs on the
    device like randomized_svd; nothing is registered in the pool (the
    reference drops its scratch matrices too)."""
    precision = as_precision(precision or a.desc.precision)
    if precision is Precision.HALF:
        raise XsvdError("half precision (storage-only in the reference) is not built on the GPU path")
    m, n = a.shape
    if rank > min(m, n):
        raise ShapeError(f"rank {rank} exceeds min{tuple(a.shape)} = {min(m, n)}")
    if q_max < 0:
        raise ValueError(f"q_max must be nonnegative, got {q_max}")
    ctx = _lib.load()
    ctx.set_power_auto(q_max, tau)
    ctx.set_gram_path(False)
    if is_sparse(a):
        if precision is not Precision.DOUBLE:
            raise XsvdError("sparse A is built for float64 only")
        rows, cols, vals = canonical_coo(a)
        if a.desc.transposed:
            rows, cols = cols, rows
        ctx.rsvd_coo(rows, cols, vals, tuple(a.shape), rank, 0, _lib.POWER_AUTO, seed)
    else:
        host = _dense_input(a).astype(precision.storage_dtype, copy=False)
        ctx.rsvd_dense(host, rank, 0, _lib.POWER_AUTO, seed)
    return ctx.last_power()[0]


def full_svd(pool, a, config=None, *, threads: int = 1, runner=None, clock=None):
    """Exact thin SVD, no sketching (pipeline.py:628-716), every step on the
    device: thin QR of the tall orientation (CholQR2 with the Householder
    fallback), the SVD of the min(m, n)-square R (Jacobi), and the big factor
    Q U_R (GEMM). Sparse input is densified first (_densify, 419-436). The
    small factor of the tall orientation is V (m >= n) or U (m < n), like
    the reference; results are registered as "U", "S", "V"."""
    m, n = a.shape
    precision = as_precision(config.precision if config is not None else a.desc.precision)
    if precision is Precision.HALF:
        raise XsvdError("half precision (storage-only in the reference) is not built on the GPU path")
    dt = np.float64 if precision is Precision.DOUBLE else np.float32
    clock = clock or (runner.clock if runner is not None else StageClock())

    def compute():
        ctx = _lib.load()
        with clock.timing(STAGE_SVD_PREP):
            arr = np.asarray(stored_to_array(a), dtype=dt)
            tall = np.ascontiguousarray(arr if m >= n else arr.T)
        with clock.timing(STAGE_ORTHO):
            q, r, deficient = ctx.thin_qr(tall)
        with clock.timing(STAGE_SVD):
            u_r, s, v_r = ctx.svd_small(r)
        with clock.timing(STAGE_POST):
            big = ctx.gemm(q, np.ascontiguousarray(u_r, dtype=dt))
        big_id, small_id = ("U", "V") if m >= n else ("V", "U")
        out["S"] = register_dense(pool, "S", np.asarray(s, dtype=np.float64).reshape(-1, 1),
                                  Precision.DOUBLE)
        out[big_id] = register_dense(pool, big_id, big.astype(precision.storage_dtype, copy=False),
                                     precision)
        out[small_id] = register_dense(pool, small_id,
                                       v_r.astype(precision.storage_dtype, copy=False), precision)
        return {"deficient": [int(c) for c in deficient]}

    out = {}
    if runner is None:
        meta = compute()
        get = out.__getitem__
    else:
        meta = runner.step("full-svd-device", stage=STAGE_SVD, inputs=[a.matrix_id],
                           outputs=["U", "S", "V"], fn=compute, self_clocked=True)
        get = runner.matrix
    s_arr = get("S").to_array().astype(np.float64).ravel()
    return RsvdResult(u=get("U"), s=s_arr, v=get("V"), chosen_q=0,
                      stage_seconds=dict(clock.seconds),
                      deficient_columns=tuple(meta.get("deficient", ())))


# -- durable command drivers (pipeline.py:719-934) --------------------------


def _export_steps(runner, outdir):
    """U.blk / S.blk / V.blk and S.txt (%.17g per line), one step each
    (pipeline.py:722-740)."""
    os.makedirs(outdir, exist_ok=True)
    for matrix_id, filename in (("U", "U.blk"), ("S", "S.blk"), ("V", "V.blk")):

        def export(matrix_id=matrix_id, filename=filename):
            mat = runner.matrix(matrix_id)
            write_block_file(os.path.join(outdir, filename), mat)
            if matrix_id == "S":
                values = mat.to_array().astype(np.float64).ravel()
                tmp = os.path.join(outdir, "S.txt.tmp")
                with open(tmp, "w") as f:
                    for value in values:
                        f.write(f"{value:.17g}\n")
                os.replace(tmp, os.path.join(outdir, "S.txt"))
            return {}

        runner.step(f"export-{matrix_id.lower()}", stage=STAGE_POST, inputs=[matrix_id], fn=export)


def _parse_step(runner, pool, config, input_path):
    from .formats import parse_matrix_market

    runner.step("parse", stage=STAGE_PARSE, outputs=["A"],
                fn=lambda: parse_matrix_market(input_path, pool, "A",
                                               precision=config.precision) and {})


def _drive_rsvd(runner, pool, config, threads, input_path, outdir):
    """pipeline.py:743-756."""
    _parse_step(runner, pool, config, input_path)
    result = randomized_svd(pool, runner.matrix("A"), config, threads=threads, runner=runner)
    _export_steps(runner, outdir)
    return result


def _drive_full_svd(runner, pool, config, threads, input_path, outdir):
    """pipeline.py:759-770."""
    _parse_step(runner, pool, config, input_path)
    result = full_svd(pool, runner.matrix("A"), config, threads=threads, runner=runner)
    _export_steps(runner, outdir)
    return result


_DRIVERS = {"rsvd": _drive_rsvd, "svd": _drive_full_svd}


def run_command(command, input_path, output_path, config: RsvdConfig, *, threads: int = 1,
                fresh: bool = True, profile_out=None):
    """One factorisation command with a durable plan in config.workdir
    (pipeline.py:838-877). `fresh` wipes any previous plan first."""
    if config.workdir is None:
        raise ValueError("run_command needs config.workdir for its plan state")
    if command not in _DRIVERS:
        raise XsvdError(f"command {command!r} is not built on the GPU path "
                        f"(have: {', '.join(sorted(_DRIVERS))})")
    clock = StageClock()
    with clock.timing(STAGE_PARSE):
        store = BlockStore(config.workdir)
        if fresh:
            store.clear_plan()
        store.save_plan_config({
            "command": command, "input": os.path.abspath(input_path),
            "output": os.path.abspath(output_path), "threads": threads,
            "profile_out": os.path.abspath(profile_out) if profile_out else None,
            "config": config.to_json(), "digest": config.digest()})
        pool = BlockPool(store, config.budget)
    runner = PlanRunner(store, pool, config.digest(), clock, abort_after=_abort_after())
    result = _DRIVERS[command](runner, pool, config, threads, input_path, output_path)
    result.stage_seconds = dict(clock.seconds)
    return result, pool, runner


def resume(workdir: str, config: RsvdConfig | None = None, *, threads: int | None = None):
    """Finish an interrupted plan; refuses to continue under changed settings
    (pipeline.py:880-934)."""
    if not os.path.exists(os.path.join(workdir, "plan", "config.json")):
        raise PlanNotFoundError(f"no execution plan under {workdir}")
    store = BlockStore(workdir)
    saved = store.load_plan_config()
    if saved is None or "config" not in saved or "digest" not in saved:
        raise PlanNotFoundError(f"plan configuration under {workdir} is unreadable")
    try:
        saved_config = RsvdConfig.from_json(saved["config"], workdir=workdir)
    except (KeyError, ValueError) as e:
        raise PlanNotFoundError(f"plan configuration under {workdir} is unreadable: {e}")
    if saved_config.digest() != saved["digest"]:
        raise ConfigMismatchError(
            "plan configuration does not match its recorded digest; refusing to resume")
    if config is not None and config.digest() != saved["digest"]:
        raise ConfigMismatchError(
            "supplied configuration differs from the one this plan was started with")
    pool = BlockPool(store, saved_config.budget)
    clock = StageClock()
    with clock.timing(STAGE_PARSE):
        completed = {sid: rec for sid, rec in store.scan_plan().items()
                     if rec.status == "done" and rec.plan_id == saved["digest"]}
    runner = PlanRunner(store, pool, saved["digest"], clock, completed=completed,
                        abort_after=_abort_after())
    if threads is None:
        threads = saved.get("threads", 1)
    command = saved.get("command")
    if command is None:
        a = runner.matrix(saved.get("input_matrix", "A"))
        result = randomized_svd(pool, a, saved_config, threads=threads, runner=runner)
    else:
        if command not in _DRIVERS:
            raise XsvdError(f"command {command!r} is not built on the GPU path")
        result = _DRIVERS[command](runner, pool, saved_config, threads, saved["input"],
                                   saved["output"])
    result.stage_seconds = dict(clock.seconds)
    return result, pool, runner
