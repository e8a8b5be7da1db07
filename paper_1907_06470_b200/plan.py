"""Durable plans around the device factorisation: a step journal in a
workdir, so an interrupted command resumes where it stopped.

Same contract as the reference's plan machinery (src/pipeline.py:163-253
PlanRunner, 719-770 command drivers, 838-934 run_command / resume): every
step writes a "pending" record, runs, makes its outputs durable in the pool's
BlockStore, then writes the record again as "done" with the metadata a
replay needs; a resumed process re-issues the same step sequence and every
step whose record is done (same op, same plan digest, outputs intact) is
answered from its record instead of running. The on-disk formats are the
reference's (store.py); the step sequence is this package's own — the whole
device factorisation is ONE step ("rsvd-device"), since it takes
milliseconds to seconds and finer records would only add fsyncs — so a
workdir the reference started is rerun from its first step here.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigMismatchError, PlanNotFoundError, XsvdError
from .pool import BlockPool, StoredMatrix
from .store import BlockStore, StepRecord, write_block_file

ABORT_ENV = "XSVD_ABORT_AFTER_STEPS"
ABORT_EXIT_CODE = 70


def abort_after_from_env():
    """Test hook (the reference's XSVD_ABORT_AFTER_STEPS): hard-exit after N
    steps, i.e. a kill between two durable steps."""
    raw = os.environ.get(ABORT_ENV)
    return int(raw) if raw else None


@dataclass
class PlanRunner:
    """Sequential step journal. `step` returns the step's metadata: from its
    record when a prior run finished it, else from running `fn`."""

    store: BlockStore | None
    pool: BlockPool
    plan_id: str
    clock: object
    completed: dict = field(default_factory=dict)
    abort_after: int | None = None
    next_id: int = 0
    ran: int = 0

    def __post_init__(self):
        self.completed = dict(self.completed or {})

    def _replayed(self, step_id: int, op: str):
        rec = self.completed.get(step_id)
        usable = (rec is not None and rec.status == "done" and rec.op == op
                  and rec.plan_id == self.plan_id)
        return dict(rec.meta) if usable else None

    def _journal(self, record: StepRecord, stage: str):
        if self.store is not None:
            with self.clock.timing(stage):
                self.store.write_step(record)

    def step(self, op, *, stage, fn, inputs=(), outputs=(), seed=None, self_clocked=False):
        step_id, self.next_id = self.next_id, self.next_id + 1
        meta = self._replayed(step_id, op)
        if meta is not None:
            return meta
        record = StepRecord(self.plan_id, step_id, op, list(inputs), list(outputs), rng_seed=seed)
        self._journal(record, stage)
        if self_clocked:  # fn books its own (device) stage times
            meta = fn() or {}
        else:
            with self.clock.timing(stage):
                meta = fn() or {}
        if self.store is not None:
            with self.clock.timing(stage):
                for matrix_id in outputs:
                    self.pool.flush_matrix(matrix_id)
        record.status, record.meta = "done", meta
        self._journal(record, stage)
        self.ran += 1
        if self.abort_after is not None and self.ran >= self.abort_after:
            os._exit(ABORT_EXIT_CODE)
        return meta

    def matrix(self, matrix_id):
        """A step output, whether produced now or by the run being resumed."""
        if matrix_id not in self.pool.known_matrices() and self.store is not None:
            self.pool.register(self.store.load_descriptor(matrix_id))
        return StoredMatrix(self.pool.descriptor(matrix_id), self.pool)


# -- command drivers ---------------------------------------------------------------


def _write_s_txt(path: str, values: np.ndarray):
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.writelines(f"{v:.17g}\n" for v in values)
    os.replace(tmp, path)


def _export(runner, outdir):
    """One step per factor: U.blk, S.blk (+ S.txt, %.17g per line), V.blk."""
    from .pipeline import STAGE_POST

    os.makedirs(outdir, exist_ok=True)

    def exporter(matrix_id):
        def run():
            mat = runner.matrix(matrix_id)
            write_block_file(os.path.join(outdir, f"{matrix_id}.blk"), mat)
            if matrix_id == "S":
                _write_s_txt(os.path.join(outdir, "S.txt"),
                             mat.to_array().astype(np.float64).ravel())
            return {}
        return run

    for matrix_id in ("U", "S", "V"):
        runner.step(f"export-{matrix_id.lower()}", stage=STAGE_POST, inputs=[matrix_id],
                    fn=exporter(matrix_id))


def _factorise_file(method):
    def drive(runner, pool, config, threads, input_path, outdir):
        from .formats import parse_matrix_market
        from .pipeline import STAGE_PARSE

        def parse():
            parse_matrix_market(input_path, pool, "A", precision=config.precision)
            return {}

        runner.step("parse", stage=STAGE_PARSE, outputs=["A"], fn=parse)
        result = method(pool, runner.matrix("A"), config, threads=threads, runner=runner)
        _export(runner, outdir)
        return result
    return drive


def _drivers():
    from .pipeline import full_svd, randomized_svd

    return {"rsvd": _factorise_file(randomized_svd), "svd": _factorise_file(full_svd)}


def run_command(command, input_path, output_path, config, *, threads: int = 1,
                fresh: bool = True, profile_out=None):
    """Factorise a Matrix Market file with a durable plan in config.workdir
    and export U/S/V to `output_path`; `fresh` wipes an earlier plan."""
    from .pipeline import STAGE_PARSE, StageClock

    if config.workdir is None:
        raise ValueError("run_command needs config.workdir for its plan state")
    drivers = _drivers()
    if command not in drivers:
        raise XsvdError(f"command {command!r} is not built on the GPU path "
                        f"(have: {', '.join(sorted(drivers))})")
    clock = StageClock()
    with clock.timing(STAGE_PARSE):
        store = BlockStore(config.workdir)
        if fresh:
            store.clear_plan()
        settings = dict(command=command, input=os.path.abspath(input_path),
                        output=os.path.abspath(output_path), threads=threads,
                        profile_out=os.path.abspath(profile_out) if profile_out else None,
                        config=config.to_json(), digest=config.digest())
        store.save_plan_config(settings)
        pool = BlockPool(store, config.budget)
    runner = PlanRunner(store, pool, config.digest(), clock, abort_after=abort_after_from_env())
    result = drivers[command](runner, pool, config, threads, input_path, output_path)
    result.stage_seconds = dict(clock.seconds)
    return result, pool, runner


def _saved_settings(store: BlockStore, workdir: str, requested):
    """The plan's saved settings and config, checked against their digest
    and against the caller's config (if any)."""
    from .pipeline import RsvdConfig

    saved = store.load_plan_config()
    if not saved or "config" not in saved or "digest" not in saved:
        raise PlanNotFoundError(f"plan configuration under {workdir} is unreadable")
    try:
        cfg = RsvdConfig.from_json(saved["config"], workdir=workdir)
    except (KeyError, ValueError) as e:
        raise PlanNotFoundError(f"plan configuration under {workdir} is unreadable: {e}")
    if cfg.digest() != saved["digest"]:
        raise ConfigMismatchError(
            "plan configuration does not match its recorded digest; refusing to resume")
    if requested is not None and requested.digest() != saved["digest"]:
        raise ConfigMismatchError(
            "supplied configuration differs from the one this plan was started with")
    return saved, cfg


def resume(workdir: str, config=None, *, threads: int | None = None):
    """Finish an interrupted plan, refusing changed settings. Returns
    (result, pool, runner)."""
    from .pipeline import STAGE_PARSE, StageClock, randomized_svd

    if not os.path.exists(os.path.join(workdir, "plan", "config.json")):
        raise PlanNotFoundError(f"no execution plan under {workdir}")
    store = BlockStore(workdir)
    saved, cfg = _saved_settings(store, workdir, config)
    clock = StageClock()
    with clock.timing(STAGE_PARSE):
        done = {sid: rec for sid, rec in store.scan_plan().items()
                if rec.status == "done" and rec.plan_id == saved["digest"]}
    pool = BlockPool(store, cfg.budget)
    runner = PlanRunner(store, pool, saved["digest"], clock, completed=done,
                        abort_after=abort_after_from_env())
    threads = saved.get("threads", 1) if threads is None else threads
    command = saved.get("command")
    if command is None:
        # a direct randomized_svd(pool-with-store, ...) call: its step 0
        # made the input durable ("ingest"); continue after it
        runner.next_id = 1
        result = randomized_svd(pool, runner.matrix(saved.get("input_matrix", "A")), cfg,
                                threads=threads, runner=runner)
    else:
        drivers = _drivers()
        if command not in drivers:
            raise XsvdError(f"command {command!r} is not built on the GPU path")
        result = drivers[command](runner, pool, cfg, threads, saved["input"], saved["output"])
    result.stage_seconds = dict(clock.seconds)
    return result, pool, runner
