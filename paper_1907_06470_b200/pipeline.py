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

Durable plans (plan.py: PlanRunner, run_command, resume; the reference's
pipeline.py:163-253, 719-770, 838-934): with a BlockStore behind the pool,
each step is journalled in the reference's on-disk formats (store.py) and a
resumed plan replays the finished ones. The device factorisation is ONE step
("rsvd-device", outputs U/S/V); a direct call on a store-backed pool first
runs an "ingest" step that makes A durable, as the reference does.
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
from .errors import ShapeError, XsvdError
from .pool import (BlockPool, StoredMatrix, canonical_coo, is_sparse, register_dense,
                   stored_to_array)


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


def _single_tile(a) -> bool:
    d = a.desc
    return not d.transposed and d.partition.n_row_tiles == 1 and d.partition.n_col_tiles == 1


def _tile_grid(a):
    """(row cuts, col cuts, get_tile, release) of A's tile grid as the
    library streams it: tiles come from the caller's pool one at a time
    (pinned while the library holds them, so a budgeted pool cannot evict
    them mid-copy) and are never assembled into one host array. A transposed
    view's tile (ti, tj) is the stored tile (tj, ti), transposed."""
    d = a.desc
    pool, mid = a.pool, d.matrix_id
    part = d.partition
    rows, cols = tuple(part.row_cuts), tuple(part.col_cuts)
    if d.transposed:
        rows, cols = cols, rows
    unpin = getattr(pool, "unpin", None)

    def key(ti, tj):
        return (tj, ti) if d.transposed else (ti, tj)

    def get_tile(ti, tj):
        si, sj = key(ti, tj)
        try:
            block = pool.get(mid, si, sj, pin=True)
        except TypeError:  # a pool without pinning
            block = pool.get(mid, si, sj)
        vals = np.asarray(block.values)
        return np.ascontiguousarray(vals.T) if d.transposed else vals

    def release(ti, tj):
        if unpin is not None:
            unpin(mid, *key(ti, tj))

    return rows, cols, get_tile, release


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
        # a store-backed pool without a runner starts a plan of its own
        # (pipeline.py:466-485): settings saved, then step 0 makes the input
        # durable, so a killed run can resume from the workdir alone
        from .plan import PlanRunner, abort_after_from_env

        runner = PlanRunner(store, pool, config.digest(), clock,
                            abort_after=abort_after_from_env())
        store.save_plan_config({"command": None, "input_matrix": a.matrix_id,
                                "config": config.to_json(), "digest": config.digest()})
        input_id = a.matrix_id

        def ingest():
            pool.flush_matrix(input_id)
            return {}

        runner.step("ingest", stage=STAGE_PARSE, outputs=[input_id], fn=ingest)
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
            rows, cols, vals = canonical_coo(a)
            if a.desc.transposed:
                rows, cols = cols, rows
            omega = None
            if precision is Precision.SINGLE:
                # float32 storage (kernels.py:85-97 with cdt = f32): the values
                # and Omega are float32 numbers (pipeline.py:281-282), carried
                # exactly in the f64 sparse engine; U, V stored as float32
                omega = ctx.gaussian(config.seed, 0, a.shape[1],
                                     config.rank + config.oversample,
                                     dtype=np.float32).astype(np.float64)
            u, s, v, deficient, stages = ctx.rsvd_coo(
                rows, cols, np.asarray(vals, dtype=np.float64), tuple(a.shape), config.rank,
                config.oversample, q, config.seed, omega=omega)
            u = u.astype(precision.storage_dtype, copy=False)
            v = v.astype(precision.storage_dtype, copy=False)
        elif _single_tile(a):
            host = _dense_input(a).astype(precision.storage_dtype, copy=False)
            u, s, v, deficient, stages = ctx.rsvd_dense(host, config.rank, config.oversample, q,
                                                        config.seed)
        else:
            # a tile grid (budgeted / store-backed / partitioned A, or a
            # transposed view): streamed tile by tile, never assembled
            rows, cols, get_tile, release = _tile_grid(a)
            u, s, v, deficient, stages = ctx.rsvd_dense_tiles(
                tuple(a.shape), rows, cols, get_tile, precision.storage_dtype, config.rank,
                config.oversample, q, config.seed, release=release)
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
        rows, cols, vals = canonical_coo(a)
        if a.desc.transposed:
            rows, cols = cols, rows
        omega = None
        if precision is Precision.SINGLE:
            omega = ctx.gaussian(seed, 0, n, rank, dtype=np.float32).astype(np.float64)
        ctx.rsvd_coo(rows, cols, np.asarray(vals, dtype=np.float64), tuple(a.shape), rank, 0,
                     _lib.POWER_AUTO, seed, omega=omega)
    elif _single_tile(a):
        host = _dense_input(a).astype(precision.storage_dtype, copy=False)
        ctx.rsvd_dense(host, rank, 0, _lib.POWER_AUTO, seed)
    else:
        rows, cols, get_tile, release = _tile_grid(a)
        ctx.rsvd_dense_tiles(tuple(a.shape), rows, cols, get_tile, precision.storage_dtype, rank,
                             0, _lib.POWER_AUTO, seed, release=release)
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


# The durable plan machinery (PlanRunner, run_command, resume) lives in
# plan.py; re-exported here under the reference's module layout.
from .plan import ABORT_ENV, ABORT_EXIT_CODE, PlanRunner, resume, run_command  # noqa: E402,F401
