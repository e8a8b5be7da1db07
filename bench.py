"""Benchmark: rank-k randomized SVD on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2]

A "step" is one full factorisation (Omega, 2q+1 products with
re-orthonormalisation, projection, small SVD, lift) of the workload's A.
Workload at N=1: config 2 (65536 x 16384 float64, k=100, p=20, q=2), the
BASELINE.json config quoted for HBM-resident single-GPU runs.

value  = matrix elements factorised per second (m*n / T_step) with A already
         resident in HBM; T_step from CUDA events on the library's compute
         stream over exactly K steps (barrier + synchronize on both sides,
         max over ranks). A (8.6 GB) is far larger than L2 (126 MB), so no
         L2 flush is needed between steps.
e2e    = the same metric through the reference-facing C ABI call
         (xb_rsvd_dense) with HOST buffers: pinned A copied H2D inside the
         timed region (overlapped with the sketch), U/s/V copied back.
roofline = the dominant kernel (the FP64 DMMA tile GEMM over A: 6 launches
         per step), achieved = 2*m*n*l flops per launch / its event-timed
         average duration, peak = the FP64 DMMA pipe peak measured in-process
         by a saturating microbenchmark (MEASURED_PEAKS.json has no FP64).
cpu_baseline = the oracle's restatement of the reference's shipped driver
         (oracle/, "port") on a bounded row sample, on this host's cores.

--impl reference prints the reference arm: the same port timed on all host
threads (the reference is pure Python and cannot travel to the GPU box).
Multi-GPU (torchrun, N>1): A's rows are sharded over ranks; see DESIGN.md.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# -- clocks during the timed region ----------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# -- workloads ---------------------------------------------------------------------

def make_device_matrix(w, rows_lo, rows_hi, device):
    """This rank's rows of the config's A, built on the GPU from the seeds."""
    import torch

    from paper_1907_06470_b200.workloads import dense_lowrank_torch

    # the full-matrix construction is seeded once; every rank builds the same
    # A and keeps its row block (construction cost is outside the timed region)
    a = dense_lowrank_torch(w.m, w.n, w.spectrum, w.noise, w.cfg, w.signal_rank,
                            dtype=torch.float64, device=device)
    if rows_lo == 0 and rows_hi == w.m:
        return a
    part = a[rows_lo:rows_hi].clone()
    del a
    torch.cuda.empty_cache()
    return part


def _time_port(w, rows: int, threads: int) -> float:
    from oracle import pipeline as OP

    # the reference's run time does not depend on A's spectrum,
    # so the CPU sample uses a seeded Gaussian A of the config's width
    a = np.random.default_rng(3000 + w.cfg).standard_normal((rows, w.n))
    t0 = time.perf_counter()
    OP.randomized_svd(a, w.k, w.p, w.q, w.cfg, "double", threads=threads)
    return time.perf_counter() - t0


def cpu_baseline(w, budget_s: float, threads: int) -> dict:
    """Oracle port of the reference's shipped driver on two row samples of A,
    extrapolated linearly in m to the full config (T = a + b*m, SURVEY §8d:
    the products and panel QR are linear in m; Omega and svd_small are not)."""
    r1 = min(w.m, 1024)
    t1 = _time_port(w, r1, threads)
    # second sample sized to use the rest of the budget
    per_row = max(t1 / r1, 1e-9)
    r2 = int(min(w.m, max(2 * r1, (budget_s - t1) / per_row * 0.6)))
    r2 = max(r1 + 256, (r2 // 256) * 256)
    r2 = min(r2, w.m)
    t2 = _time_port(w, r2, threads) if r2 > r1 else t1
    b = (t2 - t1) / (r2 - r1) if r2 > r1 else t1 / r1
    a0 = max(t1 - b * r1, 0.0)
    t_full = a0 + b * w.m
    return {"value": w.m * w.n / t_full, "unit": "elements/s", "cores": threads, "kind": "port",
            "sample": (f"oracle restatement of xsvd.randomized_svd (shipped driver: 256-cell "
                       f"block_multiply on {threads} threads, Householder thin_qr, Golub-Kahan "
                       f"svd_small) on seeded Gaussian {r1}x{w.n} ({t1:.2f} s) and {r2}x{w.n} "
                       f"({t2:.2f} s) samples, k={w.k} p={w.p} q={w.q}; extrapolated linearly in "
                       f"m to {w.m} rows: {t_full:.1f} s"),
            "seconds": t_full, "rows": r2, "sample_seconds": t2}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1907_06470_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    threads = os.cpu_count() or 1
    # calibration (counts as warm-up): fixes the sample size and the
    # m-independent part a0 of the linear time model
    base = cpu_baseline(w, args.cpu_budget_s, threads)
    rows = base["rows"]
    slope = (base["seconds"] - base["sample_seconds"]) / max(w.m - rows, 1)
    a0 = max(base["sample_seconds"] - slope * rows, 0.0)
    for _ in range(max(args.warmup - 1, 0)):
        _time_port(w, rows, threads)
    full = []
    for _ in range(args.steps):
        t = _time_port(w, rows, threads)
        full.append(a0 + (t - a0) * (w.m / rows))
    dt = float(np.mean(full))
    value = w.m * w.n / dt
    line = {
        "impl": "reference", "metric": "rank-k rSVD matrix-elements/s", "value": value,
        "unit": "elements/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg construction)",
        "config": {"workload": w.name, "sample_rows": rows,
                   "step": f"one {rows}x{w.n} sample run, extrapolated linearly in m"},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": threads, "kind": "port",
                         "sample": base["sample"]},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import CONFIGS

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    w = CONFIGS[args.config]
    if w.density != "dense" or w.precision != "double":
        raise SystemExit(f"config {args.config} ({w.density}/{w.precision}) not built yet")
    if world > 1:
        raise SystemExit("multi-GPU row sharding lands with the NCCL reducer (DESIGN.md)")
    ctx = _lib.load(local)
    m, n, k, p, q = w.m, w.n, w.k, w.p, w.q
    l = k + p
    a = make_device_matrix(w, 0, m, device)
    u = torch.empty((m, k), dtype=torch.float64, device=device)
    v = torch.empty((n, k), dtype=torch.float64, device=device)
    s = torch.empty((k,), dtype=torch.float64, device=device)
    torch.cuda.synchronize()

    def step():
        return ctx.rsvd_dense_dev(np.float64, m, n, a.data_ptr(), n, k, p, q, w.cfg,
                                  u.data_ptr(), s.data_ptr(), v.data_ptr())

    for _ in range(args.warmup):
        step()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.profile(True)
    ctx.profile_read()
    launches0 = ctx.launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        stage_tot = np.zeros(8)
        for _ in range(args.steps):
            _, stages = step()
            stage_tot += stages
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    prof = ctx.profile_read()
    ctx.profile(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = m * n / (ms * 1e-3)

    # roofline of the dominant kernel (FP64 DMMA tile GEMM on A)
    dmma_peak, dfma_peak = ctx.fp64_peaks()
    per_launch_s = prof["seconds"] / max(prof["launches"], 1)
    per_launch_flops = prof["flops"] / max(prof["launches"], 1)
    achieved = per_launch_flops / per_launch_s / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"cfg{w.cfg}")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": achieved / dmma_peak if dmma_peak else None, "traffic": traffic,
                "kernel": "dgemm_kernel (FP64 DMMA m8n8k4, NN/TN over A)",
                "launches_per_step": prof["launches"] / args.steps,
                "share_of_step": prof["seconds"] / (ms * 1e-3 * args.steps),
                "peak_source": f"in-process DMMA microbenchmark ({dmma_peak:.1f} TF/s; DFMA "
                               f"{dfma_peak:.1f} TF/s); MEASURED_PEAKS.json has no FP64 entry",
                "hbm_gbs_achieved": prof["bytes"] / prof["seconds"] / 1e9 if prof["seconds"] else None}

    # e2e through the host-buffer C ABI call (pinned A, copies inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        a_host = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
        a_host.copy_(a)
        del a
        torch.cuda.empty_cache()
        a_np = a_host.numpy()
        ctx.rsvd_dense(a_np, k, p, q, w.cfg)  # warm (allocates the host-path buffers)
        e2e_t, ingest = [], []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            U, S, V, _, st = ctx.rsvd_dense(a_np, k, p, q, w.cfg)
            e2e_t.append(time.perf_counter() - t0)
            ingest.append(st[0])
        e2e_s = float(np.median(e2e_t))
        e2e = {"value": m * n / e2e_s, "unit": "elements/s", "h2d_bytes_per_step": m * n * 8,
               "d2h_bytes_per_step": (m * k + n * k + k) * 8, "seconds": e2e_s,
               "h2d_gbs": m * n * 8 / float(np.median(ingest)) / 1e9 if min(ingest) > 0 else None,
               "timer": "host perf_counter around the synchronous C ABI call"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_budget_s, os.cpu_count() or 1)
        for key in ("seconds", "rows", "sample_seconds"):
            cpu.pop(key, None)

    stage_names = ["Text Parsing", "Preparation of O", "O*A^T", "Orthogonalization", "A^T*Q_r",
                   "SVD0 Preparation", "SVD0", "Postprocessing"]
    line = {
        "metric": "rank-k rSVD matrix-elements/s", "value": value, "unit": "elements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: A = U diag(i^-1.5) V^T + 1e-8 N(0,1), U/V Haar from seed 1002/2002 "
                "(built on the GPU with torch, outside the timed region)",
        "config": {"workload": w.name, "m": m, "n": n, "k": k, "p": p, "q": q, "l": l,
                   "omega": "gaussian_band(seed=2) generated on device each step",
                   "l2": "inputs larger than L2 (A = 8.6 GB), no flush",
                   "parallelism": f"rows{world}"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
        "clocks": clocks.summary(),
        "stage_ms": {nm: 1e3 * t / args.steps for nm, t in zip(stage_names, stage_tot)},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
