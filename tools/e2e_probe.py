"""Where does the host-buffer (e2e) time of a config go? Pinned H2D alone vs
xb_rsvd_dense with XB_TRACE=1.   python tools/e2e_probe.py --config 5"""

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    args = ap.parse_args()
    os.environ["XB_TRACE"] = "1"
    import torch

    from paper_1907_06470_b200 import _lib
    from paper_1907_06470_b200.workloads import CONFIGS

    w = CONFIGS[args.config]
    dt = torch.float64 if w.precision == "double" else torch.float32
    ctx = _lib.load(0)
    t0 = time.perf_counter()
    host = torch.empty((w.m, w.n), dtype=dt, pin_memory=True)
    host.normal_()
    print(f"pinned alloc+fill {time.perf_counter() - t0:.2f} s", flush=True)
    dev = torch.empty((w.m, w.n), dtype=dt, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(host, non_blocking=True)
        torch.cuda.synchronize()
        dtt = time.perf_counter() - t0
        print(f"H2D {host.numel() * host.element_size() / dtt / 1e9:.1f} GB/s ({dtt:.2f} s)",
              flush=True)
    del dev
    torch.cuda.empty_cache()
    a = host.numpy()
    scratch = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    hs = host.view(torch.uint8).view(-1)[: 1 << 30]
    for _ in range(3):
        t0 = time.perf_counter()
        _, _, _, _, st = ctx.rsvd_dense(a, w.k, w.p, w.q, w.cfg)
        print(f"rsvd_dense {time.perf_counter() - t0:.2f} s stages {np.round(st, 3).tolist()}",
              flush=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        scratch.copy_(hs, non_blocking=True)
        torch.cuda.synchronize()
        print(f"  torch 1 GiB H2D between calls: {(1 << 30) / (time.perf_counter() - t0) / 1e9:.1f} GB/s",
              flush=True)
    dev = torch.empty((w.m, w.n), dtype=dt, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    dtt = time.perf_counter() - t0
    print(f"H2D after: {host.numel() * host.element_size() / dtt / 1e9:.1f} GB/s", flush=True)
    del scratch
    # H2D concurrent with a long HBM-heavy kernel stream
    side = torch.cuda.Stream()
    x = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        for _ in range(200):
            y.copy_(x)
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    dtt = time.perf_counter() - t0
    torch.cuda.synchronize()
    print(f"H2D under HBM copy load: {host.numel() * host.element_size() / dtt / 1e9:.1f} GB/s",
          flush=True)


if __name__ == "__main__":
    main()
