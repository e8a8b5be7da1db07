"""Pinned H2D rate vs how full HBM is (B200 diagnostics)."""

import time

import torch


def h2d(host, dev):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    return host.numel() * host.element_size() / (time.perf_counter() - t0) / 1e9


def main():
    gib = 1 << 30
    host = torch.empty(16 * gib, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)
    dev = torch.empty(16 * gib, dtype=torch.uint8, device="cuda")
    print(f"free {torch.cuda.mem_get_info()[0] / gib:.0f} GiB: H2D {h2d(host, dev):.1f} GB/s", flush=True)
    hold = []
    for extra in (64, 32, 32, 16, 8, 4):
        try:
            hold.append(torch.empty(extra * gib, dtype=torch.uint8, device="cuda"))
        except torch.OutOfMemoryError:
            print("oom at", extra, flush=True)
            continue
        print(f"free {torch.cuda.mem_get_info()[0] / gib:.1f} GiB: H2D {h2d(host, dev):.1f} GB/s",
              flush=True)
    # same, with the held memory touched (pages committed)
    for h in hold:
        h.fill_(0)
    print(f"touched; free {torch.cuda.mem_get_info()[0] / gib:.1f} GiB: H2D {h2d(host, dev):.1f} GB/s",
          flush=True)
    # big destination sizes
    del hold
    torch.cuda.empty_cache()
    big = torch.empty(64 * gib, dtype=torch.uint8, pin_memory=True)
    big.fill_(1)
    bdev = torch.empty(64 * gib, dtype=torch.uint8, device="cuda")
    for i in range(3):
        print(f"64 GiB copy #{i}: {h2d(big, bdev):.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
