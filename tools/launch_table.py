"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_table.py gpurun_out/launches5.csv [--steps 2]
"""

import collections
import csv
import sys


def main():
    path = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 1
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:70]
        tot[name] += v
        cnt[name] += 1
    # the bench's in-process peak probes run outside the timed region: listed,
    # but not part of the step or of the shares
    probe = {k for k in tot if "_peak_kernel" in k}
    total = sum(v for k, v in tot.items() if k not in probe)
    print(f"| kernel | launches/step | ms/step | share of step |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        if k in probe:
            continue
        print(f"| `{k}` | {cnt[k] / steps:g} | {v / steps:.2f} | {100 * v / total:.1f}% |")
    n_step = sum(c for k, c in cnt.items() if k not in probe)
    print(f"| total (step) | {n_step / steps:g} | {total / steps:.1f} | |")
    for k in sorted(probe):
        print(f"| `{k}` (peak probe, outside the timed region) | {cnt[k] / steps:g} | "
              f"{tot[k] / steps:.2f} | - |")


if __name__ == "__main__":
    import signal

    signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet under | head
    main()
