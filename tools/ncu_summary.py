"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py OUT.md gpurun_out/prof_nn.ncu-rep [...] \
        [--launches gpurun_out/launches.csv] [--traffic-json profiles/ncu_traffic.json --cfg 2]
"""

import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "lts__t_bytes.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"Kernel Name": row[hdr.index("Kernel Name")]}
        stalls = {}
        for i, h in enumerate(hdr):
            if h in KEYS:
                d[h] = f"{row[i]} {units[i]}".strip()
            if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.2:
                    stalls[h.split("stalled_")[1].split("_per_issue")[0]] = round(v, 2)
        d["stalls (per issue)"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        name = d["Kernel Name"]
        name = name.split("(")[0] if "<" not in name else name.split(">(")[0] + ">"
        tot[name] += float(d["Metric Value"])
        cnt[name] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--launches")
    ap.add_argument("--traffic-json")
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--title", default="ncu summary")
    args = ap.parse_args()
    lines = [f"# {args.title}", ""]
    traffic = []
    for rep in args.reps:
        for d in raw(rep):
            lines.append(f"## {d['Kernel Name']}")
            lines.append(f"source: `{rep}`")
            lines.append("")
            for k, v in d.items():
                if k != "Kernel Name":
                    lines.append(f"- `{k}`: {v}")
            lines.append("")
            try:
                rb = d["dram__bytes_read.sum"].split()
                wb = d["dram__bytes_write.sum"].split()
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                traffic.append(float(rb[0]) * scale[rb[1]] + float(wb[0]) * scale[wb[1]])
            except (KeyError, IndexError, ValueError):
                pass
    if args.launches:
        tot, cnt = launches(args.launches)
        total = sum(tot.values())
        lines.append("## Launch list (ncu gpu__time_duration, cold-cache & serialised: compare shares)")
        lines.append("")
        lines.append("| kernel | total ms | share | launches |")
        lines.append("|---|---|---|---|")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            lines.append(f"| `{k[:110]}` | {v / 1e6:.3f} | {100 * v / total:.1f}% | {cnt[k]} |")
        lines.append("")
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if args.traffic_json and traffic:
        try:
            data = json.load(open(args.traffic_json))
        except (OSError, ValueError):
            data = {}
        data[f"cfg{args.cfg}"] = sum(traffic) / len(traffic)
        json.dump(data, open(args.traffic_json, "w"), indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
