"""Per-launch rows of an ncu --csv launch list with several metrics:
    python tools/launch_detail.py gpurun_out/launches.csv [min_ms]"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    lim = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                           "Metric Unit"))
    cur = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = cur.setdefault(r[h.index("ID")], {"name": r[ki].split("(")[0][-34:]})
        d[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    for d in cur.values():
        t = d.get("gpu__time_duration.sum", (0, ""))
        ms = t[0] * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
                     "ms": 1, "msecond": 1}.get(t[1], 1)
        if ms < lim:
            continue
        extra = " ".join(f"{k.split('__')[1][:18]}={v[0]:.3g}{v[1]}" for k, v in d.items()
                         if k not in ("name", "gpu__time_duration.sum"))
        print(f"{d['name']:36s} {ms:8.3f} ms  {extra}")


if __name__ == "__main__":
    main()
