"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA
source line: share of warp-stall samples and the top stall reasons."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
agg = defaultdict(float)
src = {}
reasons = defaultdict(lambda: defaultdict(float))
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] in ("-", ""):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    s = float(r[4] or 0)
    agg[ln] += s
    src[ln] = r[1]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") or "Stall" in h and i > 6:
            try:
                reasons[ln][h] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
for ln, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top_n]:
    rs = sorted(reasons[ln].items(), key=lambda kv: -kv[1])[:3]
    rtxt = ", ".join(f"{k.split('(')[0].strip()[:28]} {v:.0f}" for k, v in rs if v > 0)
    print(f"{100 * s / tot:5.1f}%  L{ln}: {src[ln].strip()[:90]}  [{rtxt}]")
