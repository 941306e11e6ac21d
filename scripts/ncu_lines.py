"""Aggregate an ncu source page (cuda,sass) per source line.

usage: ncu -i REP --page source --csv --print-source cuda,sass > x.csv
       python scripts/ncu_lines.py x.csv [top]
Prints, per (file, line): warp instructions, thread instructions, SIMT
efficiency and stall samples, sorted by warp instructions."""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
fname, line, src = "?", None, ""
hdr = None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10:
        continue
    if r[0]:
        line, src = r[0], r[1]
        continue
    if r[2] in ("...", "") or r[7] in ("-", ""):
        continue
    a = agg[(fname, line)]
    a[0] += int(r[7])       # Instructions Executed (warp level)
    a[1] += int(r[8])       # Thread Instructions Executed
    a[2] += int(r[4]) if r[4] not in ("-", "") else 0  # stall samples
    a[3] = src.strip()[:90]
tot_w = sum(v[0] for v in agg.values())
tot_s = sum(v[2] for v in agg.values())
print(f"total warp inst {tot_w}, samples {tot_s}")
for (f, l), (w, t, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f}:{l:>5} {100*w/tot_w:5.1f}% w  simt {t/max(w,1):5.1f}  {100*s/max(tot_s,1):5.1f}% smp  {src}")
