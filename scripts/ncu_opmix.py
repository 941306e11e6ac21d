"""Opcode mix of an ncu source page (sass rows) weighted by executed warp instructions."""
import collections
import csv
import sys

agg = collections.Counter()
thr = collections.Counter()
for r in csv.reader(open(sys.argv[1])):
    if len(r) < 10 or r[0] not in ("",) or r[2] in ("...", "") or not r[2].startswith("0x"):
        continue
    if r[7] in ("-", ""):
        continue
    ins = r[3].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0]
    agg[op] += int(r[7])
    thr[op] += int(r[8])
tot = sum(agg.values())
print("total", tot)
for op, n in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{op:24s} {100*n/tot:5.1f}%  simt {thr[op]/n:5.1f}")
