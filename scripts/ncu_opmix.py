"""Opcode mix of an .ncu-rep (SASS source page), weighted by executed warp / thread instructions.
python scripts/ncu_opmix.py REP [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Instructions Executed" in r)
ie, te = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
agg, thr = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) <= te or not r[0].startswith("0x"):
        continue
    ins = r[1].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    try:
        agg[ins.split()[0]] += int(r[ie])
        thr[ins.split()[0]] += int(r[te])
    except ValueError:
        pass
tot, tt = sum(agg.values()), sum(thr.values())
print(f"warp instructions {tot}, thread instructions {tt}, SIMT {tt / max(1, tot):.2f}")
for op, v in agg.most_common(n):
    print(f"{op:22s} {100 * v / tot:6.2f}% warp {100 * thr[op] / tt:6.2f}% thread")
