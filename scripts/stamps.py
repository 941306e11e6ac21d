"""Phase timeline of steady-state iterations from a -DKP_STAMPS build
(make -B paper_2602_02846_b200/lib/libkinoplan_b200.so NVFLAGS="... -DKP_STAMPS").
python scripts/stamps.py SCENE [BUDGET_S | iN] [rows]   -> median µs of each phase over the last 64
iterations (iN: stop after N iterations, e.g. i20 for the growth phase; rows: one line per iteration)"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2602_02846_b200 import Planner, scenarios  # noqa: E402

scene = sys.argv[1] if len(sys.argv) > 1 else "forest_di6"
arg = sys.argv[2] if len(sys.argv) > 2 else "0.1"
with Planner(scenarios.load(scene), seed=1000) as g:
    g.reset(1000)
    if arg.startswith("i"):
        g.solve(0.0, int(arg[1:]))
    else:
        g.solve(float(arg))
    buf = (C.c_uint64 * (64 * 32))()
    rc = g._lib.kp_debug_stamps(g._h, buf)
    if rc != 0:
        sys.exit(f"kp_debug_stamps rc={rc} (build with -DKP_STAMPS)")
    s = np.array(buf, dtype=np.float64).reshape(64, 32) / 1e3  # us
it = np.argsort(s[:, 0])  # iteration order by propagate entry
s = s[it]
s = s[s[:, 0] > 0]
names = {0: "P entry", 1: "P pdl", 14: "P ctl", 2: "P last exit", 3: "S max first scan done", 4: "S max writes issued",
         5: "R ctl", 6: "R last exit", 7: "S entry", 8: "S pdl", 9: "S ctl", 13: "S (unused)",
         10: "S boundary start (block 0)", 11: "S (unused)", 12: "S boundary end (block 0)", 15: "S max prefix pass done",
         16: "P max sampled", 17: "P max checks done", 18: "P max admitted", 19: "R max prune done",
         20: "R max live pruned", 21: "R max slot tested"}
base = s[:, 1]  # propagate PDL release
rows = []
for k in (0, 1, 14, 16, 17, 18, 2, 5, 20, 21, 19, 6, 7, 8, 9, 15, 3, 4, 10, 12):
    rows.append((names[k], np.median(s[:, k] - base)))
nxt = np.median(s[1:, 1] - s[:-1, 1])
print(f"{scene}: median over {len(s)} iterations, µs relative to propagate's PDL release; iteration period {nxt:.2f} µs")
for n, v in rows:
    print(f"  {n:22s} {v:8.2f}")
if len(sys.argv) > 3 and sys.argv[3] == "rows":
    print("per iteration (µs from propagate's PDL release): P ctl, P sampled, P checks, P exit | R ctl, R prune, R exit | "
          "S ctl, S prefix, S scan, S writes, boundary start, boundary end | period")
    for j in range(len(s)):
        b = s[j, 1]
        per = s[j + 1, 1] - b if j + 1 < len(s) else float("nan")
        print(" ".join(f"{s[j, k] - b:6.1f}" for k in (14, 16, 17, 2, 5, 19, 6, 9, 15, 3, 4, 10, 12)), f"| {per:6.1f}")
