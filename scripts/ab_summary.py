"""Mean of the ab_perf rounds per scene and build: python scripts/ab_summary.py gpurun_out/TAG/ab.log"""
import collections
import re
import sys

d = collections.defaultdict(lambda: collections.defaultdict(list))
cur = None
for ln in open(sys.argv[1]):
    m = re.match(r"== (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"(\S+)\s+\S+\s+sweep\s+([\d.]+).*query\s+([\d.]+).*ttfs\s+([\d.]+)", ln)
    if m and cur:
        d[m.group(1)][cur].append((float(m.group(2)), float(m.group(3)), float(m.group(4))))
for sc, v in d.items():
    print(sc)
    for k, r in sorted(v.items()):
        n = len(r)
        print(f"   {k:14s} sweep {sum(x[0] for x in r) / n:6.2f}  query {sum(x[1] for x in r) / n:5.2f}  ttfs {sum(x[2] for x in r) / n:.3f}")
