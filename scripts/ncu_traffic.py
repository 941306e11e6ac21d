"""Regenerate profiles/ncu_traffic.json from the ncu summaries of a round:
DRAM bytes per launch (roofline.traffic), issue-active share, SIMT lanes per
instruction, warp instructions and the FP32 share of thread instructions.
python scripts/ncu_traffic.py TAG   (reads profiles/TAG/ncu_*.txt and gpurun_out/TAG/*.ncu-rep)"""
import csv
import io
import json
import os
import re
import subprocess
import sys

tag = sys.argv[1]
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3, "ns": 1e-3, "%": 1, "inst": 1, "": 1}


def parse(fn):
    out, cur = [], None
    for line in open(fn):
        if "Kernel Name" in line:
            cur = {"name": line.split("=")[1].strip().split("(")[0].replace("void ", "").strip()}
            out.append(cur)
            continue
        m = re.match(r"\s+(\S+) = ([0-9.eE+-]+)\s*(\S*)", line)
        if m and cur is not None:
            cur[m.group(1)] = float(m.group(2)) * MULT.get(m.group(3), 1)
    return out


def fp32_share(rep):
    """FP32 thread instructions / all thread instructions (SASS opcode mix)."""
    if not os.path.exists(rep):
        return None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(txt)) if r]
    while rows and "Source" not in rows[0]:  # skip the "Kernel Name" line
        rows = rows[1:]
    if not rows:
        return None
    hdr = rows[0]
    try:
        isrc = hdr.index("Source")
        ith = hdr.index("Thread Instructions Executed")
    except ValueError:
        return None
    fp = tot = 0.0
    for r in rows[1:]:
        if len(r) <= max(isrc, ith):
            continue
        try:
            n = float(r[ith])
        except ValueError:
            continue
        op = r[isrc].strip().split()
        op = [t for t in op if not t.startswith("@")]
        name = op[0] if op else ""
        tot += n
        if name.split(".")[0] in ("FFMA", "FADD", "FMUL", "FSETP", "FMNMX", "FSEL", "FRND", "MUFU", "FCHK"):
            fp += n
    return fp / tot if tot else None


tr = {}
for scene, fn in [("forest_di6", "ncu_prop_forest_di6"), ("building_quad12", "ncu_prop_building_quad12"),
                  ("narrow_dubins6", "ncu_prop_narrow_dubins6"), ("forest_di6_select", "ncu_sel_forest_di6"),
                  ("building_quad12_sweep_2^22", "ncu_prop_sweep_building_quad12")]:
    path = f"profiles/{tag}/{fn}.txt"
    if not os.path.exists(path):
        continue
    tr[scene] = {}
    for k in parse(path):
        e = {"dram_bytes": round(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)),
             "duration_us": k.get("gpu__time_duration.sum"),
             "issue_active_pct": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "simt": k.get("smsp__thread_inst_executed_per_inst_executed.ratio"),
             "warp_inst": k.get("smsp__inst_executed.sum"),
             "source": f"{tag}/{fn}.txt"}
        if "propagate" in k["name"]:
            e["fp32_share"] = fp32_share(f"gpurun_out/{tag}/{fn.replace('ncu_', '')}.ncu-rep")
        tr[scene][k["name"]] = e
json.dump(tr, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(tr, indent=1))
