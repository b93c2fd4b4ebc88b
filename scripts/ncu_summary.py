"""Summarise one ncu --set full capture of k_grid into profiles/ (JSON).

usage: python scripts/ncu_summary.py <rep.ncu-rep> <cell_steps_per_launch> <out.json> [workload]

Reads the raw page (duration, DRAM bytes, issue/pipe utilisation, stall samples)
and the SASS source page (executed instructions per opcode: the FP64-pipe
instruction count per cell-step that bench.py reports next to the roofline).
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

rep, cells, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
workload = sys.argv[4] if len(sys.argv) > 4 else ""


def page(*args):
    r = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True,
                       check=True)
    return list(csv.reader(io.StringIO(r.stdout)))


raw = page("--page", "raw")
hdr, vals = raw[0], raw[2]
m = dict(zip(hdr, vals))


units = dict(zip(hdr, raw[1]))
_TIME = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def num(key):
    try:
        return float(m[key].replace(",", ""))
    except (KeyError, ValueError):
        return None


def usecs(key):
    v = num(key)
    return None if v is None else v * _TIME.get(units.get(key, "usecond"), 1.0)


src = page("--page", "source", "--print-source", "sass")
shdr = src[1]
iS, iE = shdr.index("Source"), shdr.index("Instructions Executed")
ops = Counter()
for r in src[2:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    t = r[iS].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ops[op] += n
fp64_ops = ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX", "DSET")
fp64 = sum(ops[o] for o in fp64_ops)
total = sum(ops.values())
stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(k) for k in hdr
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
ssum = sum(v for v in stalls.values() if v) or 1.0
top = sorted(((k, v / ssum) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:8]
dram = (num("dram__bytes_read.sum") or 0) + (num("dram__bytes_write.sum") or 0)
unit = m.get("dram__bytes_read.sum", "")
summary = {
    "kernel": src[0][1] if len(src[0]) > 1 else "",
    "workload": workload,
    "source": rep.split("/")[-1] + " (ncu --set full --clock-control none --import-source on)",
    "duration_us": usecs("gpu__time_duration.sum"),
    "dram_bytes_per_launch": None,
    "warp_instructions": total,
    "fp64_warp_instructions": fp64,
    "fp64_instr_per_cell_step": 32.0 * fp64 / cells,
    "instr_per_cell_step": 32.0 * total / cells,
    "opcode_mix_per_cell_step": {k: round(32.0 * v / cells, 2) for k, v in ops.most_common(16)},
    "fp64_pipe_pct_of_peak": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_per_scheduler": num("smsp__warps_active.avg.per_cycle_active"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "grid_size": num("launch__grid_size"),
    "block_size": num("launch__block_size"),
    "stall_share_top": {k: round(v, 3) for k, v in top},
    "cell_steps_per_launch": cells,
}
# raw-page DRAM byte counters come in the unit ncu picked (usually MB for this size)
rb = num("dram__bytes_read.sum")
wb = num("dram__bytes_write.sum") or 0.0
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(raw[1][hdr.index(
    "dram__bytes_read.sum")] if "dram__bytes_read.sum" in hdr else "byte", 1)
if rb is not None:
    summary["dram_bytes_per_launch"] = int(round((rb + wb) * scale))
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps(summary, indent=1))
