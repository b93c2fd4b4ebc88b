"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into JSON.

usage: python scripts/launch_summary.py launches.csv "<command>" out.json
"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
iU = hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    k = r[iK]
    tot[k][0] += 1
    tot[k][1] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
step = {k: v for k, v in tot.items() if k.startswith("void rg::k_grid") or "k_gen_soa" in k}
s = sum(v[1] for v in step.values()) or 1.0
out = {
    "command": sys.argv[2],
    "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised "
            "per launch); torch L2-flush fills and k_dfma_peak run outside the timed step",
    "all_kernels": {k: {"launches": v[0], "total_us": round(v[1], 3),
                        "mean_us": round(v[1] / v[0], 3)} for k, v in tot.items()},
    "share_within_step": {k: v[1] / s for k, v in step.items()},
}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
