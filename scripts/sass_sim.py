"""Single-warp in-order issue model of a kernel's hot path, from an ncu source
page (--page source --csv --print-source sass): instructions executed at least
THRESH x the top count, in address order, with fixed latencies per opcode.
Prints the modelled cycles per pass for 1 and 2 co-resident warps and the
dependency distance histogram of FP64 instructions.

usage: python scripts/sass_sim.py source.csv [thresh]
"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
ins = []
for r in rows[2:]:
    try:
        n = int(r[iE])
    except (ValueError, IndexError):
        continue
    ins.append((n, r[iS].strip()))
top = max(n for n, _ in ins)
th = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
hot = [s for n, s in ins if n >= th * top]

FP64 = ("DFMA", "DADD", "DMUL", "DSETP")
LAT = {"DFMA": 8, "DADD": 8, "DMUL": 8, "DSETP": 8, "MUFU": 18, "F2I": 14, "I2F": 14,
       "LDS": 30, "LDG": 400, "LDGSTS": 30, "FSEL": 4, "SEL": 4, "IMAD": 4, "ISETP": 4,
       "LOP3": 4, "IADD3": 4, "SHF": 4, "MOV": 4, "VIADD": 4, "BRA": 1, "BSSY": 1,
       "BSYNC": 1}


def regs(tok):
    out = []
    for m in re.finditer(r"\bR(\d+)\b", tok):
        out.append(int(m.group(1)))
    return out


parsed = []
for s in hot:
    s2 = re.sub(r"^@!?P\w+\s+", "", s)
    op = s2.split()[0]
    base = op.split(".")[0]
    args = s2[len(op):].strip().rstrip(";")
    parts = [a.strip() for a in args.split(",")]
    wide = base in ("DFMA", "DADD", "DMUL", "DSETP") or ".64" in op or "F64" in op
    dst, src = [], []
    if parts and parts[0] and base not in ("BRA", "BSSY", "BSYNC", "ISETP", "DSETP", "FSETP",
                                           "STS", "STG"):
        d = regs(parts[0])
        if d:
            dst = [d[0], d[0] + 1] if (wide and base != "DSETP") or base == "F2I" and False else [d[0]]
            if base in ("DFMA", "DADD", "DMUL") or (base == "I2F" and "F64" in op):
                dst = [d[0], d[0] + 1]
        srcs = parts[1:]
    else:
        srcs = parts
    for a in srcs:
        for r in regs(a):
            src += [r, r + 1] if wide else [r]
    parsed.append((base, dst, src))


def simulate(nwarps, passes=4):
    ready = [dict() for _ in range(nwarps)]
    pc = [0] * nwarps
    t_next = [0] * nwarps
    fp_free = 0
    cyc = 0
    done = [0] * nwarps
    n = len(parsed)
    rr = 0
    while min(done) < passes:
        issued = False
        for k in range(nwarps):
            w = (rr + k) % nwarps
            if done[w] >= passes:
                continue
            base, dst, src = parsed[pc[w]]
            if t_next[w] > cyc:
                continue
            if any(ready[w].get(r, 0) > cyc for r in src):
                continue
            if base in FP64 and fp_free > cyc:
                continue
            lat = LAT.get(base, 6)
            for r in dst:
                ready[w][r] = cyc + lat
            if base in FP64:
                fp_free = cyc + 2
            t_next[w] = cyc + 1
            pc[w] += 1
            if pc[w] == n:
                pc[w] = 0
                done[w] += 1
            issued = True
            rr = w + 1
            break
        cyc += 1
    return cyc / passes


c = Counter(p[0] for p in parsed)
nfp = sum(c[o] for o in FP64)
print(f"hot instructions {len(parsed)} (fp64 {nfp}); pipe bound/pass {2 * nfp} cycles")
for w in (1, 2, 3, 4):
    cyc = simulate(w)
    print(f"{w} warp(s): {cyc:.0f} cycles per pass of all warps -> {cyc / w:.0f} per warp-pass,"
          f" fp64 pipe busy {2 * nfp * w / cyc:.0%}")
