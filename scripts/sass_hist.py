"""Opcode histogram of a kernel's hottest loop (largest backward-branch body).

usage: python scripts/sass_hist.py <all.sass> <mangled-name-substring>
"""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read()
blocks = re.split(r"\n\s*Function : ", text)
fn = [b for b in blocks if b.startswith(sys.argv[2])][0]
ins = []
for line in fn.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)\s*([^;]*);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4), m.group(2) or ""))
loops = []
for a, op, args, pred in ins:
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", args)
        if t and int(t.group(1), 16) < a:
            lo = int(t.group(1), 16)
            body = [x for x in ins if lo <= x[0] <= a]
            nfp = sum(1 for x in body if x[1].split(".")[0] in ("DFMA", "DADD", "DMUL", "DSETP"))
            loops.append((nfp, lo, a, body))
loops.sort(reverse=True)
for nfp, lo, hi, body in loops[:3]:
    c = Counter(x[1].split(".")[0] for x in body)
    print(f"loop 0x{lo:x}-0x{hi:x}: {len(body)} instrs, fp64 {nfp}")
    print("  ", sorted(c.items(), key=lambda kv: -kv[1]))
