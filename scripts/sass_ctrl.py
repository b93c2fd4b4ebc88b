"""Decode the scheduling control bits (stall, yield, barriers) of a kernel's SASS.

usage: python scripts/sass_ctrl.py all.sass <mangled-prefix> <start-hex> <end-hex>
Prints each instruction with its stall count and barrier waits, and the sum of
stall counts over the range (a lower bound on single-warp cycles).
"""
import re
import sys

text = open(sys.argv[1]).read()
blocks = re.split(r"\n\s*Function : ", text)
fn = [b for b in blocks if b.startswith(sys.argv[2])][0]
lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
lines = fn.splitlines()
tot = 0
waits = 0
rows = []
for i, l in enumerate(lines):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]+) \*/", l)
    if not m:
        continue
    addr = int(m.group(1), 16)
    if not lo <= addr <= hi:
        continue
    hiword = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1]).group(1)
    h = int(hiword, 16)
    ctrl = h >> 41
    stall = ctrl & 0xF
    yld = (ctrl >> 4) & 1
    wrb = (ctrl >> 5) & 7
    rdb = (ctrl >> 8) & 7
    wmask = (ctrl >> 11) & 0x3F
    reuse = (ctrl >> 17) & 0xF
    tot += stall
    waits += wmask != 0
    rows.append((addr, stall, yld, wrb, rdb, wmask, m.group(2).strip()))
for addr, stall, yld, wrb, rdb, wmask, ins in rows:
    print(f"{addr:6x} S{stall:2d} {'Y' if yld else ' '} wr{wrb if wrb != 7 else '-'} "
          f"rd{rdb if rdb != 7 else '-'} w{wmask:06b}  {ins[:70]}")
print(f"instructions {len(rows)}, sum of stall counts {tot}, instructions waiting on barriers {waits}")
