"""Attribute ncu per-instruction counts to source lines.

    python tools/sass_lines.py NVDISASM_G_DUMP FUNCTION NCU_SASS_CSV [TOP]

NVDISASM_G_DUMP: `nvdisasm -g` of the cubin (cuobjdump -xelf all lib.so); FUNCTION:
mangled name; NCU_SASS_CSV: `ncu -i rep --page source --print-source sass --csv`.
The two listings are aligned by instruction order.
"""
import collections
import csv
import re
import sys

dump, fn, ncsv = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(dump).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(fn + ":"))
cur = ("?", 0)
seq = []
for l in lines[start + 1:]:
    if l.startswith(".") and not l.startswith(".L"):
        break
    if l.startswith("_Z") and l.endswith(":"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m:
        seq.append((cur, m.group(2)))
rows = list(csv.reader(open(ncsv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ncu = [r for r in rows[2:] if len(r) >= len(hdr)]
print(f"disasm {len(seq)} instructions, ncu {len(ncu)} rows")
n = min(len(seq), len(ncu))
bad = sum(1 for k in range(n) if seq[k][1].split()[0].lstrip("@!P0123456789T ") [:3] not in ncu[k][ix["Source"]])
print("opcode mismatches in alignment:", bad)
agg = collections.Counter()
smp = collections.Counter()
tot = 0
for k in range(n):
    e = int(ncu[k][ix["Instructions Executed"]] or 0)
    s = int(ncu[k][ix["Warp Stall Sampling (All Samples)"]] or 0)
    agg[seq[k][0]] += e
    smp[seq[k][0]] += s
    tot += e
ts = sum(smp.values())
print(f"total warp-instructions {tot}, samples {ts}")
for (f, ln), e in agg.most_common(top):
    print(f"{f}:{ln:<5d} {e:12d} {100 * e / tot:5.1f}%  samples {100 * smp[(f, ln)] / max(ts, 1):5.1f}%")
