"""Summarise an `ncu --page source --print-source sass --csv` dump: executed
instructions by opcode and the hottest instructions by stall samples."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); tot = 0; samples = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += n; tot += n
    samples.append((s, n, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:70]))
print("total warp-instructions executed:", tot)
for op, n in ops.most_common(25): print(f"{op:12s} {n:12d} {100*n/tot:5.1f}%")
print("--- hottest by stall samples")
for s, n, a, src in sorted(samples, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{s:7d} {n:10d} {a} {src}")
