"""Group an `ncu --page source --print-source sass --csv` dump into runs of equal
execution count (basic blocks) and print the heavy ones: offset, length, count,
share of executed instructions, share of stall samples, first instruction."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
ins = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    ins.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]].strip()))
base = ins[0][0]
blocks = []; cur = None
for a, n, s, src in ins:
    if cur is None or n != cur[2]:
        cur = [a - base, 0, n, 0, src]; blocks.append(cur)
    cur[1] += 1; cur[3] += s
tot = sum(b[1] * b[2] for b in blocks); ts = sum(b[3] for b in blocks) or 1
print("executed", tot, "samples", ts)
for b in blocks:
    if b[2] > 0 and b[1] * b[2] > thr * tot:
        print(f"{b[0]:05x} n={b[1]:3d} exec={b[2]/1e6:8.3f}M share={100*b[1]*b[2]/tot:5.1f}% stall={100*b[3]/ts:5.1f}%  {b[4][:50]}")
