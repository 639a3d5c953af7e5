"""Per-instruction stall reasons from an `ncu --page source --print-source sass --csv` dump:
stall_lines.py SRC.csv [N] -- the N lines with most samples, with their main stall reasons."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ins = []
base = None
for r in rows[2:]:
    if len(r) < len(hdr): continue
    a = int(r[ix["Address"]], 16); base = a if base is None else base
    st = {h[6:]: int(r[ix[h]] or 0) for h in sc}
    ins.append((a - base, int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), int(r[ix["Instructions Executed"]] or 0), st, r[ix["Source"]].strip()))
tot = sum(i[1] for i in ins) or 1
agg = {}
for i in ins:
    for k, v in i[3].items(): agg[k] = agg.get(k, 0) + v
print("all samples", tot, " ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
for off, s, n, st, src in sorted(ins, key=lambda x: -x[1])[:N]:
    top = " ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{off:05x} {100*s/tot:5.2f}% exec={n/1e6:7.3f}M {src[:48]:48s} {top}")
