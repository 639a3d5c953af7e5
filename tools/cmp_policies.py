"""Bit-compare two kernel policies on a config-4 block with fused witnesses:
cmp_policies.py POLICY_A POLICY_B [N_STREAMS] (deviates, states, checksums, power sums)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_19493_b200 import streams

n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20
res = []
for pol in sys.argv[1:3]:
    streams.set_kernel_policy(pol)
    st = streams.config_states("c4", 0, n)
    out = torch.empty((n, 256), dtype=torch.float64, device="cuda")
    ck = torch.zeros(n, dtype=torch.int64, device="cuda")
    ps = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, out, checksum=ck, psum=ps)
    res.append((out.view(torch.int64), st, ck, ps.view(torch.int64)))
streams.set_kernel_policy("auto")
names = ["deviates", "states", "checksums", "power sums"]
bad = [names[i] for i in range(4) if not torch.equal(res[0][i], res[1][i])]
print(f"{sys.argv[1]} vs {sys.argv[2]} on {n} streams:", "identical" if not bad else f"DIFFER in {bad}")
sys.exit(1 if bad else 0)
