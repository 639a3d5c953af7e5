"""Run one config's fill a few times (for ncu captures): prof_one.py CFG [N_STREAMS] [REPS]
(CFG with a trailing 's', e.g. c4s: with the fused per-stream checksums and power sums)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_19493_b200 import streams

streams.set_kernel_policy(os.environ.get("GZ_POLICY", "auto"))
cfg = sys.argv[1]
stats = cfg.endswith("s")
cfg = cfg.rstrip("s")
if cfg == "c5":
    x, sig = streams.init_population(65536, 1024, seed=2024)
    st = streams.config_states("c5", 0, 65536)
    for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
        streams.mutate(st, x, sig, 10)
    torch.cuda.synchronize()
    print("done c5")
    raise SystemExit(0)
c = streams.CONFIGS[cfg]
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else c.n_streams
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
st0 = streams.config_states(cfg, 0, n)
out = torch.empty((n, c.n_per), dtype=torch.float64, device="cuda")
kw = {}
if c.sampler == "polar":
    kw = dict(spare=torch.zeros(n, dtype=torch.float64, device="cuda"), has_spare=torch.zeros(n, dtype=torch.uint8, device="cuda"))
if stats:
    kw["checksum"] = torch.zeros(n, dtype=torch.int64, device="cuda")
    kw["psum"] = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
for _ in range(reps):
    st = st0.clone()
    streams.fill_gaussians_streams(c.sampler, c.source, st, out, **kw)
torch.cuda.synchronize()
print("done", cfg, n)
