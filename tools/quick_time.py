"""Quick device timing of each config's fill kernel (CUDA events, after warm-up)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_19493_b200 import streams

def t5(reps=5, gens=10):
    n, genes = 65536, 1024
    x, sig = streams.init_population(n, genes, seed=2024)
    st = streams.config_states("c5", 0, n)
    for _ in range(2):
        streams.mutate(st, x, sig, gens, sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        streams.mutate(st, x, sig, gens, sync=False)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nv = n * genes * gens
    print(f"c5: {n}x{genes}x{gens} {ms:.3f} ms  {nv/ms/1e6:.1f} Gvar/s  {nv*16/ms/1e6:.0f} GB/s", flush=True)


def t(cfg, n=None, reps=10):
    if cfg == "c5":
        return t5()
    checks = cfg.endswith("s")
    cfg = cfg.rstrip("s")
    c = streams.CONFIGS[cfg]
    n = n or c.n_streams
    st0 = streams.config_states(cfg, 0, n)
    out = torch.empty((n, c.n_per), dtype=torch.float64, device="cuda")
    kw = {}
    if c.sampler == "polar":
        kw = dict(spare=torch.zeros(n, dtype=torch.float64, device="cuda"), has_spare=torch.zeros(n, dtype=torch.uint8, device="cuda"))
    if checks:
        kw["checksum"] = torch.zeros(n, dtype=torch.int64, device="cuda")
        kw["psum"] = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    for _ in range(3):
        st = st0.clone(); streams.fill_gaussians_streams(c.sampler, c.source, st, out, sync=False, **kw)
    torch.cuda.synchronize()
    sts = [st0.clone() for _ in range(reps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        streams.fill_gaussians_streams(c.sampler, c.source, sts[k], out, sync=False, **kw)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nv = n * c.n_per
    print(f"{cfg}{'+stats' if checks else ''}: {n}x{c.n_per} {ms:.3f} ms  {nv/ms/1e6:.1f} Gvar/s  {nv*8/ms/1e6:.0f} GB/s", flush=True)

pol = os.environ.get("GZ_POLICY", "auto")
streams.set_kernel_policy(pol)
print("policy", pol)
for cfg in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
    t(cfg)
