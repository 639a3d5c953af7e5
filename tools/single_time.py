"""Device time of one single-stream fill (engine.fill_gaussians on a device tensor):
python tools/single_time.py SAMPLER SOURCE LOG2N [REPS]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_19493_b200 import engine, make_sampler, make_source
alg, srcid, lg = sys.argv[1], sys.argv[2], int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
n = 1 << lg
out = torch.empty(n, dtype=torch.float64, device="cuda")
smp, src = make_sampler(alg), make_source(srcid, 5)
for _ in range(3):
    engine.fill_gaussians(smp, src, out)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(reps):
    engine.fill_gaussians(smp, src, out)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / reps
print(f"{alg} {srcid} 2^{lg}: {dt*1e6:.1f} us per call, {n/dt/1e9:.2f} G/s, {dt/n*1e9:.3f} ns/op", flush=True)
