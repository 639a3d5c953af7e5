"""Device time of one fill shape: shape_time.py ALG SOURCE N_STREAMS N_PER [REPS]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2405_19493_b200 import streams

alg, source, n, n_per = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
rng = np.random.default_rng(5)
st_np = (rng.integers(0, 2 ** 48, size=n, dtype=np.uint64) if source == "lcg48"
         else rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) | np.uint64(1))
st0 = torch.from_numpy(np.ascontiguousarray(st_np).view(np.int64).copy()).cuda()
out = torch.empty((n, n_per), dtype=torch.float64, device="cuda")
for _ in range(3):
    streams.fill_gaussians_streams(alg, source, st0.clone(), out)
sts = [st0.clone() for _ in range(reps)]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(reps):
    streams.fill_gaussians_streams(alg, source, sts[k], out, sync=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"{alg} {source} {n}x{n_per}: {ms * 1e3:.1f} us  {n * n_per / ms / 1e6:.1f} G/s  env={ {k: v for k, v in os.environ.items() if k.startswith('GZ_')} }", flush=True)
