"""One single-stream fill (for ncu launch lists): one_single.py SAMPLER SOURCE [LOG2N]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2405_19493_b200 import engine, make_sampler, make_source
n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 24)
out = torch.empty(n, dtype=torch.float64, device="cuda")
engine.fill_gaussians(make_sampler(sys.argv[1]), make_source(sys.argv[2], 5), out)
torch.cuda.synchronize()
