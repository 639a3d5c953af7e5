import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2405_19493_b200 import engine, make_sampler, make_source
out = torch.empty(1 << 24, dtype=torch.float64, device="cuda")
engine.fill_gaussians(make_sampler(sys.argv[1]), make_source(sys.argv[2], 5), out)
torch.cuda.synchronize()
