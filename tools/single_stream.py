"""Single-stream fill rate through the reference-facing API (engine.fill_gaussians on one
stream), CUDA tensor out (device time) and numpy out (host round trip)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2405_19493_b200 import engine, make_sampler, make_source

for n in (1 << 20, 1 << 24):
    for src, alg in (("lcg48", "polar"), ("splitmix", "ziggurat"), ("splitmix", "modified-ziggurat")):
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        engine.fill_gaussians(make_sampler(alg), make_source(src, 1), out)
        torch.cuda.synchronize()
        t = time.perf_counter()
        engine.fill_gaussians(make_sampler(alg), make_source(src, 2), out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        buf = np.empty(n)
        t = time.perf_counter()
        engine.fill_gaussians(make_sampler(alg), make_source(src, 3), buf)
        dh = time.perf_counter() - t
        t = time.perf_counter()
        engine.fill_gaussians(make_sampler(alg), make_source(src, 4), buf)   # reused (touched) buffer
        dr = time.perf_counter() - t
        print(f"n=2^{n.bit_length()-1} {src}/{alg}: device out {dt*1e3:.2f} ms ({dt/n*1e9:.2f} ns/var), "
              f"fresh numpy out {dh*1e3:.2f} ms ({dh/n*1e9:.2f} ns/var), reused numpy {dr*1e3:.2f} ms", flush=True)
