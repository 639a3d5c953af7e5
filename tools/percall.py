import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes
from paper_2405_19493_b200 import engine, make_sampler, make_source, _lib
n = 1 << 17
for alg, srcid in (("ziggurat", "splitmix"), ("polar", "lcg48")):
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    smp, src = make_sampler(alg), make_source(srcid, 1)
    for _ in range(5): engine.fill_gaussians(smp, src, out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(50): engine.fill_gaussians(smp, src, out)
    torch.cuda.synchronize()
    print(alg, "per call us", (time.perf_counter() - t) / 50 * 1e6)
    # raw ABI call on device state
    L = _lib.load()
    st = torch.tensor([1, 0x9E3779B97F4A7C15 - (1 << 64)] if srcid == "splitmix" else [1], dtype=torch.int64, device="cuda")
    slot = 0 if alg == "polar" else engine.table_slot(smp.tables)
    a = 0 if alg == "polar" else 1
    s = torch.cuda.current_stream().cuda_stream
    P = ctypes.c_void_p
    def raw():
        _lib.check(L.gz_fill_gaussians(a, _lib.SRC[srcid], slot, 1, n, n, P(st.data_ptr()), P(st.data_ptr()), None, None, None, None, P(out.data_ptr()), None, None, 1000000, s))
    for _ in range(5): raw()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(50): raw()
    torch.cuda.synchronize()
    print(alg, "raw ABI per call us", (time.perf_counter() - t) / 50 * 1e6)
