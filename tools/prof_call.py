import sys, os, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2405_19493_b200 import engine, make_sampler, make_source, _lib
from paper_2405_19493_b200.engine import _io_words, _state_words, table_slot, _ptr
L = _lib.load()
n = 1 << 17
out = torch.empty(n, dtype=torch.float64, device="cuda")
smp, src = make_sampler("ziggurat"), make_source("splitmix", 1)
for _ in range(5): engine.fill_gaussians(smp, src, out)
torch.cuda.synchronize()
T = {}
def tick(k, t0):
    t1 = time.perf_counter(); T[k] = T.get(k, 0) + (t1 - t0); return t1
R = 200
for _ in range(R):
    t = time.perf_counter()
    st = _state_words(src); slot = table_slot(smp.tables); t = tick("prep", t)
    h, d = _io_words(out.device); hv = h.numpy(); hv[:] = 0; hv[:st.size] = st.view(np.int64); t = tick("hv", t)
    d.copy_(h, non_blocking=True); t = tick("h2d", t)
    base = d.data_ptr(); s = torch.cuda.current_stream(out.device).cuda_stream; t = tick("stream", t)
    _lib.check(L.gz_fill_gaussians(1, 1, slot, 1, n, n, ctypes.c_void_p(base), ctypes.c_void_p(base + 16), None, None, None, None, _ptr(out), None, None, 1000000, s)); t = tick("fill", t)
    h.copy_(d, non_blocking=True); t = tick("d2h", t)
    _lib.check(L.gz_stream_check(s)); t = tick("check", t)
    src.state = int(hv[2:3].view(np.uint64)[0]); t = tick("post", t)
for k, v in T.items(): print(f"{k:8s} {v / R * 1e6:7.1f} us")
print("total", sum(T.values()) / R * 1e6)
