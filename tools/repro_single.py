"""Search for single-stream polar/zig mismatches and print the first differing index."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gz_oracle as O
from paper_2405_19493_b200 import streams

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
alg = sys.argv[2] if len(sys.argv) > 2 else "polar"
source = sys.argv[3] if len(sys.argv) > 3 else "splitmix"
bad = 0
for it in range(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    n_per = int(rng.integers(32768, 300000))
    st_np = rng.integers(0, 2 ** 63, size=(1, 2), dtype=np.uint64)
    if source == "lcg48":
        st_np = st_np[:, 0] & np.uint64((1 << 48) - 1)
    else:
        st_np[:, 1] |= np.uint64(1)
    hs = np.array([it % 2], dtype=np.uint8)
    sp = np.array([0.5 * (it % 2)])
    kw = {}
    if alg == "polar":
        kw = dict(spare=torch.from_numpy(sp.copy()).cuda(), has_spare=torch.from_numpy(hs.copy()).cuda())
    st = torch.from_numpy(np.ascontiguousarray(st_np).view(np.int64).copy()).cuda()
    out = torch.empty((1, n_per), dtype=torch.float64, device="cuda")
    streams.fill_gaussians_streams(alg, source, st, out, **kw)
    ref, ref_st, _, _, _ = O.fill_gaussians(alg, source, st_np, n_per, *((sp, hs) if alg == "polar" else (None, None)))
    g = out.cpu().numpy().view(np.uint64)[0]
    r = ref.view(np.uint64)[0]
    d = np.nonzero(g != r)[0]
    stok = np.array_equal(st.cpu().numpy().view(np.uint64).reshape(ref_st.shape), ref_st)
    if len(d) or not stok:
        bad += 1
        i = d[0] if len(d) else -1
        print(f"it={it} n_per={n_per} spare={hs[0]} first_bad={i} n_bad={len(d)} state_ok={stok} "
              f"got={g[i:i+3].view(np.float64) if i >= 0 else None} ref={r[i:i+3].view(np.float64) if i >= 0 else None}",
              flush=True)
print("bad", bad)
