"""Few-stream ziggurat (k_zig_seg) against the oracle over a grid of shapes (tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gz_oracle as O
from paper_2405_19493_b200 import streams

bad = 0
for source in ("splitmix", "lcg48"):
    for alg in ("ziggurat", "modified-ziggurat"):
        for n, n_per in ((1, 512), (1, 20000), (2, 700), (7, 4096), (100, 1000), (1024, 4096), (1100, 600), (300, 513)):
            rng = np.random.default_rng(n * 7919 + n_per)
            if source == "lcg48":
                st_np = rng.integers(0, 2 ** 48, size=n, dtype=np.uint64)
            else:
                st_np = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) | np.uint64(1)
            st = torch.from_numpy(np.ascontiguousarray(st_np).view(np.int64).copy()).cuda()
            out = torch.empty((n, n_per), dtype=torch.float64, device="cuda")
            streams.fill_gaussians_streams(alg, source, st, out)
            ref, ref_st, *_ = O.fill_gaussians(alg, source, st_np, n_per)
            ok_v = np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64))
            ok_s = np.array_equal(st.cpu().numpy().view(np.uint64).reshape(ref_st.shape), ref_st)
            if not (ok_v and ok_s):
                bad += 1
                g = out.cpu().numpy().view(np.uint64)
                rows = np.nonzero((g != ref.view(np.uint64)).any(1))[0]
                print("MISMATCH", source, alg, n, n_per, "values", ok_v, "state", ok_s, "rows", rows[:5],
                      "first col", np.nonzero(g[rows[0]] != ref.view(np.uint64)[rows[0]])[0][:5] if len(rows) else None,
                      flush=True)
print("seg_check bad", bad, "env", {k: v for k, v in os.environ.items() if k.startswith("GZ_")}, flush=True)
