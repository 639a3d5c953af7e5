"""Small launches of every kernel family, for compute-sanitizer (memcheck, racecheck,
synccheck): python tools/sanitize_cases.py CASE.  Each case checks its output
against the CPU oracle so a sanitizer run also shows the results are right.

Cases: tma (k_zig_tma + fused witnesses), ring (k_zig_lane), warp (k_zig), lseg
(k_zig_lseg), single (whole-GPU single-stream ziggurat and polar), polarq
(k_polar_q), polarlane (k_polar_lqd), mutate (k_zig_lane mutate + k_zig mutate).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import gz_oracle as O  # noqa: E402
from paper_2405_19493_b200 import engine, streams  # noqa: E402
import paper_2405_19493_b200 as gz  # noqa: E402


def check_fill(alg, src, cfg, n, n_per, policy="auto", stats=False):
    streams.set_kernel_policy(policy)
    st = streams.config_states(cfg, 0, n)
    st_np = st.cpu().numpy().view(np.uint64).copy()
    out = torch.empty((n, n_per), dtype=torch.float64, device="cuda")
    kw = {}
    if alg == "polar":
        kw = dict(spare=torch.zeros(n, dtype=torch.float64, device="cuda"),
                  has_spare=torch.zeros(n, dtype=torch.uint8, device="cuda"))
    if stats:
        kw.update(checksum=torch.zeros(n, dtype=torch.int64, device="cuda"),
                  psum=torch.zeros((n, 4), dtype=torch.float64, device="cuda"))
    streams.fill_gaussians_streams(alg, src, st, out, **kw)
    ref, ref_st, *_ = O.fill_gaussians(alg, src, st_np, n_per)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref.view(np.uint64)), (alg, src, policy)
    assert np.array_equal(st.cpu().numpy().view(np.uint64), ref_st)
    streams.set_kernel_policy("auto")


def main(case):
    if case == "tma":
        check_fill("ziggurat", "lcg48", "c4", 33000, 80, "lane", stats=True)
        check_fill("modified-ziggurat", "splitmix", "c3", 33000, 48, "lane")
    elif case == "ring":
        check_fill("ziggurat", "lcg48", "c4", 33000, 80, "lane-ring", stats=True)
    elif case == "warp":
        check_fill("ziggurat", "splitmix", "c1", 500, 300, "warp", stats=True)
        check_fill("modified-ziggurat", "lcg48", "c4", 500, 100, "warp")
    elif case == "lseg":
        check_fill("ziggurat", "splitmix", "c1", 64, 4096)
    elif case == "single":
        for alg, src in (("ziggurat", "splitmix"), ("polar", "lcg48")):
            smp = gz.make_sampler(alg)
            s = gz.make_source(src, 12345)
            s0 = gz.make_source(src, 12345)
            st0 = np.array([s0.state] if src == "lcg48" else [[s0.state, s0.gamma]], dtype=np.uint64)
            buf = np.empty(1 << 16)
            engine.fill_gaussians(smp, s, buf)
            ref, *_ = O.fill_gaussians(alg, src, st0, 1 << 16)
            assert np.array_equal(buf.view(np.uint64), ref[0].view(np.uint64)), alg
    elif case == "polarq":
        check_fill("polar", "lcg48", "c2", 3000, 256)
    elif case == "polarlane":
        check_fill("polar", "splitmix", "c1", 3000, 100, "lane")
    elif case == "mutate":
        for policy, n in (("lane", 33000), ("warp", 300)):
            streams.set_kernel_policy(policy)
            st_np = O.config_states_range("c5", 0, n)
            x_np = np.random.default_rng(1).standard_normal((n, 64))
            sig = np.abs(np.random.default_rng(2).standard_normal(n))
            x = torch.from_numpy(x_np.copy()).cuda()
            st = torch.from_numpy(st_np.view(np.int64).copy()).cuda()
            streams.mutate(st, x, torch.from_numpy(sig).cuda(), 2)
            ref_st, status = O.mutate(st_np, x_np, sig, 2)
            assert status == 0 and np.array_equal(x.cpu().numpy().view(np.uint64), x_np.view(np.uint64))
        streams.set_kernel_policy("auto")
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print("ok", case)


if __name__ == "__main__":
    main(sys.argv[1])
