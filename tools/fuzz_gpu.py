"""Randomised parity sweep of the CUDA engine against the CPU oracle (test tool).

    python tools/fuzz_gpu.py SECONDS [SEED]

Random pairing, stream count, row length, states, polar spares, kernel policy and
device or host (numpy, gz_fill_gaussians_host) buffers per case, plus random
mutate (config-5) and fill_u64 cases; every output, final state and spare must equal the oracle's bit for bit.
Prints one line per 50 cases and a final summary; exits 1 on the first mismatch.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import gz_oracle as O
import paper_2405_19493_b200 as gz
from paper_2405_19493_b200 import _lib, streams
from paper_2405_19493_b200.engine import table_slot
from paper_2405_19493_b200.samplers import make_sampler

DRY = False     # main(): replay a case's random draws without running it (GZ_FUZZ_SKIP=N skips the first N cases)
LAST = ""       # the case being run, printed when it raises

PAIRINGS = [(s, a) for s in ("lcg48", "splitmix") for a in ("polar", "ziggurat", "modified-ziggurat")]


def one_case(rng):
    source, alg = PAIRINGS[rng.integers(len(PAIRINGS))]
    shape = rng.integers(4)
    if shape == 0:
        n, n_per = 1, int(rng.integers(32768, 300000))          # whole-GPU single-stream decode
    elif shape == 1:
        n, n_per = int(rng.integers(1, 200)), int(rng.integers(0, 3000))
    elif shape == 2:
        n, n_per = int(rng.integers(32768, 45000)), int(rng.integers(1, 80))
    else:
        n, n_per = int(rng.integers(200, 3000)), int(rng.integers(0, 600))
    policy = ["auto", "warp", "lane", "lane-tma"][rng.integers(4)]
    raw = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=(n, 2),
                                                                                               dtype=np.uint64)
    st_np = raw[:, 0] & np.uint64((1 << 48) - 1) if source == "lcg48" else raw.copy()
    if source == "splitmix":
        st_np[:, 1] |= np.uint64(1)
    kw, sp, hs = {}, None, None
    if alg == "polar":
        hs = rng.integers(0, 2, size=n).astype(np.uint8)
        sp = rng.standard_normal(n) * hs
        kw = dict(spare=torch.from_numpy(sp.copy()).cuda(), has_spare=torch.from_numpy(hs.copy()).cuda())
    host = bool(rng.integers(2))      # host buffers through gz_fill_gaussians_host
    guard = 1_000_000 if rng.random() < 0.8 else int(rng.integers(1, 6))
    global LAST
    LAST = f"{source}/{alg} n={n} n_per={n_per} policy={policy} host={host} guard={guard}"
    if DRY:
        return 0
    tripped = False
    streams.set_kernel_policy(policy)
    try:
        if host:
            L = _lib.load()
            a = {"polar": 0, "ziggurat": 1, "modified-ziggurat": 2}[alg]
            slot = table_slot(make_sampler(alg).tables) if a else 0
            st_in = np.ascontiguousarray(st_np)
            st_h = np.empty_like(st_in)
            out_h = np.empty((n, n_per))
            sp_o, hs_o = np.zeros(n), np.zeros(n, dtype=np.uint8)
            pp = lambda x: x.ctypes.data if x is not None else None
            _lib.check(L.gz_fill_gaussians_host(a, _lib.SRC[source], slot, n, n_per, pp(st_in), pp(st_h),
                                                pp(sp) if a == 0 else None, pp(hs) if a == 0 else None,
                                                pp(sp_o) if a == 0 else None, pp(hs_o) if a == 0 else None,
                                                pp(out_h), None, guard))
            got, got_st = out_h, st_h.reshape(-1)
            if a == 0:
                kw = dict(spare=torch.from_numpy(sp_o), has_spare=torch.from_numpy(hs_o))
        else:
            st = torch.from_numpy(np.ascontiguousarray(st_np).view(np.int64).copy()).cuda()
            out = torch.empty((n, n_per), dtype=torch.float64, device="cuda")
            streams.fill_gaussians_streams(alg, source, st, out, guard=guard, **kw)
            got, got_st = out.cpu().numpy(), st.cpu().numpy().view(np.uint64)
    except gz.RejectionLoopExceeded:
        tripped = True
    finally:
        streams.set_kernel_policy("auto")
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians(alg, source, st_np, n_per,
                                                             *((sp, hs) if alg == "polar" else (None, None)),
                                                             guard=guard)
    desc = f"{source}/{alg} n={n} n_per={n_per} policy={policy} host={host} guard={guard}"
    assert tripped == (status == 1), "guard status " + desc
    if tripped:
        return 0
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), "values " + desc
    assert np.array_equal(got_st.reshape(ref_st.shape), ref_st), "state " + desc
    if alg == "polar":
        h = kw["has_spare"].cpu().numpy()
        assert np.array_equal(h, ref_has), "has " + desc
        assert np.array_equal((kw["spare"].cpu().numpy() * h).view(np.uint64), (ref_sp * ref_has).view(np.uint64)), \
            "spare " + desc
    return n * n_per


def mutate_case(rng):
    n, genes, gens = int(rng.integers(1, 3000)), int(rng.integers(1, 700)), int(rng.integers(1, 4))
    pad = int(rng.integers(0, 3))
    policy = ["auto", "warp", "lane", "lane-tma"][rng.integers(4)]
    st_np = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64)
    st_np[:, 1] |= np.uint64(1)
    x_np = rng.standard_normal((n, genes))
    sig = np.abs(rng.standard_normal(n)) * (rng.random(n) < 0.9)
    full = torch.zeros((n, genes + pad), dtype=torch.float64, device="cuda")
    full[:, :genes] = torch.from_numpy(x_np)
    x = full[:, :genes]
    st = torch.from_numpy(st_np.view(np.int64).copy()).cuda()
    guard = 1_000_000 if rng.random() < 0.8 else int(rng.integers(1, 6))
    global LAST
    LAST = f"mutate n={n} genes={genes} gens={gens} pad={pad} policy={policy} guard={guard}"
    if DRY:
        return 0
    tripped = False
    streams.set_kernel_policy(policy)
    try:
        streams.mutate(st, x, torch.from_numpy(sig).cuda(), gens, guard=guard)
    except gz.RejectionLoopExceeded:
        tripped = True
    finally:
        streams.set_kernel_policy("auto")
    xr = x_np.copy()
    ref_st, status = O.mutate(st_np, xr, sig, gens, guard=guard)
    desc = f"mutate n={n} genes={genes} gens={gens} pad={pad} policy={policy} guard={guard}"
    assert tripped == (status == 1), "guard status " + desc
    if tripped:
        return 0
    assert np.array_equal(x.cpu().numpy().view(np.uint64), xr.view(np.uint64)), "values " + desc
    assert np.array_equal(st.cpu().numpy().view(np.uint64), ref_st), "state " + desc
    return n * genes * gens


def u64_case(rng):
    source = ["lcg48", "splitmix"][rng.integers(2)]
    n, n_per = (1, int(rng.integers(1, 400000))) if rng.integers(2) else (int(rng.integers(1, 5000)),
                                                                          int(rng.integers(0, 300)))
    st_np = rng.integers(0, 2 ** 48, size=n, dtype=np.uint64) if source == "lcg48" else \
        rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) | np.uint64(1)
    global LAST
    LAST = f"u64 {source} n={n} n_per={n_per}"
    if DRY:
        return 0
    st = torch.from_numpy(np.ascontiguousarray(st_np).view(np.int64).copy()).cuda()
    out = torch.empty((n, n_per), dtype=torch.int64, device="cuda")
    streams.fill_u64_streams(source, st, out)
    ref, ref_st = O.fill_u64(source, st_np, n_per)
    desc = f"u64 {source} n={n} n_per={n_per}"
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref), "values " + desc
    assert np.array_equal(st.cpu().numpy().view(np.uint64).reshape(ref_st.shape), ref_st), "state " + desc
    return n * n_per


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
    t_end = time.time() + secs
    cases = total = 0
    skip = int(os.environ.get("GZ_FUZZ_SKIP", "0"))
    global DRY
    while time.time() < t_end:
        DRY = cases < skip
        try:
            k = rng.random()
            total += (one_case if k < 0.7 else mutate_case if k < 0.9 else u64_case)(rng)
        except AssertionError as e:
            print("MISMATCH", e, flush=True)
            return 1
        except Exception as e:  # noqa: BLE001 -- a CUDA error: say which case
            print(f"ERROR in case {cases}: {LAST}: {e!r}", flush=True)
            return 1
        cases += 1
        if cases % 50 == 0:
            print(f"{cases} cases, {total} deviates ok", flush=True)
    print(f"fuzz ok: {cases} cases, {total} deviates, all bit-exact", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
