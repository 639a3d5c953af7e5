"""Parity of the CUDA engine with the reference (golden fixtures) and the CPU
oracle, bit for bit.  Needs a B200: run with `pytest -m gpu`.

Every test drives the product through its public API (engine.fill_gaussians /
fill_u64 with numpy or CUDA tensors, streams.*), i.e. through the C ABI of
libgzb200.so; the oracle (oracle/gz_oracle.c) and the golden fixtures
(tests/golden/golden.json, made by importing the reference) are the checkers.
"""
import ctypes
import hashlib
import zlib

import numpy as np
import pytest

from conftest import f64_to_hex, xor_hex

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import gz_oracle as O  # noqa: E402
import paper_2405_19493_b200 as gz  # noqa: E402
from paper_2405_19493_b200 import engine, streams  # noqa: E402

DEV = "cuda"
PAIRINGS = [(s, a) for s in ("lcg48", "splitmix") for a in ("polar", "ziggurat", "modified-ziggurat")]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


def spare_hex(sampler):
    return None if sampler.spare is None else f64_to_hex(np.array([sampler.spare]))[0]


def dev_states(source, states_np):
    return torch.from_numpy(np.ascontiguousarray(states_np, dtype=np.uint64).view(np.int64)).to(DEV)


# ---- reference-facing single-stream API ------------------------------------

@pytest.mark.parametrize("idx", range(6))
def test_six_pairings_300k_host_path(idx, golden):
    """tests/test_engine.py:16-28 through engine.fill_gaussians with a numpy out."""
    g = golden["pairings"][idx]
    smp = gz.make_sampler(g["sampler"])
    src = gz.make_source(g["source"], g["seed"])
    buf = np.empty(g["n"])
    engine.fill_gaussians(smp, src, buf)
    assert f64_to_hex(buf[:16]) == g["first"]
    assert sha(buf) == g["sha256"]
    assert "%016x" % src.state == g["state"]
    if g["sampler"] == "polar":
        assert spare_hex(smp) == g["spare"]


@pytest.mark.parametrize("idx", range(6))
def test_six_pairings_300k_device_tensor(idx, golden):
    g = golden["pairings"][idx]
    smp = gz.make_sampler(g["sampler"])
    src = gz.make_source(g["source"], g["seed"])
    out = torch.empty(g["n"], dtype=torch.float64, device=DEV)
    engine.fill_gaussians(smp, src, out)
    assert sha(out.cpu().numpy()) == g["sha256"]
    assert "%016x" % src.state == g["state"]
    if g["sampler"] == "polar":
        assert spare_hex(smp) == g["spare"]


def test_small_and_edge_sizes(golden):
    for g in golden["small"]:
        smp = gz.make_sampler(g["sampler"])
        src = gz.make_source(g["source"], int(g["seed"], 16))
        buf = np.empty(g["n"])
        engine.fill_gaussians(smp, src, buf)
        assert f64_to_hex(buf) == g["out"], (g["source"], g["sampler"], g["n"])
        assert "%016x" % src.state == g["state"]
        if g["sampler"] == "polar":
            assert spare_hex(smp) == g["spare"]


def test_polar_spare_carries_across_batches(golden):
    """tests/test_engine.py:58-71."""
    g = golden["polar_chunks"]
    smp = gz.make_sampler("polar")
    src = gz.make_source("lcg48", g["seed"])
    chunks = []
    for size in g["sizes"]:
        buf = np.empty(size)
        engine.fill_gaussians(smp, src, buf)
        chunks.append(buf)
    assert f64_to_hex(np.concatenate(chunks)) == g["out"]
    assert spare_hex(smp) == g["spare"]


def test_engine_and_per_call_interleave():
    """tests/test_engine.py:43-55: batch then per-call continue one stream."""
    smp, src = gz.make_sampler("ziggurat"), gz.make_source("splitmix", 7)
    buf = np.empty(1000)
    engine.fill_gaussians(smp, src, buf)
    tail = [smp.next_gaussian(src) for _ in range(20)]
    ref, *_ = O.fill_gaussians("ziggurat", "splitmix", np.array([[7, O.GOLDEN_GAMMA]], dtype=np.uint64), 1020)
    assert bits_equal(np.concatenate([buf, tail]), ref[0])


@pytest.mark.parametrize("source", ["lcg48", "splitmix"])
def test_fill_u64_matches_reference(source, golden):
    g = golden["u64"][source]
    src = gz.make_source(source, g["seed"])
    buf = np.empty(g["n"], dtype=np.uint64)
    engine.fill_u64(src, buf)
    assert sha(buf) == g["sha256"]
    assert "%016x" % src.state == g["state"]


def test_scripted_sources_replay_like_the_reference(golden_cli):
    """Scripted words (the reference's test double) replayed on the device call by call:
    fast path, sign flip, tail, wedge accept/reject, the modified layout, polar with
    spares, and exhaustion -- values, cursor and spare equal the reference's."""
    assert engine.supports(gz.ScriptedSource([1, 2, 3]))
    for r in golden_cli["scripted"]:
        smp = gz.make_sampler(r["sampler"])
        if r["spare_in"] is not None:
            smp.spare = r["spare_in"]
        src = gz.ScriptedSource([int(w, 16) for w in r["words"]])
        vals = []
        if r["exhausted"]:
            with pytest.raises(gz.ScriptExhausted):
                for _ in range(r["n"]):
                    vals.append(smp.next_gaussian(src).hex())
        else:
            buf = np.empty(r["n"])
            engine.fill_gaussians(smp, src, buf)
            vals = [float(v).hex() for v in buf]
        assert vals == r["values"], r["sampler"]
        assert src.cursor == r["cursor"]
        if not r["exhausted"]:
            assert (None if smp.__dict__.get("spare") is None else smp.spare.hex()) == r["spare_out"]


def test_tail_sample_scripted_matches_reference(golden_cli):
    for rr, words, v in golden_cli["tail"]:
        src = gz.ScriptedSource([int(w, 16) for w in words])
        assert gz.tail_sample(src, rr).hex() == v


# ---- multi-stream hot path ------------------------------------------------------

@pytest.fixture(params=["warp", "lane", "lane-ring", "lane-tma"])
def policy(request):
    streams.set_kernel_policy(request.param)
    yield request.param
    streams.set_kernel_policy("auto")


@pytest.mark.parametrize("source,alg", PAIRINGS)
@pytest.mark.parametrize("n_per", [1, 2, 7, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 1000])
def test_random_streams_vs_oracle(source, alg, n_per, policy):
    rng = np.random.default_rng(zlib.crc32(f"{source}/{alg}/{n_per}".encode()))
    n = 2011 if n_per <= 257 else 509     # not a multiple of 32: partial warps
    raw = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=(n, 2),
                                                                                                   dtype=np.uint64)
    if source == "lcg48":
        st_np = raw[:, 0] & np.uint64((1 << 48) - 1)
    else:
        st_np = raw.copy()
        st_np[:, 1] |= np.uint64(1)
    st = dev_states(source, st_np)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    kw = {}
    if alg == "polar":
        has = rng.integers(0, 2, size=n).astype(np.uint8)
        spare = rng.standard_normal(n) * has
        kw = dict(spare=torch.from_numpy(spare).to(DEV), has_spare=torch.from_numpy(has).to(DEV))
    streams.fill_gaussians_streams(alg, source, st, out, **kw)
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians(
        alg, source, st_np, n_per, *( (spare, has) if alg == "polar" else (None, None)))
    assert status == 0
    got = out.cpu().numpy()
    diff = np.nonzero((got.view(np.uint64) != ref.view(np.uint64)).any(axis=1))[0]
    assert diff.size == 0, f"{diff.size} streams differ, first {diff[:5]}"
    assert np.array_equal(u64(st), ref_st)
    if alg == "polar":
        assert np.array_equal(kw["has_spare"].cpu().numpy(), ref_has)
        assert bits_equal(kw["spare"].cpu().numpy() * (ref_has > 0), ref_sp * (ref_has > 0))


def test_strided_rows_and_fused_witnesses(policy):
    n, n_per, ld = 300, 200, 256
    st_np = O.config_states("c4", range(n))
    st = dev_states("lcg48", st_np)
    big = torch.full((n, ld), -7.0, dtype=torch.float64, device=DEV)
    out = big[:, :n_per]
    ck = torch.zeros(n, dtype=torch.int64, device=DEV)
    ps = torch.zeros((n, 4), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, out, checksum=ck, psum=ps)
    ref, *_ = O.fill_gaussians("ziggurat", "lcg48", st_np, n_per)
    assert bits_equal(out.cpu().numpy(), ref)
    assert (big[:, n_per:] == -7.0).all()
    assert [("%016x" % v) for v in u64(ck)] == [xor_hex(ref[i]) for i in range(n)]
    ps_ref = np.stack([ref.sum(1), (ref ** 2).sum(1), (ref ** 3).sum(1), (ref ** 4).sum(1)], 1)
    np.testing.assert_allclose(ps.cpu().numpy(), ps_ref, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("source", ["lcg48", "splitmix"])
@pytest.mark.parametrize("alg", ["ziggurat", "modified-ziggurat"])
@pytest.mark.parametrize("n,n_per,ld,stats", [(40000, 255, 256, True), (33000, 17, 20, False), (32768, 3, 4, True),
                                               (36000, 101, 104, False)])
def test_zig_lst_odd_rows_strided(source, alg, n, n_per, ld, stats):
    """k_zig_lst (the auto choice from 32768 streams when rows are 32-byte aligned and the
    stride a multiple of 4) on rows whose length is NOT a multiple of 4: the last partial
    chunk of a row leaves from the ring-addressed staging slots at the row transition, the
    next row starts on a chunk boundary.  With and without the fused witnesses; bit-exact
    against the oracle, the padding untouched (engine.py:75-151 per stream)."""
    rng = np.random.default_rng(n + n_per)
    if source == "lcg48":
        st_np = rng.integers(0, 1 << 48, size=n, dtype=np.uint64)
    else:
        st_np = rng.integers(0, 1 << 63, size=(n, 2), dtype=np.uint64)
        st_np[:, 1] |= np.uint64(1)
    st = dev_states(source, st_np)
    big = torch.full((n, ld), -7.0, dtype=torch.float64, device=DEV)
    out = big[:, :n_per]
    kw = {}
    if stats:
        kw = dict(checksum=torch.zeros(n, dtype=torch.int64, device=DEV),
                  psum=torch.zeros((n, 4), dtype=torch.float64, device=DEV))
    streams.fill_gaussians_streams(alg, source, st, out, **kw)
    ref, ref_st, *_ = O.fill_gaussians(alg, source, st_np, n_per)
    assert bits_equal(out.cpu().numpy(), ref)
    assert (big[:, n_per:] == -7.0).all()
    assert np.array_equal(u64(st).reshape(ref_st.shape), ref_st)
    if stats:
        ck_ref = np.bitwise_xor.reduce(ref.view(np.uint64), axis=1)
        assert np.array_equal(u64(kw["checksum"]), ck_ref)
        ps_ref = np.stack([ref.sum(1), (ref ** 2).sum(1), (ref ** 3).sum(1), (ref ** 4).sum(1)], 1)
        np.testing.assert_allclose(kw["psum"].cpu().numpy(), ps_ref, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("n,n_per,ld", [(40000, 255, 256), (33000, 17, 20), (2011, 101, 104), (700, 3, 4)])
def test_polar_lane_odd_rows_strided_with_spares(n, n_per, ld):
    """k_polar_lst (polar, a lane per stream; the auto choice from 32768 streams, policy
    'lane' below) on odd row lengths inside 32-byte-aligned strided rows: incoming
    spares first, the last pair's second deviate carried out as the spare, the padding
    untouched -- against the oracle, per stream."""
    rng = np.random.default_rng(n * 1000 + n_per)
    st_np = O.config_states("c2", range(n))
    has = rng.integers(0, 2, size=n).astype(np.uint8)
    spare = rng.standard_normal(n) * has
    st = dev_states("lcg48", st_np)
    big = torch.full((n, ld), -9.0, dtype=torch.float64, device=DEV)
    out = big[:, :n_per]
    sp = torch.from_numpy(spare).to(DEV)
    hs = torch.from_numpy(has).to(DEV)
    if n < 32768:
        streams.set_kernel_policy("lane")
    try:
        streams.fill_gaussians_streams("polar", "lcg48", st, out, spare=sp, has_spare=hs)
    finally:
        streams.set_kernel_policy("auto")
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians("polar", "lcg48", st_np, n_per, spare, has)
    assert status == 0
    assert bits_equal(out.cpu().numpy(), ref)
    assert (big[:, n_per:] == -9.0).all()
    assert np.array_equal(u64(st), ref_st)
    assert np.array_equal(hs.cpu().numpy(), ref_has)
    assert bits_equal(sp.cpu().numpy() * (ref_has > 0), ref_sp * (ref_has > 0))


# ---- the five configs ---------------------------------------------------------

def test_config1_full(golden):
    g = golden["configs"]["c1"]
    st = streams.config_states("c1", 0, 1024)
    out = torch.empty((1024, 4096), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams("ziggurat", "splitmix", st, out)
    got = out.cpu().numpy()
    assert [xor_hex(got[i]) for i in range(1024)] == g["xor"]
    assert ["%016x" % v for v in u64(st)[:, 0]] == g["state"]
    assert sha(got) == g["sha256"]


def _sampled(cfg, golden, n_total, n_per, alg, source):
    recs = golden["configs"][cfg]
    st = streams.config_states(cfg, 0, n_total)
    out = torch.empty((n_total, n_per), dtype=torch.float64, device=DEV)
    kw = {}
    if alg == "polar":
        kw = dict(spare=torch.zeros(n_total, dtype=torch.float64, device=DEV),
                  has_spare=torch.zeros(n_total, dtype=torch.uint8, device=DEV))
    ck = torch.zeros(n_total, dtype=torch.int64, device=DEV)
    streams.fill_gaussians_streams(alg, source, st, out, checksum=ck, **kw)
    ids = [r["id"] for r in recs if r["id"] < n_total]
    rows = out[ids].cpu().numpy()
    sts = u64(st)
    cks = u64(ck)
    for k, r in enumerate([r for r in recs if r["id"] < n_total]):
        assert xor_hex(rows[k]) == r["xor"] and "%016x" % cks[r["id"]] == r["xor"]
        assert f64_to_hex(rows[k, :4]) == r["first"]
        assert "%016x" % int(sts.reshape(n_total, -1)[r["id"], 0]) == r["state"]
    return out, st, ck


def test_config2_full_size(golden):
    out, st, ck = _sampled("c2", golden, 1 << 20, 256, "polar", "lcg48")
    # every stream of a 64k-stream block against the oracle
    ref, ref_st, *_ = O.fill_gaussians("polar", "lcg48", O.config_states("c2", range(65536)), 256)
    assert bits_equal(out[:65536].cpu().numpy(), ref)
    assert np.array_equal(u64(st)[:65536], ref_st)


def test_config3_full_size(golden):
    out, st, ck = _sampled("c3", golden, 1 << 20, 1024, "modified-ziggurat", "splitmix")
    ids = np.random.default_rng(3).choice(1 << 20, 4096, replace=False)
    ref, *_ = O.fill_gaussians("modified-ziggurat", "splitmix", O.config_states("c3", ids), 1024)
    assert bits_equal(out[torch.from_numpy(ids).to(DEV)].cpu().numpy(), ref)


def test_config4_shards_and_moments(golden):
    """Config 4 on GPU 0's shard plus the sampled ids of other shards (seeded by
    first_id), per-stream checksums and the global moments of a block."""
    recs = golden["configs"]["c4"]
    for r in recs:
        st = streams.config_states("c4", r["id"], 1)
        out = torch.empty((1, 256), dtype=torch.float64, device=DEV)
        streams.fill_gaussians_streams("ziggurat", "lcg48", st, out)
        assert xor_hex(out.cpu().numpy()[0]) == r["xor"]
        assert "%016x" % int(u64(st)[0]) == r["state"]
    g = golden["configs"]["c4_moments_first4096"]
    st = streams.config_states("c4", 0, 4096)
    out = torch.empty((4096, 256), dtype=torch.float64, device=DEV)
    ps = torch.zeros((4096, 4), dtype=torch.float64, device=DEV)
    ck = torch.zeros(4096, dtype=torch.int64, device=DEV)
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, out, psum=ps, checksum=ck)
    assert sha(out.cpu().numpy()) == g["sha256"]
    assert "%016x" % streams.xor_fold(ck) == g["xor_all"]
    m = streams.moments_from_psum(ps, 256)
    assert m.n == g["n"]
    assert abs(m.mean - float.fromhex(g["mean"])) < 1e-12
    assert abs(m.variance / float.fromhex(g["variance"]) - 1) < 1e-11
    assert abs(m.skewness - float.fromhex(g["skewness"])) < 1e-9
    assert abs(m.excess_kurtosis - float.fromhex(g["excess_kurtosis"])) < 1e-9


def test_config5_mutation(golden):
    n_ind, n_genes = 65536, 1024
    x, sigma = streams.init_population(n_ind, n_genes, seed=2024, device=DEV)
    st = streams.config_states("c5", 0, n_ind)
    recs = golden["configs"]["c5"]
    ids = [r["id"] for r in recs]
    for r in recs:
        assert sha(x[r["id"]].cpu().numpy()) == r["x0_sha256"]
        assert float(sigma[r["id"]]) == float.fromhex(r["sigma"])
    for gen in range(3):
        streams.mutate(st, x, sigma, 1)
        for r in recs:
            gg = r["gens"][gen]
            assert sha(x[r["id"]].cpu().numpy()) == gg["sha256"], (r["id"], gen)
            assert "%016x" % int(u64(st)[r["id"], 0]) == gg["state"]
    # the same three generations fused in one launch
    x2, _ = streams.init_population(n_ind, n_genes, seed=2024, device=DEV)
    st2 = streams.config_states("c5", 0, n_ind)
    streams.mutate(st2, x2, sigma, 3)
    assert torch.equal(x2, x) and torch.equal(st2, st)
    del ids


@pytest.mark.parametrize("n,genes,gens,pad", [(100, 32, 3, 0), (2011, 48, 2, 0), (700, 64, 5, 2), (333, 1024, 2, 0),
                                              (97, 96, 3, 1), (64, 40, 2, 0), (40, 16, 4, 0),
                                              (2011, 192, 3, 0), (1000, 256, 2, 4), (40000, 192, 2, 0),
                                              (70, 400, 1, 2)])
def test_mutate_vs_oracle(n, genes, gens, pad, policy):
    """gz_mutate on both kernel families: rows of any length, strided (pad) and
    8-byte-aligned-only (odd ld) rows, several generations per launch."""
    st_np = O.config_states("c5", range(n))
    x_np = np.random.default_rng(genes).standard_normal((n, genes))
    sig_np = np.abs(np.random.default_rng(n).standard_normal(n))
    full = torch.zeros((n, genes + pad), dtype=torch.float64, device=DEV)
    full[:, :genes] = torch.from_numpy(x_np)
    x = full[:, :genes]
    st = dev_states("splitmix", st_np)
    streams.mutate(st, x, torch.from_numpy(sig_np).to(DEV), gens)
    xr = x_np.copy()
    ref_st, status = O.mutate(st_np, xr, sig_np, gens)
    assert status == 0
    assert bits_equal(x.cpu().numpy(), xr) and np.array_equal(u64(st), ref_st)
    assert (full[:, genes:] == 0).all()


def test_mutate_short_rows_loop_generations():
    n, genes = 100, 40  # rows shorter than a window: one launch per generation
    st_np = O.config_states("c5", range(n))
    x_np = np.random.default_rng(5).standard_normal((n, genes))
    sig_np = np.abs(np.random.default_rng(6).standard_normal(n))
    x = torch.from_numpy(x_np.copy()).to(DEV)
    st = dev_states("splitmix", st_np)
    streams.mutate(st, x, torch.from_numpy(sig_np).to(DEV), 4)
    xr = x_np.copy()
    ref_st, status = O.mutate(st_np, xr, sig_np, 4)
    assert status == 0
    assert bits_equal(x.cpu().numpy(), xr) and np.array_equal(u64(st), ref_st)


# ---- guards, libm, misc ---------------------------------------------------------

@pytest.mark.parametrize("alg,source,guard", [("polar", "lcg48", 1), ("polar", "splitmix", 2),
                                              ("ziggurat", "splitmix", 1), ("ziggurat", "lcg48", 1),
                                              ("modified-ziggurat", "splitmix", 1)])
def test_guard_status_matches_oracle(alg, source, guard, policy):
    n, n_per = 4096, 64
    cfg = "c2" if source == "lcg48" else "c3"
    st_np = O.config_states(cfg, range(n))
    *_, status = O.fill_gaussians(alg, source, st_np, n_per, guard=guard)
    st = dev_states(source, st_np)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    if status == 1:
        with pytest.raises(gz.RejectionLoopExceeded):
            streams.fill_gaussians_streams(alg, source, st, out, guard=guard)
    else:
        streams.fill_gaussians_streams(alg, source, st, out, guard=guard)
    # and with a guard that cannot trip, the same streams succeed
    st = dev_states(source, st_np)
    streams.fill_gaussians_streams(alg, source, st, out, guard=1000)


def test_guard_exact_for_each_stream(policy):
    """Per stream, the device trips the guard exactly when the oracle does."""
    n_per, guard = 16, 2
    for sid in range(64):
        st_np = O.config_states("c2", [sid])
        *_, status = O.fill_gaussians("polar", "lcg48", st_np, n_per, guard=guard)
        out = torch.empty((1, n_per), dtype=torch.float64, device=DEV)
        try:
            streams.fill_gaussians_streams("polar", "lcg48", dev_states("lcg48", st_np), out, guard=guard)
            got = 0
        except gz.RejectionLoopExceeded:
            got = 1
        assert got == status, sid


@pytest.mark.parametrize("alg,source", [("ziggurat", "splitmix"), ("ziggurat", "lcg48"),
                                        ("modified-ziggurat", "splitmix")])
@pytest.mark.parametrize("guard", [2, 3])
def test_zig_guard_counts_per_call(alg, source, guard, policy):
    """The ziggurat guard counts consecutive rejected attempts of ONE call
    (samplers.py:95-115): any accepted deviate, fast path included, resets it.
    Per stream, the device trips exactly when the oracle does, and the streams
    that do not trip match it bit for bit."""
    n, n_per = 96, 700
    cfg = "c4" if source == "lcg48" else "c1"
    st_np = O.config_states(cfg, range(n))
    trips = 0
    for sid in range(n):
        one = st_np[sid:sid + 1]
        ref, ref_st, *_, status = O.fill_gaussians(alg, source, one, n_per, guard=guard)
        out = torch.empty((1, n_per), dtype=torch.float64, device=DEV)
        st = dev_states(source, one)
        try:
            streams.fill_gaussians_streams(alg, source, st, out, guard=guard)
            got = 0
        except gz.RejectionLoopExceeded:
            got = 1
        assert got == status, (sid, got, status)
        trips += status
        if not status:
            assert bits_equal(out.cpu().numpy(), ref) and np.array_equal(u64(st).reshape(ref_st.shape), ref_st)
    if guard == 2:
        assert 0 < trips < n    # distinguishes per-call from cumulative counting


@pytest.mark.parametrize("fn", [0, 1])
def test_device_libm_bit_exact_sweep(fn):
    """The kernels' exp/log restatement equals the host glibc bit for bit."""
    import ctypes

    from paper_2405_19493_b200 import _lib

    L = _lib.load()
    xs = O.sweep_inputs(fn, 1 << 24, 11 + fn)
    d_in = torch.from_numpy(xs).to(DEV)
    d_out = torch.empty_like(d_in)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.gz_libm_eval_device(fn, ctypes.c_void_p(d_in.data_ptr()), ctypes.c_void_p(d_out.data_ptr()),
                                     xs.size, s))
    bad, first = O.libm_mismatches(fn, xs, d_out.cpu().numpy())
    assert bad == 0, f"{bad} mismatches, first input {xs[first]!r}"


def test_unit_affine_and_seeding_match_oracle():
    st = streams.config_states("c1", 5, 100)
    assert np.array_equal(u64(st), O.config_states("c1", range(5, 105)))
    st = streams.config_states("c2", 123, 50)
    assert np.array_equal(u64(st), O.config_states("c2", range(123, 173)))
    st = streams.config_states("c5", 7, 9)
    assert np.array_equal(u64(st), O.config_states("c5", range(7, 16)))
    x, sig = streams.init_population(4, 1024, seed=2024, first_ind=8191, total_ind=65536)
    u, _ = O.fill_u64("splitmix", np.array([[(2024 + 8191 * 1024 * O.GOLDEN_GAMMA) & O.MASK64, O.GOLDEN_GAMMA]],
                                           dtype=np.uint64), 4096)
    ref = -5.0 + 10.0 * ((u[0] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53)
    assert bits_equal(x.reshape(-1).cpu().numpy(), ref)


def test_zero_sizes(policy):
    st = streams.config_states("c2", 0, 8)
    out = torch.empty((8, 0), dtype=torch.float64, device=DEV)
    before = st.clone()
    sp = torch.full((8,), 0.5, dtype=torch.float64, device=DEV)
    hs = torch.ones(8, dtype=torch.uint8, device=DEV)
    streams.fill_gaussians_streams("polar", "lcg48", st, out, spare=sp, has_spare=hs)
    assert torch.equal(st, before) and (hs == 1).all() and (sp == 0.5).all()


@pytest.mark.parametrize("layers", [8, 64, 512, 1024])
@pytest.mark.parametrize("alg,source", [("ziggurat", "lcg48"), ("modified-ziggurat", "splitmix"),
                                        ("ziggurat", "splitmix")])
def test_custom_layer_counts(layers, alg, source, policy):
    n, n_per = 777, 300
    st_np = O.config_states("c4" if source == "lcg48" else "c3", range(1000, 1000 + n))
    smp = gz.make_sampler(alg, layers=layers)
    st = dev_states(source, st_np)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams(smp, source, st, out)
    ref, ref_st, *_ , status = O.fill_gaussians(alg, source, st_np, n_per, layers=layers)
    assert status == 0
    assert bits_equal(out.cpu().numpy(), ref)
    assert np.array_equal(u64(st), ref_st)


# ---- on-device verification statistics ---------------------

def test_device_chi_square_and_ks_match_reference(golden):
    from paper_2405_19493_b200 import verify as V

    g = golden["stats"]["gof_zig_lcg_424242"]
    out = torch.empty(300_000, dtype=torch.float64, device=DEV)
    engine.fill_gaussians(gz.make_sampler("ziggurat"), gz.make_source("lcg48", 424242), out)
    edges = V.equal_probability_edges(100)
    counts = V.histogram(out, edges)
    ref_counts = np.bincount(np.searchsorted(np.array(edges), out.cpu().numpy(), side="right"), minlength=len(edges) + 1)
    assert np.array_equal(counts, ref_counts)
    r = V.chi_square_gof(out, edges)
    assert r.dof == g["dof"]
    assert r.statistic == pytest.approx(float.fromhex(g["statistic"]), rel=1e-12)
    assert r.p_value == pytest.approx(float.fromhex(g["p_value"]), rel=1e-9)
    k = V.ks_test(out)
    assert k.n == g["n"]
    assert k.d_statistic == pytest.approx(float.fromhex(g["ks_d"]), abs=1e-14)


@pytest.mark.parametrize("source", ["lcg48", "splitmix"])
def test_device_low_bits_chi_square_matches_reference(source, golden):
    from paper_2405_19493_b200 import verify as V

    g = golden["stats"]["lowbits_" + source]
    r = V.low_bits_chi_square(gz.make_source(source, g["seed"]), g["k"], g["n"])
    assert r.dof == g["dof"]
    assert r.statistic == pytest.approx(float.fromhex(g["statistic"]), rel=1e-12)


# ---- benchmark harness with the reference's schema -------------

@pytest.mark.parametrize("source,alg", [p for p in PAIRINGS if p != ("lcg48", "modified-ziggurat")])
def test_benchmark_witness_equals_reference_checksum(source, alg, golden):
    from paper_2405_19493_b200 import benchmark as B

    cfg = B.BenchConfig.smoke(seed=60)
    r = B.run_benchmark(alg, source, cfg)
    assert "%016x" % r.checksum == golden["bench_witness"]["%s/%s/60" % (source, alg)]
    assert r.ns_per_op > 0 and len(r.per_iteration_ns_per_op) == cfg.measure_iters
    assert r.engine_used == "cuda"
    text = B.render_table([r], "md")
    assert text.startswith("| PRNG |") and source in text


def test_benchmark_refuses_unsanctioned_pairing():
    from paper_2405_19493_b200 import benchmark as B

    with pytest.raises(gz.UnsanctionedPairing):
        B.run_benchmark("modified-ziggurat", "lcg48", B.BenchConfig.smoke())


@pytest.mark.parametrize("layers", [8, 128, 256, 1024])
def test_wedge_prefilter_error_budget(layers):
    """The float/__expf wedge pre-filters fall back to the exact glibc exp within
    2^-15 of the accept boundary; their measured errors must stay below 2^-17."""
    from paper_2405_19493_b200 import _lib
    from paper_2405_19493_b200.engine import table_slot
    from paper_2405_19493_b200.samplers import _default_tables

    L = _lib.load()
    slot = table_slot(_default_tables(layers))
    out = torch.zeros(3, dtype=torch.float64, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.gz_wedge_filter_error(slot, 1 << 24, 12345 + layers, ctypes.c_void_p(out.data_ptr()), s))
    _lib.check(L.gz_stream_check(s))
    ey, ef, ex = out.cpu().tolist()
    assert 0 < ey < 2.0 ** -20
    assert 0 < ef < 2.0 ** -17
    assert 0 < ex < 2.0 ** -17


def test_branch_free_divide_and_sqrt_are_correctly_rounded():
    """The polar drains' divide/sqrt without special-case branches equal div.rn /
    sqrt.rn bit for bit over 2^28 samples of the polar operand domain."""
    from paper_2405_19493_b200 import _lib

    L = _lib.load()
    out = torch.zeros(2, dtype=torch.int64, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.gz_polar_ops_selftest(1 << 28, 20240531, ctypes.c_void_p(out.data_ptr()), s))
    _lib.check(L.gz_stream_check(s))
    assert out.cpu().tolist() == [0, 0]


@pytest.mark.parametrize("source,alg", PAIRINGS)
@pytest.mark.parametrize("n", [32768, 32769, 100001, (1 << 20) + 3])
def test_single_long_stream_vs_oracle(source, alg, n):
    """One stream, many deviates: the whole-GPU decode (gz_single.cuh) equals the
    sequential reference loop, incl. polar spares in and out and the final state."""
    rng = np.random.default_rng(zlib.crc32(f"single/{source}/{alg}/{n}".encode()))
    if source == "lcg48":
        st_np = rng.integers(0, 2 ** 48, size=1, dtype=np.uint64)
    else:
        st_np = rng.integers(0, 2 ** 63, size=(1, 2), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    kw, sp, hs = {}, None, None
    if alg == "polar":
        has = 1 if n in (32768, 100001) else 0     # spare in with an odd and an even remainder
        hs = np.array([has], dtype=np.uint8)
        sp = np.array([0.25 * has])
        kw = dict(spare=torch.from_numpy(sp.copy()).to(DEV), has_spare=torch.from_numpy(hs.copy()).to(DEV))
    st = dev_states(source, st_np)
    out = torch.empty((1, n), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams(alg, source, st, out, **kw)
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians(alg, source, st_np, n, *((sp, hs) if alg == "polar" else (None, None)))
    assert status == 0
    got = out.cpu().numpy()
    bad = np.nonzero(got.view(np.uint64) != ref.view(np.uint64))[1]
    assert bad.size == 0, f"{bad.size} deviates differ, first at {bad[:5]}"
    assert np.array_equal(u64(st).reshape(ref_st.shape), ref_st)
    if alg == "polar":
        assert np.array_equal(kw["has_spare"].cpu().numpy(), ref_has)
        if ref_has[0]:
            assert bits_equal(kw["spare"].cpu().numpy(), ref_sp)


def test_single_long_stream_matches_warp_kernel():
    """The same call through the warp-per-stream kernel (policy 'warp' disables the
    whole-GPU decode) gives the same bits."""
    for source, alg in PAIRINGS:
        src = gz.make_source(source, 99)
        a = torch.empty(200_000, dtype=torch.float64, device=DEV)
        engine.fill_gaussians(gz.make_sampler(alg), src, a)
        s_a = src.state
        streams.set_kernel_policy("warp")
        try:
            src = gz.make_source(source, 99)
            b = torch.empty(200_000, dtype=torch.float64, device=DEV)
            engine.fill_gaussians(gz.make_sampler(alg), src, b)
        finally:
            streams.set_kernel_policy("auto")
        assert torch.equal(a, b) and src.state == s_a, (source, alg)


@pytest.mark.parametrize("source,alg", [("lcg48", "polar"), ("splitmix", "ziggurat")])
def test_large_numpy_output_staged_copy(source, alg):
    """numpy outputs above 8 MiB go through the pinned staging pieces: same bits as a
    device-tensor fill of the same stream, and a non-multiple of the piece size."""
    n = (5 << 20) + 12345          # 40+ MiB: two 32 MiB pieces plus a tail
    a = np.empty(n)
    src_a = gz.make_source(source, 31337)
    engine.fill_gaussians(gz.make_sampler(alg), src_a, a)
    b = torch.empty(n, dtype=torch.float64, device=DEV)
    src_b = gz.make_source(source, 31337)
    engine.fill_gaussians(gz.make_sampler(alg), src_b, b)
    assert bits_equal(a, b.cpu().numpy()) and src_a.state == src_b.state
    ref, ref_st, *_ = O.fill_gaussians(alg, source, np.array([[src_a.state, 0]], dtype=np.uint64)[:, :1]
                                       if source == "lcg48" else np.array([[src_a.state, src_a.gamma]], dtype=np.uint64), 1000)
    c = np.empty(1000)
    engine.fill_gaussians(gz.make_sampler(alg), src_a, c)
    assert bits_equal(c, ref[0])


@pytest.mark.parametrize("source", ["lcg48", "splitmix"])
@pytest.mark.parametrize("n", [32768, 1_000_003])
def test_fill_u64_single_long_stream(source, n):
    """engine.fill_u64 on one source: a thread per draw (gz_single.cuh) == the oracle."""
    st_np = (np.array([[123456789]], dtype=np.uint64) if source == "lcg48"
             else np.array([[987654321, O.GOLDEN_GAMMA]], dtype=np.uint64))
    src = gz.make_source(source, 0)
    src.state = int(st_np[0, 0])
    out = torch.empty(n, dtype=torch.int64, device=DEV)
    engine.fill_u64(src, out)
    ref, ref_st = O.fill_u64(source, st_np[:, 0] if source == "lcg48" else st_np, n)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref[0])
    assert src.state == int(ref_st.reshape(-1)[0])


@pytest.mark.parametrize("n", [40001, 65536, 65537])
def test_polar_single_stream_host_path_with_spare(n):
    """numpy output, cached spare in and out, one long stream (gz_fill_gaussians_host ->
    the whole-GPU decode) against the per-call oracle semantics."""
    smp = gz.make_sampler("polar")
    src = gz.make_source("lcg48", 2024)
    smp.spare = -0.75
    buf = np.empty(n)
    engine.fill_gaussians(smp, src, buf)
    st0 = np.array([gz.make_source("lcg48", 2024).state], dtype=np.uint64)
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians("polar", "lcg48", st0, n, np.array([-0.75]),
                                                             np.array([1], dtype=np.uint8))
    assert status == 0 and bits_equal(buf, ref[0])
    assert src.state == int(ref_st[0])
    assert (smp.spare is not None) == bool(ref_has[0])
    if ref_has[0]:
        assert bits_equal(np.array([smp.spare]), ref_sp)


def test_single_stream_segments_hand_over():
    """The single-stream decode in many small segments (GZ_SINGLE_SEG) gives the same
    bits: each segment starts at the previous one's next attempt boundary."""
    import subprocess
    import sys

    code = r"""
import numpy as np, torch
import paper_2405_19493_b200 as gz
from paper_2405_19493_b200 import engine
res = []
for source, alg in (("lcg48", "polar"), ("splitmix", "ziggurat"), ("lcg48", "modified-ziggurat")):
    out = torch.empty(300001, dtype=torch.float64, device="cuda")
    src = gz.make_source(source, 77)
    engine.fill_gaussians(gz.make_sampler(alg), src, out)
    res.append((out.cpu().numpy().view(np.uint64).tobytes().hex()[:64], int(np.bitwise_xor.reduce(out.cpu().numpy().view(np.uint64))), src.state))
print(repr(res))
"""
    import os

    env = dict(os.environ)
    outs = []
    for seg in ("", "40000"):
        env["GZ_SINGLE_SEG"] = seg
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("source", ["lcg48", "splitmix"])
def test_tail_sample_matches_oracle(source):
    for seed in range(20):
        src = gz.make_source(source, seed)
        st = engine._state_words(src)
        r = 3.4426198558966377 if seed % 2 else 0.5
        v = gz.tail_sample(src, r)
        rv, rst, status = O.tail_sample(source, st, r)
        assert status == 0 and v == rv and src.state == int(rst[0])
    with pytest.raises(ValueError):
        gz.tail_sample(gz.make_source(source, 1), 0.0)


def test_abi_rejects_bad_arguments_and_recovers():
    """Every invalid call returns GZ_ERR_INVALID (2) with a message and launches
    nothing; the next valid call works (no sticky error state)."""
    from paper_2405_19493_b200 import _lib

    L = _lib.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    st = torch.zeros(8, 2, dtype=torch.int64, device=DEV)
    out = torch.zeros(8, 16, dtype=torch.float64, device=DEV)
    x = torch.zeros(8, 16, dtype=torch.float64, device=DEV)
    sig = torch.ones(8, dtype=torch.float64, device=DEV)
    sp = torch.zeros(8, dtype=torch.float64, device=DEV)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    slot = engine.table_slot(gz.make_sampler("ziggurat").tables)
    G = 1_000_000

    def fill(alg=1, src=1, sl=slot, n=8, n_per=16, ld=16, si=True, so=True, o=True, spi=None, hi=None, guard=G):
        return L.gz_fill_gaussians(alg, src, sl, n, n_per, ld, P(st) if si else None, P(st) if so else None,
                                   spi, hi, None, None, P(out) if o else None, None, None, guard, s)

    bad = {
        "alg": fill(alg=3), "alg-neg": fill(alg=-1), "src": fill(src=2), "n": fill(n=-1), "n_per": fill(n_per=-1),
        "ld": fill(ld=15), "guard": fill(guard=0), "state_in": fill(si=False), "state_out": fill(so=False),
        "out": fill(o=False), "slot": fill(sl=63), "slot-neg": fill(sl=-1),
        "spare-without-flag": fill(alg=0, spi=P(sp)),
        "polar-row-limit": fill(alg=0, n=1, n_per=1 << 30, ld=1 << 30),
        "u64-src": L.gz_fill_u64(5, 8, 16, 16, P(st), P(st), P(out), s),
        "u64-ld": L.gz_fill_u64(1, 8, 16, 8, P(st), P(st), P(out), s),
        "mutate-slot": L.gz_mutate(63, 8, 16, 16, P(st), P(st), P(x), P(sig), 1, G, s),
        "mutate-ld": L.gz_mutate(slot, 8, 16, 8, P(st), P(st), P(x), P(sig), 1, G, s),
        "mutate-gens": L.gz_mutate(slot, 8, 16, 16, P(st), P(st), P(x), P(sig), -1, G, s),
        "seed-scheme": L.gz_seed_streams(99, 1, 0, 8, P(st), s),
    }
    for name, status in bad.items():
        assert status == 2, (name, status)
        assert L.gz_last_error().decode(), name
    assert (out == 0).all() and (x == 0).all()
    # nothing sticky: a valid call right after succeeds and matches the oracle
    st_np = O.config_states("c1", range(8))
    st.copy_(torch.from_numpy(st_np.view(np.int64)))
    assert fill() == 0
    _lib.check(L.gz_stream_check(s))
    ref, *_ = O.fill_gaussians("ziggurat", "splitmix", st_np, 16)
    assert bits_equal(out.cpu().numpy(), ref)
    # n_streams == 0 and n_per == 0 are valid no-ops
    assert fill(n=0) == 0 and fill(n_per=0, ld=0) == 0


@pytest.mark.parametrize("source,alg", [("splitmix", "ziggurat"), ("lcg48", "ziggurat"),
                                        ("splitmix", "modified-ziggurat"), ("lcg48", "modified-ziggurat")])
@pytest.mark.parametrize("pos", ["0", "1"])
def test_few_long_streams_segmented_vs_oracle(source, alg, pos, monkeypatch):
    """Fewer streams than the GPU holds warps: G warps per stream decode speculative
    segments (gz_k_seg.cuh; pos=1: the position decode, gz_k_pos.cuh) -- values and final
    states equal the oracle's for row lengths around the segment sizes and stream counts
    up to one wave."""
    monkeypatch.setenv("GZ_POS", pos)
    for n, n_per in ((1, 512), (1, 20000), (2, 700), (7, 4096), (300, 513), (1024, 4096), (1100, 600)):
        rng = np.random.default_rng(zlib.crc32(f"seg/{source}/{alg}/{n}/{n_per}".encode()))
        if source == "lcg48":
            st_np = rng.integers(0, 2 ** 48, size=n, dtype=np.uint64)
        else:
            st_np = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) | np.uint64(1)
        st = dev_states(source, st_np)
        out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
        streams.fill_gaussians_streams(alg, source, st, out)
        ref, ref_st, *_ = O.fill_gaussians(alg, source, st_np, n_per)
        assert bits_equal(out.cpu().numpy(), ref), (n, n_per)
        assert np.array_equal(u64(st).reshape(ref_st.shape), ref_st), (n, n_per)


@pytest.mark.parametrize("knob", ["GZ_SEG_GUESS=1", "GZ_SEG_FALLBACK=1", "GZ_POS=1", "GZ_POS=1,GZ_POS_FALLBACK=1",
                                  "GZ_POS=1,GZ_POS_SERIAL=1", "GZ_SEG=0"])
def test_segmented_redecode_and_fallback_paths(knob):
    """The rare paths of the few-long-streams decodes, forced: the speculative segment
    decode (k_zig_lseg, the default) with every segment re-decoded from its true entry
    (wrong guesses) or every stream handed to the exact warp loop; the position decode
    (k_zig_pos, GZ_POS=1) as it runs, handing every stream to the exact loop, or parsing
    every chunk sequentially; and both paths disabled -- all give the default run's bits."""
    import os
    import subprocess
    import sys

    code = r"""
import numpy as np, torch
from paper_2405_19493_b200 import streams
res = []
for source, alg in (("splitmix", "ziggurat"), ("lcg48", "modified-ziggurat")):
    st = streams.config_states("c1" if source == "splitmix" else "c4", 0, 500)
    out = torch.empty((500, 3000), dtype=torch.float64, device="cuda")
    streams.fill_gaussians_streams(alg, source, st, out)
    v = out.cpu().numpy().view(np.uint64)
    res.append((int(np.bitwise_xor.reduce(v.ravel())), v[:, -1].tobytes().hex()[:48], st.cpu().numpy().tobytes().hex()[:64]))
print(repr(res))
"""
    outs = []
    for env_kv in ("", knob):
        env = dict(os.environ)
        for k in ("GZ_SEG", "GZ_SEG_GUESS", "GZ_SEG_FALLBACK", "GZ_POS", "GZ_POS_FALLBACK", "GZ_POS_SERIAL"):
            env.pop(k, None)
        for kv in filter(None, env_kv.split(",")):
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1]


@pytest.mark.parametrize("source,alg", [("splitmix", "ziggurat"), ("lcg48", "ziggurat"),
                                        ("splitmix", "modified-ziggurat"), ("lcg48", "modified-ziggurat")])
def test_position_decode_many_passes_and_strides(source, alg, monkeypatch):
    """k_zig_pos over rows of many passes (2176 positions per full pass; the last pass
    sized to the remaining deviates), row lengths around the pass sizes, strided rows
    (ld > n_per, the padding left untouched), and a second call continuing the states."""
    monkeypatch.setenv("GZ_POS", "1")
    for n, n_per, pad in ((3, 100003, 0), (64, 2093, 5), (129, 2300, 1), (40, 4352, 0), (5, 65536, 3)):
        rng = np.random.default_rng(zlib.crc32(f"pos/{source}/{alg}/{n}/{n_per}".encode()))
        if source == "lcg48":
            st_np = rng.integers(0, 2 ** 48, size=n, dtype=np.uint64)
        else:
            st_np = rng.integers(0, 2 ** 63, size=(n, 2), dtype=np.uint64) | np.uint64(1)
        st = dev_states(source, st_np)
        full = torch.full((n, n_per + pad), 7.0, dtype=torch.float64, device=DEV)
        out = full[:, :n_per]
        ref_st = st_np
        for call in range(2):
            streams.fill_gaussians_streams(alg, source, st, out)
            ref, ref_st, *_ = O.fill_gaussians(alg, source, ref_st, n_per)
            assert bits_equal(out.cpu().numpy(), ref), (n, n_per, call)
            assert np.array_equal(u64(st).reshape(ref_st.shape), ref_st), (n, n_per, call)
        if pad:
            assert (full[:, n_per:] == 7.0).all()


@pytest.mark.parametrize("guard", [1, 2, 3, 5, 40])
def test_position_decode_small_guards(guard, monkeypatch):
    """Guard trips under the position decode: the parse counts consecutive rejections
    across passes and hands a tripping stream to the exact loop, which raises the
    status; the status and the streams that do not trip equal the oracle's."""
    monkeypatch.setenv("GZ_POS", "1")
    n, n_per = 200, 3000
    for source, alg in (("splitmix", "ziggurat"), ("lcg48", "modified-ziggurat")):
        st_np = O.config_states("c1" if source == "splitmix" else "c4", range(n))
        st = dev_states(source, st_np)
        out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
        ref, ref_st, _, _, status = O.fill_gaussians(alg, source, st_np, n_per, guard=guard)
        try:
            streams.fill_gaussians_streams(alg, source, st, out, guard=guard)
            got = 0
        except gz.RejectionLoopExceeded:
            got = 1
        assert got == status, (source, alg, guard)
        if status == 0:
            assert bits_equal(out.cpu().numpy(), ref)
            assert np.array_equal(u64(st).reshape(ref_st.shape), ref_st)


# ---- maximum sizes: one launch of more than 2^32 output elements ---------------

@pytest.mark.parametrize("alg,source", [("polar", "lcg48"), ("ziggurat", "lcg48"),
                                        ("modified-ziggurat", "splitmix")])
def test_output_beyond_2p32_elements(alg, source):
    """2^24 + 5 streams x 257 deviates (4.3e9 elements, 34.5 GB) in one call: the rows
    whose element offsets straddle 2^31 and 2^32, and the first and last rows, equal
    the oracle bit for bit (states and polar spares included); the whole output equals
    a second kernel's (polar: the fused-witness kernel; ziggurats: the warp-per-stream
    kernel) bit for bit."""
    n, n_per = (1 << 24) + 5, 257
    need = 2 * n * n_per * 8 + (1 << 30)
    if torch.cuda.mem_get_info()[0] < need:
        pytest.skip("needs ~70 GB of free device memory")
    rng = np.random.default_rng(2032)
    st_np = rng.integers(0, 2 ** 63, size=(n, 1 if source == "lcg48" else 2), dtype=np.uint64)
    if source == "lcg48":
        st_np = (st_np[:, 0] & np.uint64((1 << 48) - 1)).copy()
    else:
        st_np[:, 1] |= np.uint64(1)              # odd gammas
    rows = sorted({0, 1, 2, n - 2, n - 1,
                   (1 << 31) // n_per - 1, (1 << 31) // n_per, (1 << 31) // n_per + 1,
                   (1 << 32) // n_per - 1, (1 << 32) // n_per, (1 << 32) // n_per + 1})
    kw = {}
    if alg == "polar":
        kw = dict(spare=torch.zeros(n, dtype=torch.float64, device=DEV),
                  has_spare=torch.zeros(n, dtype=torch.uint8, device=DEV))
    st = dev_states(source, st_np)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams(alg, source, st, out, **kw)
    ref, ref_st, ref_sp, ref_has, status = O.fill_gaussians(alg, source, st_np[rows], n_per)
    assert status == 0
    idx = torch.tensor(rows, device=DEV)
    assert bits_equal(out[idx].cpu().numpy(), ref)
    assert np.array_equal(u64(st).reshape(n, -1)[rows], ref_st.reshape(len(rows), -1))
    if alg == "polar":
        assert np.array_equal(kw["has_spare"][idx].cpu().numpy(), ref_has)
        assert bits_equal(kw["spare"][idx].cpu().numpy(), ref_sp)
    # the same launch through a second kernel, compared over all 4.3e9 elements
    out2 = torch.empty_like(out)
    st2 = dev_states(source, st_np)
    if alg == "polar":
        ck = torch.zeros(n, dtype=torch.int64, device=DEV)
        streams.fill_gaussians_streams(alg, source, st2, out2, checksum=ck,
                                       spare=torch.zeros(n, dtype=torch.float64, device=DEV),
                                       has_spare=torch.zeros(n, dtype=torch.uint8, device=DEV))
    else:
        streams.set_kernel_policy("warp")
        try:
            streams.fill_gaussians_streams(alg, source, st2, out2)
        finally:
            streams.set_kernel_policy("auto")
    assert torch.equal(out.view(torch.int64), out2.view(torch.int64))
    assert torch.equal(st, st2)
