"""Full-size parity: EVERY stream of configs 2, 3 and 4 (GPU shards 0 and 7) and
all 65 536 individuals of config 5 over all 100 generations, bit for bit
against the CPU oracle (oracle/gz_oracle.c, pinned to the reference by
tests/golden/).  Needs a B200: `pytest -m gpu`.

The oracle runs in digest mode (gzo_fill_digest: the reference's per-stream
loop, engine.py:235-270, folding each deviate into order-sensitive per-stream
witnesses instead of storing 8 GiB); the device output is digested the same way
on the GPU.  Each test prints the oracle's wall time (run with -s to see it).
"""
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from oracle import gz_oracle as O  # noqa: E402
from paper_2405_19493_b200 import streams  # noqa: E402

DEV = "cuda"


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def device_digest(out, chunk=1 << 18):
    """O.digest_rows of a CUDA [n, n_per] float64 tensor, computed on the GPU:
    (xor, sum (j+1)*(bits>>32), sum (j+1)*(bits & 0xffffffff)) per row, mod 2^64."""
    n, n_per = out.shape
    w = torch.arange(1, n_per + 1, dtype=torch.int64, device=out.device)
    res = torch.empty((n, 3), dtype=torch.int64, device=out.device)
    for a in range(0, n, chunk):
        b = out[a:a + chunk].contiguous().view(torch.int64)
        x = b
        while x.shape[1] > 1:
            if x.shape[1] & 1:
                x = torch.cat([x, torch.zeros_like(x[:, :1])], 1)
            h = x.shape[1] // 2
            x = x[:, :h] ^ x[:, h:]
        res[a:a + chunk, 0] = x[:, 0] if n_per else 0
        res[a:a + chunk, 1] = (((b >> 32) & 0xffffffff) * w).sum(1)
        res[a:a + chunk, 2] = ((b & 0xffffffff) * w).sum(1)
        del b, x
    return res.cpu().numpy().view(np.uint64)


def oracle_digest(alg, source, cfg, first, count, n_per, psum=False):
    t0 = time.perf_counter()
    st = O.config_states_range(cfg, first, count)
    dig, st_out, sp, hs, ps, status = O.fill_digest(alg, source, st, n_per, psum=psum)
    dt = time.perf_counter() - t0
    assert status == 0
    print(f"\n[oracle] {cfg} ids [{first}, {first + count}) x {n_per}: {dt:.2f} s "
          f"({count * n_per / dt / 1e9:.2f} G variates/s)")
    return dig, st_out, sp, hs, ps


def test_config2_every_stream():
    """Polar x LCG48, 2^20 streams x 256 (BASELINE configs[1]), all streams."""
    n, n_per = 1 << 20, 256
    st = streams.config_states("c2", 0, n)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    sp = torch.zeros(n, dtype=torch.float64, device=DEV)
    hs = torch.zeros(n, dtype=torch.uint8, device=DEV)
    streams.fill_gaussians_streams("polar", "lcg48", st, out, spare=sp, has_spare=hs)
    got = device_digest(out)
    del out
    dig, st_ref, sp_ref, hs_ref, _ = oracle_digest("polar", "lcg48", "c2", 0, n, n_per)
    bad = np.nonzero((got != dig).any(1))[0]
    assert bad.size == 0, f"{bad.size} streams differ, first {bad[:8]}"
    assert np.array_equal(u64(st), st_ref)
    assert np.array_equal(hs.cpu().numpy(), hs_ref)
    assert np.array_equal(sp.cpu().numpy().view(np.uint64), sp_ref.view(np.uint64))


def test_config2_odd_rows_carry_spares():
    """Config 2 streams with 255 deviates per row (every stream ends holding a
    spare) and a second call that starts from those spares."""
    n, n_per = 1 << 18, 255
    st = streams.config_states("c2", 0, n)
    sp = torch.zeros(n, dtype=torch.float64, device=DEV)
    hs = torch.zeros(n, dtype=torch.uint8, device=DEV)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    st_np = O.config_states_range("c2", 0, n)
    sp_np, hs_np = np.zeros(n), np.zeros(n, dtype=np.uint8)
    for _ in range(2):
        streams.fill_gaussians_streams("polar", "lcg48", st, out, spare=sp, has_spare=hs)
        dig, st_np, sp_np, hs_np, _, status = O.fill_digest("polar", "lcg48", st_np, n_per, spare=sp_np, has=hs_np)
        assert status == 0
        assert np.array_equal(device_digest(out), dig)
        assert np.array_equal(u64(st), st_np)
        assert np.array_equal(hs.cpu().numpy(), hs_np)
        assert np.array_equal(sp.cpu().numpy().view(np.uint64), sp_np.view(np.uint64))


def test_config3_every_stream():
    """Modified ziggurat x SplitMix64, 2^20 streams x 1024 (box-wide), all streams."""
    n, n_per = 1 << 20, 1024
    st = streams.config_states("c3", 0, n)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams("modified-ziggurat", "splitmix", st, out)
    got = device_digest(out)
    del out
    dig, st_ref, *_ = oracle_digest("modified-ziggurat", "splitmix", "c3", 0, n, n_per)
    bad = np.nonzero((got != dig).any(1))[0]
    assert bad.size == 0, f"{bad.size} streams differ, first {bad[:8]}"
    assert np.array_equal(u64(st), st_ref)


@pytest.mark.parametrize("shard", [0, 7])
def test_config4_every_stream_of_shard(shard):
    """Ziggurat x LCG48, GPU `shard`'s 2^22 streams x 256 with the fused per-stream
    checksums and power sums on (the bench headline launch), all streams."""
    n, n_per = 1 << 22, 256
    first = shard * n
    st = streams.config_states("c4", first, n)
    out = torch.empty((n, n_per), dtype=torch.float64, device=DEV)
    ck = torch.zeros(n, dtype=torch.int64, device=DEV)
    ps = torch.zeros((n, 4), dtype=torch.float64, device=DEV)
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, out, checksum=ck, psum=ps)
    got = device_digest(out)
    del out
    dig, st_ref, _, _, ps_ref = oracle_digest("ziggurat", "lcg48", "c4", first, n, n_per, psum=True)
    bad = np.nonzero((got != dig).any(1))[0]
    assert bad.size == 0, f"{bad.size} streams differ, first {bad[:8]}"
    assert np.array_equal(u64(ck), dig[:, 0]), "fused checksums differ"
    assert np.array_equal(ps.cpu().numpy().view(np.uint64), ps_ref.view(np.uint64)), "fused power sums differ"
    assert np.array_equal(u64(st), st_ref)


def test_config5_all_individuals_100_generations():
    """Fused mutation, 65 536 individuals x 1024 genes, all 100 generations (one
    launch of 100 generations, and 10 launches of 10), against the oracle."""
    n_ind, n_genes, gens = 65536, 1024, 100
    x, sigma = streams.init_population(n_ind, n_genes, seed=2024, device=DEV)
    x_np = x.cpu().numpy().copy()
    sig_np = sigma.cpu().numpy().copy()
    st = streams.config_states("c5", 0, n_ind)
    x2 = x.clone()
    st2 = st.clone()
    streams.mutate(st, x, sigma, gens)
    for _ in range(gens // 10):
        streams.mutate(st2, x2, sigma, 10)
    assert torch.equal(x, x2) and torch.equal(st, st2)
    t0 = time.perf_counter()
    st_ref, status = O.mutate(O.config_states_range("c5", 0, n_ind), x_np, sig_np, gens)
    dt = time.perf_counter() - t0
    print(f"\n[oracle] c5 65536 x 1024 x {gens} generations: {dt:.2f} s "
          f"({n_ind * n_genes * gens / dt / 1e9:.2f} G updates/s)")
    assert status == 0
    got = x.cpu().numpy()
    bad = np.nonzero((got.view(np.uint64) != x_np.view(np.uint64)).any(1))[0]
    assert bad.size == 0, f"{bad.size} individuals differ, first {bad[:8]}"
    assert np.array_equal(u64(st), st_ref)
