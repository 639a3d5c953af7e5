"""The N>1 path on CPU: two gloo ranks each compute their shard of a config-4
block (with the CPU oracle standing in for the device fill), then merge the
per-rank moments and xor checksums with paper_2405_19493_b200.dist; the result
must equal the single-process computation over the whole block."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import gz_oracle as O

N_STREAMS, N_PER = 512, 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _central(x):
    n = x.size
    mean = float(np.mean(x))
    d = x - mean
    return (float(n), mean, float(np.sum(d ** 2)), float(np.sum(d ** 3)), float(np.sum(d ** 4)))


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2405_19493_b200 import dist as gzdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = gzdist.shard(N_STREAMS, world, rank)
    vals, *_ = O.fill_gaussians("ziggurat", "lcg48", O.config_states("c4", range(first, first + count)), N_PER)
    xr = 0
    for row in vals:
        xr ^= O.checksum(row)
    merged = gzdist.gather_moments(_central(vals.reshape(-1)))
    gx = gzdist.gather_xor(xr)
    out[rank] = (merged, gx, first, count)
    dist.destroy_process_group()


def test_shards_cover_all_ids():
    from paper_2405_19493_b200 import dist as gzdist

    for world in (1, 2, 3, 8):
        got = []
        for r in range(world):
            f, c = gzdist.shard(1000, world, r)
            got.extend(range(f, f + c))
        assert got == list(range(1000))


def test_two_rank_merge_equals_single_process():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    vals, *_ = O.fill_gaussians("ziggurat", "lcg48", O.config_states("c4", range(N_STREAMS)), N_PER)
    ref = _central(vals.reshape(-1))
    xr = O.checksum(vals)
    for rank in (0, 1):
        merged, gx, *_ = out[rank]
        assert gx == xr
        assert merged[0] == ref[0]
        assert merged[1] == pytest.approx(ref[1], abs=1e-15)
        for k in (2, 3, 4):
            assert merged[k] == pytest.approx(ref[k], rel=1e-10, abs=1e-9)
    # the merged moments also match the reference's one-pass statistics
    n, mean, var, skew, kurt = O.moments_summary(O.moments_accumulate(vals))
    from paper_2405_19493_b200.streams import summarize

    m = summarize(*out[0][0])
    assert m.n == n and m.mean == pytest.approx(mean, abs=1e-12)
    assert m.variance == pytest.approx(var, rel=1e-12)
    assert m.excess_kurtosis == pytest.approx(kurt, abs=1e-9)
