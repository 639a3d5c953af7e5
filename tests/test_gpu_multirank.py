"""The N>1 path through the real device fill: two processes share cuda:0 (the
box has one GPU for tests), each generating its contiguous shard of a config-4
block with the CUDA engine (fused per-stream checksums and power sums), then
merging the per-rank moments and xor with paper_2405_19493_b200.dist over gloo.
The ranks' kernels never wait on one another (the generation path has no
collective), so sharing one GPU changes nothing but the timing.  The merged
witnesses, per-stream checksums and final states must equal a single process
filling the whole block.  Needs a B200: `pytest -m gpu`.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

N_STREAMS, N_PER = 1 << 20, 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2405_19493_b200 import dist as gzdist
    from paper_2405_19493_b200 import streams

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    first, count = gzdist.shard(N_STREAMS, world, rank)
    st = streams.config_states("c4", first, count)
    o = torch.empty((count, N_PER), dtype=torch.float64, device="cuda")
    ck = torch.zeros(count, dtype=torch.int64, device="cuda")
    ps = torch.zeros((count, 4), dtype=torch.float64, device="cuda")
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, o, checksum=ck, psum=ps)
    cen = streams.central_from_psum(ps, N_PER)
    merged = gzdist.gather_moments(cen)
    gx = gzdist.gather_xor(streams.xor_fold(ck))
    out[rank] = (merged, gx, first, count, ck.cpu().numpy().copy(), st.cpu().numpy().copy())
    dist.destroy_process_group()


def test_two_processes_on_device_equal_one():
    import torch.multiprocessing as mp

    from paper_2405_19493_b200 import streams

    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")

    st = streams.config_states("c4", 0, N_STREAMS)
    o = torch.empty((N_STREAMS, N_PER), dtype=torch.float64, device="cuda")
    ck = torch.zeros(N_STREAMS, dtype=torch.int64, device="cuda")
    ps = torch.zeros((N_STREAMS, 4), dtype=torch.float64, device="cuda")
    streams.fill_gaussians_streams("ziggurat", "lcg48", st, o, checksum=ck, psum=ps)
    ref = streams.central_from_psum(ps, N_PER).cpu().tolist()
    ref_x = streams.xor_fold(ck)
    ck_np, st_np = ck.cpu().numpy(), st.cpu().numpy()
    for rank in (0, 1):
        merged, gx, first, count, rck, rst = out[rank]
        assert gx == ref_x
        assert merged[0] == ref[0]
        assert merged[1] == pytest.approx(ref[1], abs=1e-15)
        for k in (2, 3, 4):
            assert merged[k] == pytest.approx(ref[k], rel=1e-11)
        assert np.array_equal(rck, ck_np[first:first + count])
        assert np.array_equal(rst, st_np[first:first + count])
    m = streams.summarize(*out[0][0])
    assert m.n == N_STREAMS * N_PER
    assert abs(m.mean) < 1e-3 and abs(m.variance - 1) < 1e-3 and abs(m.excess_kurtosis) < 1e-2
