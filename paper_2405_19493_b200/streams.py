"""Many independent streams at once -- the B200 hot path.

`fill_gaussians_streams` generates a [n_streams, n_per] float64 CUDA tensor
whose row s equals what the reference's engine.fill_gaussians
(engine.py:235-270) writes for stream s, with per-stream state in/out on the
device.  Stream state tensors use torch.int64 as 64-bit containers (bit
patterns): shape [n] for lcg48, [n, 2] = {state, gamma} for splitmix.

Also here: device seeding for the five BASELINE configs, the fused config-5
mutation and the per-stream checksum / moment reductions of config 4.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import DEFAULT_GUARD, check
from .samplers import GaussianSampler, make_sampler
from .sources import GOLDEN_GAMMA, MASK64, SplitMix64

__all__ = ["fill_gaussians_streams", "fill_u64_streams", "seed_streams", "config_states", "mutate",
           "init_population", "moments_from_psum", "xor_fold", "MomentSummary", "CONFIGS"]


def _torch():
    import torch

    return torch


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(device, stream=None):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _source_id(source) -> str:
    return source if isinstance(source, str) else source.source_id


def fill_gaussians_streams(sampler, source, states, out, *, spare=None, has_spare=None, spare_out=None,
                           has_spare_out=None, states_out=None, checksum=None, psum=None,
                           guard: int = DEFAULT_GUARD, stream=None, sync: bool = True) -> None:
    """Fill out[s, :n_per] for every stream s.

    sampler: a GaussianSampler or sampler id; source: 'lcg48' / 'splitmix'.
    states (int64 CUDA tensor) is advanced in place unless states_out is given.
    Polar: spare/has_spare carry the cached deviate in, spare_out/has_spare_out
    receive it (default: written back into spare/has_spare when given).
    checksum (int64 [n]) / psum (float64 [n, 4]) receive the fused per-row xor
    checksum and power sums.  sync=False leaves guard checking to the caller
    (engine_check(stream)).
    """
    torch = _torch()
    L = _lib.load()
    smp = make_sampler(sampler) if isinstance(sampler, str) else sampler
    alg = {"polar": 0, "ziggurat": 1, "modified-ziggurat": 2}[smp.algorithm_id]
    src = _lib.SRC[_source_id(source)]
    if out.dtype != torch.float64 or out.dim() != 2 or out.stride(1) != 1 or not out.is_cuda:
        raise ValueError("out must be a float64 CUDA tensor [n_streams, n_per] with unit column stride")
    n, n_per = out.shape
    ld = out.stride(0) if n > 1 else n_per
    want = (n,) if src == 0 else (n, 2)
    if tuple(states.shape) != want or states.dtype != torch.int64 or not states.is_contiguous():
        raise ValueError(f"states must be a contiguous int64 tensor of shape {want}")
    slot = 0
    if alg:
        from .engine import table_slot

        slot = table_slot(smp.tables)
    if states_out is None:
        states_out = states
    if alg == 0:
        if spare_out is None:
            spare_out = spare if spare is not None else torch.zeros(n, dtype=torch.float64, device=out.device)
        if has_spare_out is None:
            has_spare_out = has_spare if has_spare is not None else torch.zeros(n, dtype=torch.uint8,
                                                                                device=out.device)
    s = _stream_handle(out.device, stream)
    check(L.gz_fill_gaussians(alg, src, slot, n, n_per, ld, _p(states), _p(states_out),
                              _p(spare) if alg == 0 else None, _p(has_spare) if alg == 0 else None,
                              _p(spare_out) if alg == 0 else None, _p(has_spare_out) if alg == 0 else None,
                              _p(out), _p(checksum), _p(psum), guard, s))
    if sync:
        check(L.gz_stream_check(s))


def set_kernel_policy(policy: str) -> None:
    """'auto', 'warp' (one warp decodes one stream) or 'lane' (one lane per stream)."""
    L = _lib.load()
    check(L.gz_set_kernel_policy({"auto": 0, "warp": 1, "lane": 2, "lane-ring": 3, "lane-tma": 4}[policy]))


def fill_u64_streams(source, states, out, *, stream=None, sync: bool = True) -> None:
    """Raw draws: out[s, j] = j-th u64 of stream s (engine.py:224-232)."""
    L = _lib.load()
    n, n_per = out.shape
    s = _stream_handle(out.device, stream)
    check(L.gz_fill_u64(_lib.SRC[_source_id(source)], n, n_per, out.stride(0) if n > 1 else n_per, _p(states),
                        _p(states), _p(out), s))
    if sync:
        check(L.gz_stream_check(s))


def engine_check(stream=None, device=None) -> None:
    """Synchronise and raise RejectionLoopExceeded if a guard tripped."""
    L = _lib.load()
    check(L.gz_stream_check(_stream_handle(device, stream)))


# ---- seeding conventions of the BASELINE configs ----

@dataclass(frozen=True)
class ConfigSpec:
    name: str
    sampler: str
    source: str
    scheme: str
    master: int
    n_per: int
    n_streams: int   # per GPU for configs that shard weakly; box-wide for c3


CONFIGS = {
    "c1": ConfigSpec("c1", "ziggurat", "splitmix", "sm_output_of_master", 42, 4096, 1024),
    "c2": ConfigSpec("c2", "polar", "lcg48", "lcg_master_plus_id", 7, 256, 1 << 20),
    "c3": ConfigSpec("c3", "modified-ziggurat", "splitmix", "sm_output_of_master", 1234, 1024, 1 << 20),
    "c4": ConfigSpec("c4", "ziggurat", "lcg48", "lcg_master_plus_id", 99, 256, 1 << 22),
    "c5": ConfigSpec("c5", "ziggurat", "splitmix", "sm_id_xor_master", 0xC0FFEE, 1024, 65536),
}


def seed_streams(scheme: str, master: int, first_id: int, count: int, device="cuda", stream=None):
    """Device-seeded stream states for ids first_id .. first_id+count-1."""
    torch = _torch()
    L = _lib.load()
    code = _lib.SEED[scheme]
    shape = (count,) if code == 0 else (count, 2)
    st = torch.empty(shape, dtype=torch.int64, device=device)
    s = _stream_handle(st.device, stream)
    check(L.gz_seed_streams(code, master & MASK64, first_id, count, _p(st), s))
    return st


def config_states(cfg: str, first_id: int, count: int, device="cuda", stream=None):
    c = CONFIGS[cfg]
    return seed_streams(c.scheme, c.master, first_id, count, device, stream)


def mutate(states, x, sigma, generations: int = 1, *, tables=None, guard: int = DEFAULT_GUARD, stream=None,
           sync: bool = True) -> None:
    """x[i, :] += sigma[i] * z (two roundings) with the original ziggurat over
    individual i's SplitMix64 stream, `generations` times (config 5)."""
    torch = _torch()
    L = _lib.load()
    from .engine import table_slot
    from .samplers import _default_tables

    t = tables if tables is not None else _default_tables(128)
    slot = table_slot(t)
    n_ind, n_genes = x.shape
    if x.dtype != torch.float64 or x.stride(1) != 1:
        raise ValueError("x must be float64 [n_ind, n_genes] with unit column stride")
    s = _stream_handle(x.device, stream)
    check(L.gz_mutate(slot, n_ind, n_genes, x.stride(0) if n_ind > 1 else n_genes, _p(states), _p(states), _p(x),
                      _p(sigma), generations, guard, s))
    if sync:
        check(L.gz_stream_check(s))


def init_population(n_ind: int, n_genes: int, seed: int = 2024, first_ind: int = 0, total_ind: int | None = None,
                    device="cuda"):
    """Config-5 population: x[i, g] = -5 + 10*u over SplitMix64(seed), draws in
    row-major (i, g) order; sigma_i = 10**(-3 + 3*u) from the same stream after
    all total_ind*n_genes genes (pow on the host: libm, init only).  Returns
    (x [n_ind, n_genes] float64 CUDA, sigma [n_ind] float64 CUDA) for
    individuals first_ind .. first_ind + n_ind - 1 (a shard of the population)."""
    torch = _torch()
    L = _lib.load()
    total_ind = n_ind if total_ind is None else total_ind
    x = torch.empty((n_ind, n_genes), dtype=torch.float64, device=device)
    start = (seed + first_ind * n_genes * GOLDEN_GAMMA) & MASK64
    st = torch.tensor(np.array([start, GOLDEN_GAMMA], dtype=np.uint64).view(np.int64), device=device)
    s = _stream_handle(x.device)
    check(L.gz_fill_unit_affine(1, _p(st), n_ind * n_genes, -5.0, 10.0, _p(x), s))
    sig = np.empty(n_ind)
    base = seed + total_ind * n_genes * GOLDEN_GAMMA
    for k in range(n_ind):
        u = SplitMix64((base + (first_ind + k) * GOLDEN_GAMMA) & MASK64).next_f64_unit()
        sig[k] = 10.0 ** (-3.0 + 3.0 * u)
    check(L.gz_stream_check(s))
    return x, torch.from_numpy(sig).to(device)


# ---- reductions -----------------------------------------------------------------

@dataclass
class MomentSummary:
    """Same fields as the reference's stats.MomentSummary (stats.py:232-259)."""

    n: int
    mean: float
    variance: float
    skewness: float
    excess_kurtosis: float

    def to_json_dict(self) -> dict:
        """stats.py:164-172 field layout."""
        return {"test": "moments", "n": self.n, "mean": self.mean, "variance": self.variance,
                "skewness": self.skewness, "excess_kurtosis": self.excess_kurtosis}


def central_from_psum(psum, values_per_row: int, stream=None):
    """Deterministic device reduction of per-row power sums -> (n, mean, M2, M3, M4)."""
    torch = _torch()
    L = _lib.load()
    out5 = torch.empty(5, dtype=torch.float64, device=psum.device)
    s = _stream_handle(psum.device, stream)
    check(L.gz_moments_reduce(_p(psum), psum.shape[0], values_per_row, _p(out5), s))
    return out5


def merge_central(parts):
    """Pebay/Chan pairwise merge of (n, mean, M2, M3, M4) tuples, in order."""
    n, mean, m2, m3, m4 = parts[0]
    for (nb, mb, m2b, m3b, m4b) in parts[1:]:
        na = n
        nn = na + nb
        delta = mb - mean
        d_n = delta / nn
        m4 = (m4 + m4b + delta * d_n ** 3 * na * nb * (na * na - na * nb + nb * nb)
              + 6.0 * d_n * d_n * (na * na * m2b + nb * nb * m2) + 4.0 * d_n * (na * m3b - nb * m3))
        m3 = m3 + m3b + delta * d_n * d_n * na * nb * (na - nb) + 3.0 * d_n * (na * m2b - nb * m2)
        m2 = m2 + m2b + delta * d_n * na * nb
        mean = mean + d_n * nb
        n = nn
    return n, mean, m2, m3, m4


def summarize(n, mean, m2, m3, m4) -> MomentSummary:
    """stats.py:249-258 conventions (unbiased variance, population kurtosis)."""
    n = int(round(n))
    if n < 4:
        raise ValueError(f"moments requires n >= 4, got {n}")
    if m2 == 0.0:
        return MomentSummary(n, mean, m2 / (n - 1), 0.0, 0.0)
    return MomentSummary(n, mean, m2 / (n - 1), math.sqrt(float(n)) * m3 / m2 ** 1.5, n * m4 / (m2 * m2) - 3.0)


def moments_from_psum(psum, values_per_row: int) -> MomentSummary:
    return summarize(*central_from_psum(psum, values_per_row).cpu().tolist())


def xor_fold(checksums) -> int:
    """Global xor of per-stream checksums (device reduction)."""
    torch = _torch()
    L = _lib.load()
    out = torch.zeros(1, dtype=torch.int64, device=checksums.device)
    s = _stream_handle(checksums.device)
    check(L.gz_xor_reduce(_p(checksums), checksums.numel(), _p(out), s))
    check(L.gz_stream_check(s))
    return int(out.cpu().numpy().view(np.uint64)[0])
