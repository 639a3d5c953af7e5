"""Gaussian samplers: the API surface of the reference's samplers.py.

The classes keep the reference's names, constructor arguments and mutable
state (`tables`, the polar `spare`) -- samplers.py:60-200 -- but every draw runs
on the GPU through engine.fill_gaussians: `next_gaussian(src)` is a
one-element fill, `sample(src, n)` an n-element fill.  The pairing gate
(samplers.py:203-222) is kept at caller level exactly as in the reference.
"""
from __future__ import annotations

import abc
import ctypes

import numpy as np

from ._lib import RejectionLoopExceeded
from .tables import ZigguratTables, build_ziggurat_tables

LOOP_GUARD = 1_000_000
SAMPLER_IDS = ("polar", "ziggurat", "modified-ziggurat")
_UNSAFE_PAIRINGS = {("lcg48", "modified-ziggurat")}

__all__ = ["LOOP_GUARD", "SAMPLER_IDS", "GaussianSampler", "ZigguratSampler", "ModifiedZigguratSampler",
           "PolarSampler", "RejectionLoopExceeded", "UnsanctionedPairing", "gaussian_affine", "is_sanctioned",
           "require_sanctioned", "make_sampler"]


def tail_sample(src, r: float, guard: int = LOOP_GUARD) -> float:
    """One deviate from the normal tail beyond r > 0 (samplers.py:40-57), drawn from
    `src` on the device (one thread); advances src like the reference."""
    import torch

    from . import engine
    from ._lib import SRC, check, load

    if not r > 0.0:
        raise ValueError(f"tail boundary must be positive, got {r}")
    L = load()
    from .sources import ScriptedSource

    if isinstance(src, ScriptedSource):
        words = np.array(src.words[src.cursor:], dtype=np.uint64)
        d_w = torch.from_numpy(words.view(np.int64).copy()).to("cuda")
        d_c = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        check(L.gz_tail_scripted(ctypes.c_void_p(d_w.data_ptr()), words.size, ctypes.c_void_p(d_c.data_ptr()),
                                 float(r), guard, ctypes.c_void_p(out.data_ptr()), s))
        try:
            check(L.gz_stream_check(s))
        finally:
            src.cursor += int(d_c.cpu()[0])
        return float(out.cpu()[0])
    st = engine._state_words(src)
    d = torch.from_numpy(st.view(np.int64).copy()).to("cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    check(L.gz_tail_sample(SRC[src.source_id], ctypes.c_void_p(d.data_ptr()), float(r), guard,
                           ctypes.c_void_p(out.data_ptr()), s))
    check(L.gz_stream_check(s))
    src.state = int(d.cpu().numpy().view(np.uint64)[0])
    return float(out.cpu()[0])


class UnsanctionedPairing(ValueError):
    """The modified ziggurat over the LCG (low state bits have short periods)."""


class GaussianSampler(abc.ABC):
    """A standard-normal sampler fed by an external uniform source."""

    algorithm_id = "abstract"

    def next_gaussian(self, src) -> float:
        """One N(0, 1) deviate (a one-element GPU fill)."""
        from . import engine

        buf = np.empty(1)
        engine.fill_gaussians(self, src, buf)
        return float(buf[0])

    def sample(self, src, n: int) -> list:
        """n deviates as a list."""
        from . import engine

        buf = np.empty(n)
        engine.fill_gaussians(self, src, buf)
        return buf.tolist()


class _ZigguratBase(GaussianSampler):
    default_layers = 128

    def __init__(self, tables: ZigguratTables | None = None):
        self.tables = tables if tables is not None else _default_tables(self.default_layers)

    def sample_with_occupancy(self, src, n_calls: int):
        """(deviates, per-layer selection counts over all attempts) of n_calls
        calls, advancing src (samplers.py:89-93, 138-142); run on the device."""
        from . import engine

        return engine.fill_with_occupancy(self, src, n_calls)


_TABLE_CACHE: dict = {}


def _default_tables(n):
    if n not in _TABLE_CACHE:
        _TABLE_CACHE[n] = build_ziggurat_tables(n)
    return _TABLE_CACHE[n]


class ZigguratSampler(_ZigguratBase):
    """Original (GSL-style) ziggurat: sign bit 63, layer index in the next
    index_bits, mantissa below (samplers.py:74-115)."""

    algorithm_id = "ziggurat"
    default_layers = 128


class ModifiedZigguratSampler(_ZigguratBase):
    """Single-draw ziggurat: layer index from the LOW bits, sign just above it,
    mantissa in the remaining high bits (samplers.py:118-165)."""

    algorithm_id = "modified-ziggurat"
    default_layers = 256


class PolarSampler(GaussianSampler):
    """Marsaglia polar method with the one-deep spare cache (samplers.py:168-192)."""

    algorithm_id = "polar"

    def __init__(self):
        self.spare = None

    def reset(self) -> None:
        self.spare = None


def gaussian_affine(src, sampler: GaussianSampler, mu: float, sigma: float) -> float:
    """mu + sigma * z with two roundings (samplers.py:195-200)."""
    if sigma < 0.0:
        raise ValueError(f"sigma must be >= 0, got {sigma}")
    return mu + sigma * sampler.next_gaussian(src)


def is_sanctioned(source_id: str, sampler_id: str) -> bool:
    return (source_id, sampler_id) not in _UNSAFE_PAIRINGS


def require_sanctioned(source_id: str, sampler_id: str) -> None:
    if not is_sanctioned(source_id, sampler_id):
        raise UnsanctionedPairing(
            f"{sampler_id} over {source_id} is refused: the modified ziggurat takes its layer index from the "
            "low-order bits of each draw, and the LCG's low-order state bits have short periods")


def make_sampler(sampler_id: str, layers: int | None = None) -> GaussianSampler:
    """Sampler by identifier, optionally with a custom layer count."""
    if sampler_id == "polar":
        if layers is not None:
            raise ValueError("polar sampler takes no layer count")
        return PolarSampler()
    if sampler_id == "ziggurat":
        return ZigguratSampler(build_ziggurat_tables(layers) if layers else None)
    if sampler_id == "modified-ziggurat":
        return ModifiedZigguratSampler(build_ziggurat_tables(layers) if layers else None)
    raise ValueError(f"unknown sampler id: {sampler_id!r}")
