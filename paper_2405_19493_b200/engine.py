"""Batch engine: the drop-in for the reference's engine.py, on the B200.

`fill_gaussians(sampler, source, out)` and `fill_u64(source, out)` keep the
signatures and state write-back of /root/reference/pkg/src/gausszig/engine.py
(fill_u64 224-232, fill_gaussians 235-270, supports 199-201, available 46-47,
warm_up 273-281): the source's `state` and the polar sampler's `spare` are read
before the call and written back after it, so batch calls and per-call calls
interleave exactly as in the reference.

`out` may be a numpy array (host memory: the call copies the stream state in,
generates on the GPU and copies the deviates back -- gz_fill_gaussians_host)
or a CUDA torch tensor (generated in place -- gz_fill_gaussians).

Differences by design: there is no CPU fallback.  A source without a kernel
(ScriptedSource) raises TypeError instead of running the per-call Python loop,
and without libgzb200.so or a CUDA device every call raises EngineUnavailable.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from ._lib import DEFAULT_GUARD, EngineUnavailable, RejectionLoopExceeded, check
from .samplers import GaussianSampler, ModifiedZigguratSampler, PolarSampler, ZigguratSampler
from .sources import Lcg48, ScriptedSource, ScriptExhausted, SplitMix64, UniformSource, make_source
from .tables import ZigguratTables

__all__ = ["available", "supports", "fill_u64", "fill_gaussians", "warm_up", "table_slot", "EngineUnavailable",
           "RejectionLoopExceeded"]


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else ctypes.c_void_p(a.data_ptr())


def available() -> bool:
    """True when libgzb200.so loads and a CUDA device is visible."""
    try:
        _lib.load()
        return True
    except (EngineUnavailable, OSError):
        return False


def supports(source: UniformSource) -> bool:
    """Whether a device kernel exists for this source (engine.py:199-201): the two
    PRNGs, and the scripted test double (replayed call by call by one device thread)."""
    return isinstance(source, (Lcg48, SplitMix64, ScriptedSource)) and available()


def _fill_scripted(sampler: GaussianSampler, source: ScriptedSource, out, guard: int) -> None:
    """Scripted words replayed on the device (gz_fill_scripted): the sampler loop of
    samplers.py by one thread; the source's cursor and the polar spare advance like
    the reference's per-call path."""
    import torch

    L = _lib.load()
    alg = _alg_of(sampler)
    slot = 0 if alg == 0 else table_slot(sampler.tables)
    n = len(out)
    words = np.array(source.words[source.cursor:], dtype=np.uint64)
    d_w = torch.from_numpy(words.view(np.int64).copy()).to("cuda")
    d_c = torch.zeros(1, dtype=torch.int64, device="cuda")
    d_out = out if _is_cuda_tensor(out) else torch.empty(n, dtype=torch.float64, device="cuda")
    polar = alg == 0
    sp = torch.tensor([sampler.spare if polar and sampler.spare is not None else 0.0], dtype=torch.float64,
                      device="cuda")
    hs = torch.tensor([1 if polar and sampler.spare is not None else 0], dtype=torch.uint8, device="cuda")
    spo = torch.zeros(1, dtype=torch.float64, device="cuda")
    hso = torch.zeros(1, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    check(L.gz_fill_scripted(alg, slot, _ptr(d_w), words.size, _ptr(d_c), n, _ptr(d_out),
                             _ptr(sp) if polar else None, _ptr(hs) if polar else None,
                             _ptr(spo) if polar else None, _ptr(hso) if polar else None, guard, s))
    try:
        check(L.gz_stream_check(s))
    finally:
        source.cursor += int(d_c.cpu()[0])
    if not _is_cuda_tensor(out):
        out[...] = d_out.cpu().numpy()
    if polar:
        sampler.spare = float(spo.cpu()[0]) if int(hso.cpu()[0]) else None


# ---- table slots --------------------------------------------------------------

_slots: dict = {}     # (device, id(tables)) -> (slot, tables)
_next_slot: dict = {}


def _current_device() -> int:
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except ImportError:  # pragma: no cover
        return 0


def table_slot(tables: ZigguratTables) -> int:
    """Device table slot holding `tables` (uploaded on first use; replaces the
    lru_cache'd _table_arrays of engine.py:216-221)."""
    L = _lib.load()
    dev = _current_device()
    key = (dev, id(tables))
    hit = _slots.get(key)
    if hit is not None and hit[1] is tables:
        return hit[0]
    slot = _next_slot.get(dev, 0)
    if slot >= 16:  # recycle: drop every slot of this device
        for k in [k for k in _slots if k[0] == dev]:
            del _slots[k]
        slot = 0
    _next_slot[dev] = slot + 1
    k = np.ascontiguousarray(tables.ktab, dtype=np.uint64)
    w = np.ascontiguousarray(tables.wtab, dtype=np.float64)
    y = np.ascontiguousarray(tables.ytab, dtype=np.float64)
    check(L.gz_tables_upload(slot, tables.n, _ptr(k), _ptr(w), _ptr(y), tables.r))
    _slots[key] = (slot, tables)
    return slot


def _alg_of(sampler: GaussianSampler) -> int:
    if isinstance(sampler, PolarSampler):
        return _lib.ALG["polar"]
    if isinstance(sampler, ModifiedZigguratSampler):
        return _lib.ALG["modified-ziggurat"]
    if isinstance(sampler, ZigguratSampler):
        return _lib.ALG["ziggurat"]
    raise TypeError(f"no engine kernel for sampler {getattr(sampler, 'algorithm_id', sampler)!r}")


def _state_words(source: UniformSource) -> np.ndarray:
    """engine.py:204-209 `_state_array`."""
    if isinstance(source, Lcg48):
        return np.array([source.state], dtype=np.uint64)
    if isinstance(source, SplitMix64):
        return np.array([source.state, source.gamma], dtype=np.uint64)
    raise TypeError(f"no engine support for source {source.source_id!r} (the B200 engine has no CPU fallback)")


_io = threading.local()


def _io_words(dev):
    """A pinned host int64[8] and a device int64[8] for one call's small inputs and
    outputs (state in/out, spare in/out, flags), cached per thread and device:
    one H2D and one D2H copy per call instead of five tensors."""
    import torch

    key = dev.index if dev.index is not None else torch.cuda.current_device()
    cache = getattr(_io, "bufs", None)
    if cache is None:
        cache = _io.bufs = {}
    if key not in cache:
        cache[key] = (torch.zeros(8, dtype=torch.int64).pin_memory(),
                      torch.zeros(8, dtype=torch.int64, device=torch.device("cuda", key)))
    return cache[key]


def _is_cuda_tensor(out) -> bool:
    return hasattr(out, "is_cuda") and bool(out.is_cuda)


def fill_u64(source: UniformSource, out) -> None:
    """Fill `out` (uint64, 1-D) with draws, advancing the source in place."""
    if isinstance(source, ScriptedSource):
        n = len(out)
        if source.remaining() < n:
            source.cursor = len(source.words)
            raise ScriptExhausted(f"script exhausted after {len(source.words)} words")
        words = np.array(source.words[source.cursor:source.cursor + n], dtype=np.uint64)
        source.cursor += n
        if _is_cuda_tensor(out):
            import torch

            out.copy_(torch.from_numpy(words.view(np.int64)))
        else:
            np.asarray(out).view(np.uint64)[...] = words
        return
    L = _lib.load()
    st = _state_words(source)
    src = _lib.SRC[source.source_id]
    if _is_cuda_tensor(out):
        import torch

        if out.dim() != 1 or not out.is_contiguous() or out.element_size() != 8:
            raise ValueError("out must be a contiguous 1-D 64-bit CUDA tensor")
        d_st = torch.from_numpy(st.view(np.int64)).to(out.device)
        s = torch.cuda.current_stream(out.device).cuda_stream
        check(L.gz_fill_u64(src, 1, out.numel(), out.numel(), _ptr(d_st), _ptr(d_st), _ptr(out), s))
        check(L.gz_stream_check(s))
        st = d_st.cpu().numpy().view(np.uint64)
    else:
        import torch

        buf = np.ascontiguousarray(out) if isinstance(out, np.ndarray) else np.asarray(out)
        if buf.dtype != np.uint64 or buf.ndim != 1:
            raise ValueError("out must be a 1-D uint64 array")
        d_st = torch.from_numpy(st.view(np.int64)).cuda()
        d_out = torch.empty(buf.shape[0], dtype=torch.int64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        check(L.gz_fill_u64(src, 1, buf.shape[0], buf.shape[0], _ptr(d_st), _ptr(d_st), _ptr(d_out), s))
        check(L.gz_stream_check(s))
        buf[...] = d_out.cpu().numpy().view(np.uint64)
        if buf is not out:
            out[...] = buf
        st = d_st.cpu().numpy().view(np.uint64)
    source.state = int(st[0])


def fill_gaussians(sampler: GaussianSampler, source: UniformSource, out, guard: int = DEFAULT_GUARD) -> None:
    """Fill `out` (float64, 1-D) with deviates, advancing sampler and source
    state exactly as `sampler.next_gaussian(source)` called len(out) times would."""
    if isinstance(source, ScriptedSource):
        _alg_of(sampler)
        return _fill_scripted(sampler, source, out, guard)
    L = _lib.load()
    alg = _alg_of(sampler)
    st = _state_words(source)
    src = _lib.SRC[source.source_id]
    slot = 0 if alg == 0 else table_slot(sampler.tables)
    polar = alg == 0
    spare_in = np.array([sampler.spare if polar and sampler.spare is not None else 0.0])
    has_in = np.array([1 if polar and sampler.spare is not None else 0], dtype=np.uint8)
    spare_out = np.zeros(1)
    has_out = np.zeros(1, dtype=np.uint8)
    if _is_cuda_tensor(out):
        import torch

        if out.dim() != 1 or not out.is_contiguous() or out.dtype != torch.float64:
            raise ValueError("out must be a contiguous 1-D float64 CUDA tensor")
        dev = out.device
        h, d = _io_words(dev)
        hv = h.numpy()
        hv[:] = 0
        hv[:st.size] = st.view(np.int64)
        if polar:
            hv[4] = spare_in.view(np.int64)[0]
            hv[5] = int(has_in[0])
        d.copy_(h, non_blocking=True)
        base = d.data_ptr()
        s = torch.cuda.current_stream(dev).cuda_stream
        n = out.numel()
        check(L.gz_fill_gaussians(alg, src, slot, 1, n, n, ctypes.c_void_p(base), ctypes.c_void_p(base + 16),
                                  ctypes.c_void_p(base + 32) if polar else None,
                                  ctypes.c_void_p(base + 40) if polar else None,
                                  ctypes.c_void_p(base + 48) if polar else None,
                                  ctypes.c_void_p(base + 56) if polar else None,
                                  _ptr(out), None, None, guard, s))
        h.copy_(d, non_blocking=True)
        check(L.gz_stream_check(s))          # synchronises the stream: h holds the results
        st = hv[2:2 + st.size].copy().view(np.uint64)
        spare_out = hv[6:7].copy().view(np.float64)
        has_out = np.array([hv[7] & 0xFF], dtype=np.uint8)
    else:
        buf = out if (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.ndim == 1
                      and out.flags.c_contiguous) else np.empty(len(out), dtype=np.float64)
        st_out = np.empty_like(st)
        check(L.gz_fill_gaussians_host(alg, src, slot, 1, buf.shape[0], _ptr(st), _ptr(st_out),
                                       _ptr(spare_in) if polar else None, _ptr(has_in) if polar else None,
                                       _ptr(spare_out) if polar else None, _ptr(has_out) if polar else None,
                                       _ptr(buf), None, guard))
        if buf is not out:
            out[...] = buf
        st = st_out
    source.state = int(st[0])
    if polar:
        sampler.spare = float(spare_out[0]) if has_out[0] else None


def fill_with_occupancy(sampler: GaussianSampler, source: UniformSource, n_calls: int, guard: int = DEFAULT_GUARD):
    """n_calls ziggurat calls on the device by one thread, counting the layer of
    every attempt (gz_zig_occupancy): returns (deviates list, counts list) and
    advances `source` like the reference's sample_with_occupancy."""
    import torch

    L = _lib.load()
    alg = _alg_of(sampler)
    if alg == 0:
        raise TypeError("layer occupancy is defined for the ziggurat samplers only")
    if n_calls < 0:
        raise ValueError(f"n_calls must be >= 0, got {n_calls}")
    st = _state_words(source)
    src = _lib.SRC[source.source_id]
    slot = table_slot(sampler.tables)
    d_st = torch.from_numpy(st.view(np.int64)).to("cuda")
    d_out = torch.empty(max(n_calls, 1), dtype=torch.float64, device="cuda")
    d_cnt = torch.zeros(sampler.tables.n, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    check(L.gz_zig_occupancy(alg, src, slot, _ptr(d_st), _ptr(d_st), n_calls, _ptr(d_out), _ptr(d_cnt), guard, s))
    check(L.gz_stream_check(s))
    source.state = int(d_st.cpu().numpy().view(np.uint64)[0])
    return d_out[:n_calls].cpu().tolist(), [int(c) for c in d_cnt.cpu().tolist()]


def warm_up(sampler: GaussianSampler, source_id: str) -> None:
    """Upload tables and run one small fill so a timed region sees no first-use cost."""
    if not available():
        return
    fill_gaussians(sampler, make_source(source_id, 0), np.empty(64))
