"""ctypes binding for the CPU oracle (oracle/gz_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker.  Imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg; never by the product
package (paper_2405_19493_b200/), which must fail loudly without its CUDA
library instead of falling back to this code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgzoracle.so")

ALG = {"polar": 0, "ziggurat": 1, "modified-ziggurat": 2}
SRC = {"lcg48": 0, "splitmix": 1}
GUARD = 1_000_000  # samplers.py:27 LOOP_GUARD / engine.py:37 _GUARD
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


class GzoTables(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("r", ctypes.c_double), ("v", ctypes.c_double),
                ("x", ctypes.c_double * 1025), ("ktab", ctypes.c_uint64 * 1024),
                ("wtab", ctypes.c_double * 1024), ("ytab", ctypes.c_double * 1025)]


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.gzo_build_tables.argtypes = [ctypes.c_int, ctypes.POINTER(GzoTables)]
        L.gzo_fill_gaussians.argtypes = [ctypes.c_int, ctypes.c_int, P, i64, i64, i64, P, P, P, P, P, P, P,
                                         i64, ctypes.c_int]
        L.gzo_fill_digest.argtypes = [ctypes.c_int, ctypes.c_int, P, i64, i64, P, P, P, P, P, P, P, P, i64,
                                      ctypes.c_int]
        L.gzo_fill_u64.argtypes = [ctypes.c_int, i64, i64, i64, P, P, P]
        L.gzo_occupancy.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, i64, P, P, i64]
        L.gzo_tail_sample.argtypes = [ctypes.c_int, P, P, ctypes.c_double, i64, P]
        L.gzo_mutate.argtypes = [P, i64, i64, i64, P, P, P, P, ctypes.c_int, i64, ctypes.c_int]
        L.gzo_checksum.argtypes = [P, i64]
        L.gzo_checksum.restype = ctypes.c_uint64
        L.gzo_moments_accumulate.argtypes = [P, i64, P]
        L.gzo_mix64.argtypes = [ctypes.c_uint64]
        L.gzo_mix64.restype = ctypes.c_uint64
        L.gzo_mix_gamma.argtypes = [ctypes.c_uint64]
        L.gzo_mix_gamma.restype = ctypes.c_uint64
        for f in ("gzo_exp", "gzo_log"):
            getattr(L, f).argtypes = [ctypes.c_double]
            getattr(L, f).restype = ctypes.c_double
        L.gzo_libm_mismatches.argtypes = [ctypes.c_int, P, P, i64, ctypes.POINTER(ctypes.c_int64)]
        L.gzo_libm_mismatches.restype = ctypes.c_int64
        L.gzo_pow.argtypes = [ctypes.c_double, ctypes.c_double]
        L.gzo_pow.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Tables:
    """Oracle ziggurat tables (tables.py:107-131 restated in C)."""

    def __init__(self, n):
        self.raw = GzoTables()
        st = lib().gzo_build_tables(int(n), ctypes.byref(self.raw))
        if st == 2:
            raise ValueError(f"layer count must be a power of two >= 8, got {n}")
        if st != 0:
            raise RuntimeError(f"table construction failed for n={n}")
        self.n = n
        self.r = self.raw.r
        self.v = self.raw.v
        self.x = np.ctypeslib.as_array(self.raw.x)[: n + 1].copy()
        self.ktab = np.ctypeslib.as_array(self.raw.ktab)[:n].copy()
        self.wtab = np.ctypeslib.as_array(self.raw.wtab)[:n].copy()
        self.ytab = np.ctypeslib.as_array(self.raw.ytab)[: n + 1].copy()


_TABLES = {}


def tables(n):
    if n not in _TABLES:
        _TABLES[n] = Tables(n)
    return _TABLES[n]


def default_layers(alg):
    return 256 if alg == "modified-ziggurat" else 128


def fill_gaussians(alg, source, states, n_per, spare=None, has=None, layers=None, guard=GUARD,
                   nthreads=0):
    """Multi-stream fill.  states: uint64[n] (lcg48) or uint64[n, 2] (splitmix).
    Returns (out[n, n_per], states_out, spare_out, has_out, status)."""
    states = np.ascontiguousarray(states, dtype=np.uint64)
    n = states.shape[0]
    out = np.zeros((n, n_per), dtype=np.float64)
    st_out = np.empty_like(states)
    t = None if alg == "polar" else tables(layers or default_layers(alg))
    spare_out = np.zeros(n) if alg == "polar" else None
    has_out = np.zeros(n, dtype=np.uint8) if alg == "polar" else None
    if spare is not None:
        spare = np.ascontiguousarray(spare, dtype=np.float64)
        has = np.ascontiguousarray(has, dtype=np.uint8)
    status = lib().gzo_fill_gaussians(ALG[alg], SRC[source], None if t is None else ctypes.byref(t.raw), n,
                                      n_per, n_per, _p(states), _p(st_out), _p(spare), _p(has),
                                      _p(spare_out), _p(has_out), _p(out), guard, nthreads)
    return out, st_out, spare_out, has_out, status


def fill_digest(alg, source, states, n_per, spare=None, has=None, layers=None, guard=GUARD, nthreads=0,
                psum=False):
    """fill_gaussians without the output buffer (full-size parity checks).
    Returns (digest uint64[n, 3], states_out, spare_out, has_out, psum f64[n, 4] or None, status);
    digest = (xor of bit patterns, sum (j+1)*(bits>>32), sum (j+1)*(bits & 0xffffffff)) mod 2^64."""
    states = np.ascontiguousarray(states, dtype=np.uint64)
    n = states.shape[0]
    dig = np.zeros((n, 3), dtype=np.uint64)
    st_out = np.empty_like(states)
    t = None if alg == "polar" else tables(layers or default_layers(alg))
    spare_out = np.zeros(n) if alg == "polar" else None
    has_out = np.zeros(n, dtype=np.uint8) if alg == "polar" else None
    ps = np.zeros((n, 4)) if psum else None
    if spare is not None:
        spare = np.ascontiguousarray(spare, dtype=np.float64)
        has = np.ascontiguousarray(has, dtype=np.uint8)
    status = lib().gzo_fill_digest(ALG[alg], SRC[source], None if t is None else ctypes.byref(t.raw), n, n_per,
                                   _p(states), _p(st_out), _p(spare), _p(has), _p(spare_out), _p(has_out),
                                   _p(dig), _p(ps), guard, nthreads)
    return dig, st_out, spare_out, has_out, ps, status


def digest_rows(rows):
    """The fill_digest witnesses of materialised rows (numpy float64 [n, n_per])."""
    b = np.ascontiguousarray(rows, dtype=np.float64).view(np.uint64)
    w = np.arange(1, b.shape[1] + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return np.stack([np.bitwise_xor.reduce(b, axis=1), ((b >> np.uint64(32)) * w).sum(1, dtype=np.uint64),
                         ((b & np.uint64(0xffffffff)) * w).sum(1, dtype=np.uint64)], 1)


def occupancy(alg, source, state_words, n_calls, layers=None, guard=GUARD):
    """One stream's sample_with_occupancy (samplers.py:89-93): (deviates, counts, state_out, status)."""
    st = np.ascontiguousarray(state_words, dtype=np.uint64)
    st_out = np.empty_like(st)
    t = tables(layers or default_layers(alg))
    out = np.zeros(max(n_calls, 1))
    counts = np.zeros(t.n, dtype=np.uint64)
    status = lib().gzo_occupancy(ALG[alg], SRC[source], ctypes.byref(t.raw), _p(st), _p(st_out), n_calls, _p(out),
                                 _p(counts), guard)
    return out[:n_calls], counts, st_out, status


def tail_sample(source, state_words, r, guard=GUARD):
    """samplers.py:40-57 on one stream: (value, state_out, status)."""
    st = np.ascontiguousarray(state_words, dtype=np.uint64)
    st_out = np.empty_like(st)
    out = np.zeros(1)
    status = lib().gzo_tail_sample(SRC[source], _p(st), _p(st_out), float(r), guard, _p(out))
    return float(out[0]), st_out, status


def fill_u64(source, states, n_per):
    states = np.ascontiguousarray(states, dtype=np.uint64)
    n = states.shape[0]
    out = np.zeros((n, n_per), dtype=np.uint64)
    st_out = np.empty_like(states)
    lib().gzo_fill_u64(SRC[source], n, n_per, n_per, _p(states), _p(st_out), _p(out))
    return out, st_out


def mutate(states, x, sigma, generations, guard=GUARD, nthreads=0):
    """x (n_ind, n_genes) float64 updated in place; states uint64[n, 2] (splitmix)."""
    states = np.ascontiguousarray(states, dtype=np.uint64)
    st_out = np.empty_like(states)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    n_ind, n_genes = x.shape
    status = lib().gzo_mutate(ctypes.byref(tables(128).raw), n_ind, n_genes, n_genes, _p(states), _p(st_out),
                              _p(x), _p(sigma), generations, guard, nthreads)
    return st_out, status


def libm_mismatches(fn, xs, got):
    """(count, first index) of got[k] != libm exp/log(xs[k]) bitwise (fn 0 exp, 1 log)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    got = np.ascontiguousarray(got, dtype=np.float64)
    first = ctypes.c_int64()
    bad = lib().gzo_libm_mismatches(fn, _p(xs), _p(got), xs.size, ctypes.byref(first))
    return int(bad), int(first.value)


def sweep_inputs(fn, n, seed):
    """Inputs for the exp/log sweeps: the samplers' domains plus raw bit patterns."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 2 ** 64 - 1, n // 4, dtype=np.uint64, endpoint=True).view(np.float64)
    if fn == 0:  # wedge test argument -0.5*x*x, x < r(256) = 3.654...
        dom = -0.5 * (3.7 * rng.random(n)) ** 2
    else:        # tail uniforms (53-bit grid) and polar s in (0, 1)
        grid = rng.integers(1, 2 ** 53, n // 2, dtype=np.uint64).astype(np.float64) * 2.0 ** -53
        dom = np.concatenate([grid, rng.random(n - n // 2)])
        raw = np.abs(raw)
    return np.concatenate([dom, raw])


def checksum(buf):
    buf = np.ascontiguousarray(buf, dtype=np.float64).reshape(-1)
    return int(lib().gzo_checksum(_p(buf), buf.size))


def moments_accumulate(xs, acc=None):
    xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1)
    acc = np.zeros(5) if acc is None else acc
    lib().gzo_moments_accumulate(_p(xs), xs.size, _p(acc))
    return acc


def moments_summary(acc):
    """stats.py:249-258 from the accumulated (n, mean, m2, m3, m4)."""
    import math
    n, mean, m2, m3, m4 = acc
    n = int(n)
    variance = m2 / (n - 1)
    if m2 == 0.0:
        return n, mean, variance, 0.0, 0.0
    skew = math.sqrt(float(n)) * m3 / m2 ** 1.5
    kurt = n * m4 / (m2 * m2) - 3.0
    return n, mean, variance, skew, kurt


# ---- seeding conventions of the five configs ----

def mix64(z):
    return int(lib().gzo_mix64(z & MASK64))


def lcg_state(seed):
    return ((seed ^ 0x5DEECE66D) & ((1 << 48) - 1))


def sm_output_seed(master, i):
    return mix64((master + (i + 1) * GOLDEN_GAMMA) & MASK64)


def mix64_np(z):
    """sources.py:83-87 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def config_states_range(cfg, first, count):
    """config_states(cfg, range(first, first + count)), vectorised (large shards)."""
    ids = np.arange(first, first + count, dtype=np.uint64)
    g = np.uint64(GOLDEN_GAMMA)
    with np.errstate(over="ignore"):
        if cfg in ("c2", "c4"):
            base = np.uint64(7 if cfg == "c2" else 99)
            return ((base + ids) ^ np.uint64(0x5DEECE66D)) & np.uint64((1 << 48) - 1)
        if cfg in ("c1", "c3"):
            m = np.uint64(42 if cfg == "c1" else 1234)
            s = mix64_np(m + (ids + np.uint64(1)) * g)
        elif cfg == "c5":
            s = ids ^ np.uint64(0xC0FFEE)
        else:
            raise ValueError(cfg)
    return np.stack([s, np.full_like(s, g)], 1)


def config_states(cfg, ids):
    """Initial per-stream states of config `cfg` for the given stream ids."""
    ids = [int(i) for i in ids]
    if cfg == "c1":
        return np.array([[sm_output_seed(42, i), GOLDEN_GAMMA] for i in ids], dtype=np.uint64)
    if cfg == "c2":
        return np.array([lcg_state(7 + i) for i in ids], dtype=np.uint64)
    if cfg == "c3":
        return np.array([[sm_output_seed(1234, i), GOLDEN_GAMMA] for i in ids], dtype=np.uint64)
    if cfg == "c4":
        return np.array([lcg_state(99 + i) for i in ids], dtype=np.uint64)
    if cfg == "c5":
        return np.array([[i ^ 0xC0FFEE, GOLDEN_GAMMA] for i in ids], dtype=np.uint64)
    raise ValueError(cfg)
