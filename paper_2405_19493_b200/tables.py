"""Ziggurat layer tables: the API surface of the reference's tables.py.

`build_ziggurat_tables(n)` (reference tables.py:107-131) runs the native host
builder `gz_build_tables` of libgzb200.so -- the boundary bisection, the
equal-area layer recursion and the ktab/wtab/ytab derivation restated in C++
against the same libm -- and returns the same immutable record
(`ZigguratTables`, tables.py:38-64), bit for bit.  The JSON wire format
(tables.py:156-183: reals with 17 significant digits) round-trips exactly.
"""
from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

SOLVE_TOLERANCE = 1e-12
SOLVE_MAX_ITER = 200


class TableConstructionError(RuntimeError):
    """The boundary solve did not converge or the tables failed validation."""


def density(x: float) -> float:
    """Unnormalised normal density exp(-x^2/2) (tables.py:24-26)."""
    return math.exp(-0.5 * x * x)


def tail_area(r: float) -> float:
    """Integral of exp(-x^2/2) over [r, inf) (tables.py:29-31)."""
    return math.sqrt(math.pi / 2.0) * math.erfc(r / math.sqrt(2.0))


@dataclass(frozen=True)
class ZigguratTables:
    """x[0..n] layer abscissas (x[0] = v/f(r) virtual base width, x[1] = r,
    x[n] = 0); ktab[i] integer fast-path threshold; wtab[i] mantissa scale;
    ytab[0..n] densities with ytab[n] = 1."""

    n: int
    r: float
    v: float
    x: tuple
    ktab: tuple
    wtab: tuple
    ytab: tuple

    @property
    def index_bits(self) -> int:
        return self.n.bit_length() - 1

    @property
    def mantissa_bits(self) -> int:
        return 63 - self.index_bits


def build_ziggurat_tables(n: int) -> ZigguratTables:
    """Tables for an n-layer ziggurat, n a power of two >= 8."""
    if not isinstance(n, int) or n < 8 or n & (n - 1):
        raise ValueError(f"layer count must be a power of two >= 8, got {n}")
    L = _lib.load(require_device=False)
    x = np.zeros(n + 1)
    ytab = np.zeros(n + 1)
    ktab = np.zeros(n, dtype=np.uint64)
    wtab = np.zeros(n)
    r, v = ctypes.c_double(), ctypes.c_double()
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    st = L.gz_build_tables(n, ctypes.byref(r), ctypes.byref(v), p(x), p(ktab), p(wtab), p(ytab))
    if st == _lib.GZ_ERR_INVALID:
        raise ValueError(f"layer count must be a power of two >= 8, got {n}")
    if st != _lib.GZ_OK:
        raise TableConstructionError(L.gz_last_error().decode())
    t = ZigguratTables(n=n, r=r.value, v=v.value, x=tuple(x.tolist()), ktab=tuple(int(k) for k in ktab),
                       wtab=tuple(wtab.tolist()), ytab=tuple(ytab.tolist()))
    validate(t)
    return t


def validate(t: ZigguratTables) -> None:
    """The structural checks of tables.py:134-149."""
    n = t.n
    if t.x[n] != 0.0 or t.x[1] != t.r:
        raise TableConstructionError("boundary anchors corrupted")
    if any(not t.x[i] > t.x[i + 1] for i in range(n)):
        raise TableConstructionError("x not strictly decreasing")
    if any(not t.ytab[i] < t.ytab[i + 1] for i in range(n)):
        raise TableConstructionError("ytab not increasing")
    if abs(t.r * density(t.r) + tail_area(t.r) - t.v) > 1e-9 * t.v:
        raise TableConstructionError("base layer area mismatch")
    for i in range(1, n):
        if abs(t.x[i] * (t.ytab[i + 1] - t.ytab[i]) - t.v) > 1e-9 * t.v:
            raise TableConstructionError(f"layer {i} area off")


def _g17(v: float) -> str:
    return format(v, ".17g")


def tables_to_json(t: ZigguratTables) -> str:
    """JSON document; reals carry 17 significant digits (exact round trip)."""
    reals = lambda seq: "[" + ", ".join(_g17(v) for v in seq) + "]"  # noqa: E731
    return ('{"n": %d, "r": %s, "v": %s, "x": %s, "ktab": [%s], "wtab": %s, "ytab": %s}'
            % (t.n, _g17(t.r), _g17(t.v), reals(t.x), ", ".join(str(k) for k in t.ktab), reals(t.wtab),
               reals(t.ytab)))


def tables_from_json(text: str) -> ZigguratTables:
    """Inverse of tables_to_json (validated)."""
    d = json.loads(text)
    t = ZigguratTables(n=int(d["n"]), r=float(d["r"]), v=float(d["v"]), x=tuple(map(float, d["x"])),
                       ktab=tuple(map(int, d["ktab"])), wtab=tuple(map(float, d["wtab"])),
                       ytab=tuple(map(float, d["ytab"])))
    validate(t)
    return t
