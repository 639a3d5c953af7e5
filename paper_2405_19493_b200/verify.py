"""Statistical verification of generated deviates, on the GPU.

The counterpart of the reference's stats.py gates (stats.py:232-353) and the
`verify` / `bits` commands (cli.py:147-208, 239-256), for deviates that already
live in device memory: binning (equal-probability chi-square), the KS distance
(device radix sort) and the low-bits histogram run as kernels
(csrc/gz_verify.cu); only the O(bins) bookkeeping and the p-value special
functions run on the host.  Report fields match the reference's
GofReport / KsReport (stats.py:178-229).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

_SQRT2 = math.sqrt(2.0)


def _torch():
    import torch

    return torch


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check(st):
    if st == _lib.GZ_ERR_INVALID:
        raise ValueError("invalid argument to a verification kernel")
    if st != _lib.GZ_OK:
        raise RuntimeError("CUDA error in a verification kernel")


# ---- host special functions ------------------------------------------------------

def normal_cdf(x: float) -> float:
    """Phi(x) = erfc(-x / sqrt 2) / 2 (the reference's formula, stats.py:24-28)."""
    if not math.isfinite(x):
        raise ValueError(f"normal_cdf requires finite x, got {x}")
    return 0.5 * math.erfc(-x / _SQRT2)


def normal_quantile(p: float) -> float:
    """Phi^-1(p) by 200 bisection steps on [-40, 40] (stats.py:31-42)."""
    if not 0.0 < p < 1.0:
        raise ValueError(f"quantile requires 0 < p < 1, got {p}")
    lo, hi = -40.0, 40.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if normal_cdf(mid) < p:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def equal_probability_edges(bins: int) -> list:
    """Interior edges splitting the normal line into `bins` equal-mass bins (stats.py:356-360)."""
    if bins < 2:
        raise ValueError(f"need at least 2 bins, got {bins}")
    return [normal_quantile(j / bins) for j in range(1, bins)]


def chi_square_sf(statistic: float, dof: int) -> float:
    """P(X >= statistic) for X ~ chi^2(dof): the regularized upper incomplete gamma
    Q(dof/2, statistic/2), by series below s + 1 and a Lentz continued fraction above."""
    if dof < 1:
        raise ValueError(f"dof must be >= 1, got {dof}")
    if statistic < 0.0:
        raise ValueError(f"statistic must be >= 0, got {statistic}")
    s, x = 0.5 * dof, 0.5 * statistic
    if x == 0.0:
        return 1.0
    log_pref = -x + s * math.log(x) - math.lgamma(s)
    if x < s + 1.0:
        term = total = 1.0 / s
        a = s
        for _ in range(1000):
            a += 1.0
            term *= x / a
            total += term
            if abs(term) < abs(total) * 1e-17:
                break
        return max(0.0, 1.0 - total * math.exp(log_pref))
    tiny = 1e-300
    b = x + 1.0 - s
    c, d = 1.0 / tiny, 1.0 / b
    h = d
    for i in range(1, 1000):
        an = -i * (i - s)
        b += 2.0
        d = an * d + b
        d = tiny if abs(d) < tiny else d
        c = b + an / c
        c = tiny if abs(c) < tiny else c
        d = 1.0 / d
        h *= d * c
        if abs(d * c - 1.0) < 1e-17:
            break
    return h * math.exp(log_pref)


def _beta_continued_fraction(a: float, b: float, x: float) -> float:
    """The continued fraction of I_x(a, b) (modified Lentz evaluation)."""
    tiny = 1e-300
    apb, ap1, am1 = a + b, a + 1.0, a - 1.0
    c, d = 1.0, 1.0 - apb * x / ap1
    d = 1.0 / (tiny if abs(d) < tiny else d)
    h = d
    for m in range(1, 300):
        m2 = 2 * m
        for num in (m * (b - m) * x / ((am1 + m2) * (a + m2)),
                    -(a + m) * (apb + m) * x / ((a + m2) * (ap1 + m2))):
            d = 1.0 + num * d
            d = 1.0 / (tiny if abs(d) < tiny else d)
            c = 1.0 + num / c
            c = tiny if abs(c) < tiny else c
            h *= d * c
        if abs(d * c - 1.0) < 1e-16:
            break
    return h


def regularized_beta(a: float, b: float, x: float) -> float:
    """Regularized incomplete beta I_x(a, b) (the reference's stats.py:137-151 helper)."""
    if x <= 0.0:
        return 0.0
    if x >= 1.0:
        return 1.0
    front = math.exp(math.lgamma(a + b) - math.lgamma(a) - math.lgamma(b) + a * math.log(x) + b * math.log1p(-x))
    if x < (a + 1.0) / (a + b + 2.0):
        return front * _beta_continued_fraction(a, b, x) / a
    return 1.0 - front * _beta_continued_fraction(b, a, 1.0 - x) / b


def _as_device(x):
    """A float64 CUDA tensor view of x (CUDA tensors pass through; numpy arrays and
    sequences are copied to the device -- the statistics then run there)."""
    torch = _torch()
    if hasattr(x, "is_cuda") and x.is_cuda:
        return x
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")


@dataclass
class GofReport:
    statistic: float
    dof: int
    p_value: float

    def passes(self, alpha: float) -> bool:
        return self.p_value > alpha

    def verdict_at(self, alphas) -> dict:
        return {a: self.passes(a) for a in alphas}

    def to_json_dict(self, test: str, alpha: float, n: int, seed=None) -> dict:
        """stats.py:189-199 field layout."""
        return {"test": test, "statistic": self.statistic, "dof": self.dof, "p_value": self.p_value, "alpha": alpha,
                "verdict": "pass" if self.passes(alpha) else "fail", "n": n, "seed": seed}


@dataclass
class KsReport:
    d_statistic: float
    n: int

    def critical_value(self, alpha: float) -> float:
        return math.sqrt(-0.5 * math.log(alpha / 2.0)) / math.sqrt(self.n)

    def passes(self, alpha: float) -> bool:
        return self.d_statistic < self.critical_value(alpha)

    def to_json_dict(self, alpha: float, seed=None) -> dict:
        """stats.py:216-227 field layout."""
        return {"test": "ks", "statistic": self.d_statistic, "dof": None, "p_value": None,
                "critical_value": self.critical_value(alpha), "alpha": alpha,
                "verdict": "pass" if self.passes(alpha) else "fail", "n": self.n, "seed": seed}


# ---- device statistics --------------------------------------------------------------

def histogram(x, edges) -> np.ndarray:
    """Counts of x (float64 CUDA tensor) in the len(edges)+1 bins of the sorted interior
    edges, numpy.searchsorted(edges, x, side='right') semantics.  Exact."""
    torch = _torch()
    L = _lib.load()
    xs = _as_device(x).reshape(-1).contiguous()
    e = torch.tensor(sorted(float(v) for v in edges), dtype=torch.float64, device=xs.device)
    counts = torch.zeros(e.numel() + 1, dtype=torch.int64, device=xs.device)
    s = _stream(xs.device)
    _check(L.gz_hist_edges(_p(xs), xs.numel(), _p(e), e.numel(), _p(counts), s))
    return counts.cpu().numpy().astype(np.int64)


def chi_square_gof(x, bin_edges) -> GofReport:
    """Chi-square goodness of fit of x against N(0,1) over the given interior edges;
    adjacent bins merge left to right until each expected count is >= 5 (the
    reference's rule, stats.py:276-315)."""
    counts = histogram(x, bin_edges).astype(np.float64)
    n = float(counts.sum())
    edges = sorted(float(v) for v in bin_edges)
    probs = np.diff([0.0] + [normal_cdf(e) for e in edges] + [1.0])
    expected = probs * n
    mo, me = [], []
    ao = ae = 0.0
    for o, e in zip(counts, expected):
        ao += o
        ae += e
        if ae >= 5.0:
            mo.append(ao)
            me.append(ae)
            ao = ae = 0.0
    if ao > 0.0 or ae > 0.0:
        if me:
            mo[-1] += ao
            me[-1] += ae
        else:
            mo, me = [ao], [ae]
    if len(me) < 2:
        raise ValueError("fewer than 2 bins left after merging")
    stat = float(sum((o - e) ** 2 / e for o, e in zip(mo, me)))
    dof = len(me) - 1
    return GofReport(stat, dof, chi_square_sf(stat, dof))


def ks_test(x) -> KsReport:
    """Two-sided KS distance of x against N(0,1) (device sort + reduction)."""
    torch = _torch()
    L = _lib.load()
    xs = _as_device(x).reshape(-1).contiguous()
    d = torch.zeros(2, dtype=torch.float64, device=xs.device)
    _check(L.gz_ks_stat(_p(xs), xs.numel(), _p(d), _stream(xs.device)))
    dp, dm = d.cpu().tolist()
    return KsReport(max(dp, dm), xs.numel())


def moments(x):
    """MomentSummary of x (float64 CUDA tensor, or any float sequence) by device power sums
    (gz_moments_buffer): stats.py:232-259 conventions (unbiased variance,
    population excess kurtosis)."""
    torch = _torch()
    from .streams import summarize

    L = _lib.load()
    xs = _as_device(x).reshape(-1).contiguous()
    if xs.numel() < 4:
        raise ValueError(f"moments requires n >= 4, got {xs.numel()}")
    out5 = torch.empty(5, dtype=torch.float64, device=xs.device)
    _check(L.gz_moments_buffer(_p(xs), xs.numel(), _p(out5), _stream(xs.device)))
    return summarize(*out5.cpu().tolist())


def uniform_counts_gof(counts) -> GofReport:
    counts = np.asarray(counts, dtype=np.float64)
    total, cells = counts.sum(), counts.shape[0]
    if cells < 2 or total <= 0:
        raise ValueError("need >= 2 cells and a non-empty histogram")
    exp = total / cells
    stat = float(((counts - exp) ** 2 / exp).sum())
    return GofReport(stat, cells - 1, chi_square_sf(stat, cells - 1))


def low_bits_counts(u64, k_bits: int) -> np.ndarray:
    """Histogram of the low k bits of a u64 CUDA tensor (int64 container)."""
    torch = _torch()
    L = _lib.load()
    xs = u64.reshape(-1).contiguous()
    counts = torch.zeros(1 << k_bits, dtype=torch.int64, device=xs.device)
    _check(L.gz_lowbits_hist(_p(xs), xs.numel(), k_bits, _p(counts), _stream(xs.device)))
    return counts.cpu().numpy().astype(np.int64)


def low_bits_chi_square(source, k_bits: int, n: int) -> GofReport:
    """Frequency chi-square of the low k bits of the next n draws of `source`
    (advanced in place), stats.py:334-353."""
    torch = _torch()
    from . import engine

    if not 1 <= k_bits <= 8:
        raise ValueError(f"k_bits must be in 1..8, got {k_bits}")
    if n < 100 * (1 << k_bits):
        raise ValueError(f"need n >= {100 * (1 << k_bits)} draws for k={k_bits}, got {n}")
    buf = torch.empty(n, dtype=torch.int64, device="cuda")
    engine.fill_u64(source, buf)
    return uniform_counts_gof(low_bits_counts(buf, k_bits))
