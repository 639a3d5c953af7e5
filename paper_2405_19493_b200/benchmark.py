"""Benchmark harness with the reference's result schema, timing the B200 engine.

Mirrors /root/reference/pkg/src/gausszig/bench.py for the CUDA engine
(SURVEY 8f row 2): `run_benchmark(sampler_id, source_id, cfg)` returns a
`BenchResult` with the same fields (ns_per_op, ci_half_width,
per_iteration_ns_per_op, ops_total, checksum, seed, confidence, engine_used)
and `render_table` prints them as markdown / CSV / JSON in the reference's
formats, so GPU rows sit beside the paper's Table-3 CPU rows.

Differences by design: one "op" is one N(0,1) deviate; on the GPU the
deviates of an iteration come from `streams` independent streams at once
(seeded like the reference's source from `seed + stream id` / the stream id's
SplitMix64 output), timed with CUDA events.  The checksum witness is the
reference's: the xor fold (bench.py:174-175) of the first WITNESS_OPS deviates
of ONE stream seeded `seed`, so it equals the reference's BenchResult.checksum.
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field

import numpy as np

from . import engine
from .samplers import make_sampler, require_sanctioned
from .sources import make_source

BATCH_OPS = 1 << 17
WITNESS_OPS = 1 << 20
DEFAULT_SEED = 0x5EEDBA5E


@dataclass
class BenchConfig:
    warmup_iters: int = 3
    measure_iters: int = 10
    streams: int = 1 << 14       # independent streams per iteration
    per_stream: int = 256        # deviates per stream per iteration
    seed: int = DEFAULT_SEED
    confidence: float = 0.999
    # "streams": `streams` x `per_stream` deviates per iteration from independent streams;
    # "single": the reference's own call shape (bench.py:199-203) -- one source,
    # engine.fill_gaussians of `per_stream` deviates per call into a device buffer,
    # state carried from call to call, per-call overhead included
    layout: str = "streams"

    def __post_init__(self):
        if self.measure_iters < 2:
            raise ValueError("need at least 2 measurement iterations for a CI")
        if self.warmup_iters < 0:
            raise ValueError("warmup_iters must be >= 0")
        if self.streams < 1 or self.per_stream < 1:
            raise ValueError("streams and per_stream must be >= 1")
        if not 0.0 < self.confidence < 1.0:
            raise ValueError("confidence must be in (0, 1)")
        if self.layout not in ("streams", "single"):
            raise ValueError(f"unknown layout: {self.layout!r}")

    @classmethod
    def paper(cls, seed: int = DEFAULT_SEED) -> "BenchConfig":
        return cls(warmup_iters=5, measure_iters=20, streams=1 << 20, per_stream=256, seed=seed)

    @classmethod
    def smoke(cls, seed: int = DEFAULT_SEED) -> "BenchConfig":
        return cls(warmup_iters=1, measure_iters=3, streams=1 << 12, seed=seed)

    @classmethod
    def single(cls, seed: int = DEFAULT_SEED, batch: int = BATCH_OPS) -> "BenchConfig":
        """The reference harness's exact call shape: one stream, `batch` deviates per call."""
        return cls(warmup_iters=3, measure_iters=10, streams=1, per_stream=batch, seed=seed, layout="single")


@dataclass
class BenchResult:
    sampler_id: str
    source_id: str
    ns_per_op: float
    ci_half_width: float
    per_iteration_ns_per_op: list = field(default_factory=list)
    ops_total: int = 0
    checksum: int = 0
    seed: int = DEFAULT_SEED
    confidence: float = 0.999
    engine_used: str = "cuda"

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass
class ComparisonRow:
    """Percent-faster relation between two results on the same source (bench.py:106-115)."""

    baseline: BenchResult
    candidate: BenchResult
    percent_faster: float = field(init=False)

    def __post_init__(self):
        self.percent_faster = percent_faster(self.baseline.ns_per_op, self.candidate.ns_per_op)


def checksum_fold(buf) -> int:
    """xor of the raw 64-bit patterns (bench.py:174-175)."""
    a = np.ascontiguousarray(buf, dtype=np.float64)
    return int(np.bitwise_xor.reduce(a.view(np.uint64))) if a.size else 0


def student_t_quantile(confidence: float, dof: int) -> float:
    """Two-sided Student-t quantile (bench.py:118-140): bisection of the t survival
    function 0.5 * I_{dof/(dof+t^2)}(dof/2, 1/2)."""
    from .verify import regularized_beta

    if not 0.0 < confidence < 1.0:
        raise ValueError(f"confidence must be in (0, 1), got {confidence}")
    if dof < 1:
        raise ValueError(f"dof must be >= 1, got {dof}")
    tail = 0.5 * (1.0 - confidence)
    lo, hi = 0.0, 1e8
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if 0.5 * regularized_beta(0.5 * dof, 0.5, dof / (dof + mid * mid)) > tail:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def confidence_interval(xs, level: float):
    """Two-sided Student-t interval (lo, hi) of the mean of xs (bench.py:143-152)."""
    xs = list(xs)
    n = len(xs)
    if n < 2:
        raise ValueError(f"confidence interval needs n >= 2, got {n}")
    mean = sum(xs) / n
    var = sum((x - mean) ** 2 for x in xs) / (n - 1)
    half = student_t_quantile(level, n - 1) * math.sqrt(var / n)
    return mean - half, mean + half


def percent_faster(baseline_ns: float, candidate_ns: float) -> float:
    """How much faster the candidate is than the baseline, in percent (bench.py:155-160)."""
    if baseline_ns <= 0.0 or candidate_ns <= 0.0:
        raise ValueError("ns/op inputs must be positive")
    return 100.0 * (1.0 - candidate_ns / baseline_ns)


def run_benchmark(sampler_id: str, source_id: str, cfg: BenchConfig | None = None) -> BenchResult:
    import torch

    from . import streams as S

    cfg = cfg or BenchConfig()
    require_sanctioned(source_id, sampler_id)
    # witness: the reference's checksum of one stream's first WITNESS_OPS deviates
    witness = np.empty(WITNESS_OPS)
    engine.fill_gaussians(make_sampler(sampler_id), make_source(source_id, cfg.seed), witness)
    checksum = checksum_fold(witness)
    if cfg.layout == "single":
        return _run_single(sampler_id, source_id, cfg, checksum)
    # many independent streams per iteration
    scheme = "lcg_master_plus_id" if source_id == "lcg48" else "sm_output_of_master"
    st = S.seed_streams(scheme, cfg.seed, 0, cfg.streams)
    out = torch.empty((cfg.streams, cfg.per_stream), dtype=torch.float64, device="cuda")
    kw = {}
    if sampler_id == "polar":
        kw = dict(spare=torch.zeros(cfg.streams, dtype=torch.float64, device="cuda"),
                  has_spare=torch.zeros(cfg.streams, dtype=torch.uint8, device="cuda"))
    smp = make_sampler(sampler_id)
    for _ in range(cfg.warmup_iters):
        S.fill_gaussians_streams(smp, source_id, st, out, sync=False, **kw)
    S.engine_check()
    per_iter = []
    ops = cfg.streams * cfg.per_stream
    for _ in range(cfg.measure_iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.fill_gaussians_streams(smp, source_id, st, out, sync=False, **kw)
        e1.record()
        e1.synchronize()
        per_iter.append(e0.elapsed_time(e1) * 1e6 / ops)
    S.engine_check()
    lo, hi = confidence_interval(per_iter, cfg.confidence)
    return BenchResult(sampler_id, source_id, sum(per_iter) / len(per_iter), 0.5 * (hi - lo), per_iter,
                       ops * cfg.measure_iters, checksum, cfg.seed, cfg.confidence, "cuda")


def _run_single(sampler_id: str, source_id: str, cfg: BenchConfig, checksum: int) -> BenchResult:
    """bench.py:217-244 on the GPU: fresh seed-determined stream, fills of per_stream
    deviates per call through engine.fill_gaussians (device buffer), CUDA-event timed."""
    import torch

    buf = torch.empty(cfg.per_stream, dtype=torch.float64, device="cuda")
    smp, src = make_sampler(sampler_id), make_source(source_id, cfg.seed)
    for _ in range(cfg.warmup_iters):
        engine.fill_gaussians(smp, src, buf)
    smp, src = make_sampler(sampler_id), make_source(source_id, cfg.seed)
    per_iter = []
    for _ in range(cfg.measure_iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        engine.fill_gaussians(smp, src, buf)
        e1.record()
        e1.synchronize()
        per_iter.append(e0.elapsed_time(e1) * 1e6 / cfg.per_stream)
    lo, hi = confidence_interval(per_iter, cfg.confidence)
    return BenchResult(sampler_id, source_id, sum(per_iter) / len(per_iter), 0.5 * (hi - lo), per_iter,
                       cfg.per_stream * cfg.measure_iters, checksum, cfg.seed, cfg.confidence, "cuda")


_CSV_HEADER = "source,sampler,ns_per_op,ci_half_width,iters,ops_total,seed"


def render_table(rows, fmt: str) -> str:
    """markdown (sources x samplers), csv or json -- the reference's formats (bench.py:263-300)."""
    rows = list(rows)
    if not rows:
        raise ValueError("no benchmark results to render")
    if fmt == "json":
        return json.dumps([r.to_dict() for r in rows], indent=2)
    if fmt == "csv":
        return "\n".join([_CSV_HEADER] + [
            f"{r.source_id},{r.sampler_id},{r.ns_per_op:.3f},{r.ci_half_width:.3f},"
            f"{len(r.per_iteration_ns_per_op)},{r.ops_total},{r.seed}" for r in rows])
    if fmt == "md":
        samplers = list(dict.fromkeys(r.sampler_id for r in rows))
        sources = list(dict.fromkeys(r.source_id for r in rows))
        cell = {(r.source_id, r.sampler_id): r for r in rows}
        lines = ["| PRNG | " + " | ".join(samplers) + " |", "|---" * (len(samplers) + 1) + "|"]
        for src in sources:
            cells = [f"{cell[(src, s)].ns_per_op:.4f} ± {cell[(src, s)].ci_half_width:.4f} ns/op"
                     if (src, s) in cell else "n/a" for s in samplers]
            lines.append("| " + src + " | " + " | ".join(cells) + " |")
        return "\n".join(lines)
    raise ValueError(f"unknown table format: {fmt!r}")


def main(argv=None) -> int:
    import argparse

    ap = argparse.ArgumentParser(description="B200 engine benchmark in the reference's Table-3 layout")
    ap.add_argument("--format", default="md", choices=["md", "csv", "json"])
    ap.add_argument("--seed", type=lambda v: int(v, 0), default=DEFAULT_SEED)
    ap.add_argument("--smoke", action="store_true")
    ap.add_argument("--layout", default="streams", choices=["streams", "single"])
    args = ap.parse_args(argv)
    if args.layout == "single":
        cfg = BenchConfig.single(args.seed)
    else:
        cfg = BenchConfig.smoke(args.seed) if args.smoke else BenchConfig(seed=args.seed)
    rows = [run_benchmark(alg, src, cfg) for src in ("lcg48", "splitmix")
            for alg in ("polar", "ziggurat", "modified-ziggurat") if (src, alg) != ("lcg48", "modified-ziggurat")]
    print(render_table(rows, args.format))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
