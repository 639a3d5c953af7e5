#!/usr/bin/env python3
"""Benchmark of the B200 Gaussian variate engine (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload = BASELINE.json configs[1] (config 2): the polar method over
the 48-bit Java LCG, 2^20 independent streams seeded Lcg48(7 + stream id), 256
fp64 variates per stream per step, per GPU (weak scaling: rank r owns stream
ids [r*2^20, (r+1)*2^20)).  One step = every stream emits its next 256 variates
(the streams continue from step to step).  The output (2 GiB per GPU) is
larger than L2, so no flush is needed between steps.

value   = variates/s over all ranks (device time, CUDA events, max over ranks)
e2e     = the same work through the reference-facing host-buffer C-ABI call
          (gz_fill_gaussians_host): stream states in from pinned host memory,
          deviates and states back to pinned host memory, every step.
roofline= HBM-store bound of the fill kernel (8 B per variate) against the
          measured copy bandwidth of MEASURED_PEAKS.json.
cpu_baseline = the CPU oracle port (oracle/gz_oracle.c, OpenMP over streams)
          on a bounded sample of the same workload, rank 0, N=1 only.
Also reported under "configs": the other four BASELINE configs (device time).

--impl reference: the reference algorithm's CPU implementation (the oracle
port; the Python reference cannot travel to the GPU box) on all host threads,
same metric and config, one bounded sample per step.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

STREAMS_PER_GPU = 1 << 20
N_PER = 256
METRIC = "fp64 Gaussian variates/sec (polar x LCG48, config 2)"
UNIT = "variates/s"
REF_SAMPLE_STREAMS = 1 << 17     # CPU sample per step: 2^17 streams x 256 = 33.5M variates


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_record(cfg):
    """dram read + write bytes per launch of the headline kernel, from the committed
    `ncu --set full` capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f).get(cfg)
        return None if rec is None else rec["bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 6 for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_setup(n_gpus):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch

    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        torch.cuda.synchronize()


def time_fill(cfg, first_id, n_streams, steps, warmup, world, checks=False):
    """Device-timed steps of one config's fill on this rank.  Returns dict."""
    import torch

    from paper_2405_19493_b200 import streams

    c = streams.CONFIGS[cfg]
    st = streams.config_states(cfg, first_id, n_streams)
    out = torch.empty((n_streams, c.n_per), dtype=torch.float64, device="cuda")
    kw = {}
    if c.sampler == "polar":
        kw = dict(spare=torch.zeros(n_streams, dtype=torch.float64, device="cuda"),
                  has_spare=torch.zeros(n_streams, dtype=torch.uint8, device="cuda"))
    ck = ps = None
    if checks:
        ck = torch.zeros(n_streams, dtype=torch.int64, device="cuda")
        ps = torch.zeros((n_streams, 4), dtype=torch.float64, device="cuda")
    for _ in range(warmup):
        streams.fill_gaussians_streams(c.sampler, c.source, st, out, checksum=ck, psum=ps, sync=False, **kw)
    streams.engine_check()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        streams.fill_gaussians_streams(c.sampler, c.source, st, out, checksum=ck, psum=ps, sync=False, **kw)
    e1.record()
    e1.synchronize()
    streams.engine_check()
    ms = e0.elapsed_time(e1) / steps
    res = {"ms_per_step": ms, "variates_per_step": n_streams * c.n_per, "launches": steps}
    if checks:
        res["checksum"] = ck
        res["psum"] = ps
    del out
    return res


def time_mutate(first_ind, n_ind, generations, steps, warmup, world):
    import torch

    from paper_2405_19493_b200 import streams

    x, sigma = streams.init_population(n_ind, 1024, seed=2024, first_ind=first_ind, total_ind=65536)
    st = streams.config_states("c5", first_ind, n_ind)
    for _ in range(warmup):
        streams.mutate(st, x, sigma, generations, sync=False)
    streams.engine_check()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        streams.mutate(st, x, sigma, generations, sync=False)
    e1.record()
    e1.synchronize()
    streams.engine_check()
    return {"ms_per_step": e0.elapsed_time(e1) / steps, "variates_per_step": n_ind * 1024 * generations,
            "launches": steps}


# the polar x LCG48 path is bounded by HBM stores (8 B/variate), the
# integer pipe and (for polar) the FP64 pipe.  Algorithmic operations per variate:
#   int : 1.2725 u64/variate x ~10 SASS int ops per LCG48 u64 (2 x mul-add + shifts)
#         + ~10 for extraction / compare / conversion                      = 22.7
#   fp64: per attempt (0.6363/variate) 2 x (int->f64, 2u-1) + s (3) + 2 compares = 9;
#         per pair (0.5/variate) glibc log table path 15, -2*log 1, divide 8,
#         square root 9, the two products 2                                 = 35
#         -> 0.6363 * 9 + 0.5 * 35                                          = 23.2
# Pipe rates per SM per clock: int32 64 (CUDA throughput table, cc 10.0); FP64 62
# (measured, tools/calib/calib_pipes.cu).  Clock: the median sampled under load.
INT_OPS_PER_VARIATE = 22.7
FP64_OPS_PER_VARIATE = 23.2
INT_OPS_PER_SM_CLK = 64
FP64_OPS_PER_SM_CLK = 62


def compute_bounds(variates_per_s, hbm_gbs, clocks):
    import torch

    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    hz = mhz * 1e6
    b = {"hbm": hbm_gbs * 1e9 / 8, "int": sms * hz * INT_OPS_PER_SM_CLK / INT_OPS_PER_VARIATE,
         "fp64": sms * hz * FP64_OPS_PER_SM_CLK / FP64_OPS_PER_VARIATE}
    lim = min(b, key=b.get)
    out = {"unit": "variates/s", "sm_mhz": mhz, "sms": sms, **b, "min": lim,
           "frac_of_min": variates_per_s / b[lim]}
    # the bound the headline kernel actually meets: instruction issue (4 warp-instructions
    # per SM clock) at the warp-instruction count ncu measured per launch
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            rec = json.load(f)["c2"]
        wipv = rec["warp_instructions_per_launch"] / rec["variates_per_launch"]
        ceiling = sms * hz * 4 / wipv
        out["issue"] = {"warp_instr_per_variate": wipv, "ceiling": ceiling, "frac": variates_per_s / ceiling,
                        "source": rec["source"]}
    except Exception:
        pass
    return out


def e2e_host(first_id, n_streams, steps, warmup):
    """Reference-facing path: host buffers through gz_fill_gaussians_host."""
    import ctypes

    import numpy as np

    from paper_2405_19493_b200 import _lib

    L = _lib.load()
    pin = []

    def pinned(nbytes):
        p = ctypes.c_void_p()
        _lib.check(L.gz_host_alloc(ctypes.byref(p), nbytes))
        pin.append(p)
        return p

    n_out = n_streams * N_PER
    p_out, p_st_in, p_st_out = pinned(n_out * 8), pinned(n_streams * 8), pinned(n_streams * 8)
    p_sp, p_hs = pinned(n_streams * 8), pinned(n_streams)
    st_in = np.frombuffer((ctypes.c_uint64 * n_streams).from_address(p_st_in.value), dtype=np.uint64)
    st_out = np.frombuffer((ctypes.c_uint64 * n_streams).from_address(p_st_out.value), dtype=np.uint64)
    ids = np.arange(first_id, first_id + n_streams, dtype=np.uint64)
    st_in[:] = ((np.uint64(7) + ids) ^ np.uint64(0x5DEECE66D)) & np.uint64((1 << 48) - 1)

    def step():
        _lib.check(L.gz_fill_gaussians_host(0, 0, 0, n_streams, N_PER, p_st_in, p_st_out, None, None, p_sp, p_hs,
                                            p_out, None, 1_000_000))
        st_in[:] = st_out   # the streams continue (host-side hand-off, like the reference's write-back)

    for _ in range(warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t0) / steps
    for p in pin:
        L.gz_host_free(p)
    return {"s_per_step": dt, "h2d": n_streams * 8, "d2h": n_out * 8 + n_streams * 8 + n_streams * 9}


def cpu_reference(n_streams, steps, warmup, first_id=0):
    """The reference algorithm on the host cores (oracle port, OpenMP)."""
    import numpy as np

    from oracle import gz_oracle as O

    O.lib()
    threads = os.cpu_count() or 1
    st = np.array([O.lcg_state(7 + i) for i in range(first_id, first_id + n_streams)], dtype=np.uint64)
    for _ in range(warmup):
        out, st, *_ = O.fill_gaussians("polar", "lcg48", st, N_PER, nthreads=threads)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out, st, sp, hs, status = O.fill_gaussians("polar", "lcg48", st, N_PER, nthreads=threads)
        ts.append(time.perf_counter() - t0)
        assert status == 0
    dt = statistics.median(ts)
    return {"value": n_streams * N_PER / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{n_streams} streams x {N_PER} variates of config 2 (polar x Lcg48(7+id)) per step, "
                      f"median of {steps} steps, OpenMP over streams on {threads} threads"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cb = cpu_reference(REF_SAMPLE_STREAMS, max(1, args.steps), max(1, min(args.warmup, 1)))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded streams)",
            "config": {"workload": "config 2: polar x LCG48, 2^20 streams x 256 per GPU", "streams": REF_SAMPLE_STREAMS,
                       "n_per": N_PER, "sample": "bounded CPU sample (see cpu_baseline.sample)"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}, "world_size": world}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the other four configs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(3, args.warmup)

    import torch

    world, rank, local = dist_setup(args.gpus)
    hbm_peak, peak_kind = peaks()

    # ---- headline: config 2 on every rank (weak scaling) ----
    first = rank * STREAMS_PER_GPU
    with ClockSampler(local) as clk:
        time.sleep(0.3)   # let nvidia-smi start sampling before the timed region
        r = time_fill("c2", first, STREAMS_PER_GPU, args.steps, args.warmup, world)
    ms = allmax(r["ms_per_step"], world)
    value = world * r["variates_per_step"] / (ms / 1e3)
    clocks = clk.summary()
    kernel_bytes = r["variates_per_step"] * 8
    achieved = kernel_bytes / (r["ms_per_step"] / 1e3) / 1e9

    # ---- e2e through the host-buffer C-ABI call ----
    e = e2e_host(first, STREAMS_PER_GPU, max(3, min(10, args.steps // 10)), 1)
    e_s = allmax(e["s_per_step"] * 1e3, world) / 1e3
    e2e = {"value": world * STREAMS_PER_GPU * N_PER / e_s, "unit": UNIT, "h2d_bytes_per_step": e["h2d"],
           "d2h_bytes_per_step": e["d2h"], "s_per_step": e_s}

    # ---- the other configs (device time) ----
    extra = {}
    launches = r["launches"]
    if not args.no_extra:
        c1 = time_fill("c1", 0, 1024, max(100, args.steps), args.warmup, world)
        extra["c1"] = {"value": world * c1["variates_per_step"] / (allmax(c1["ms_per_step"], world) / 1e3),
                       "ms_per_step": c1["ms_per_step"], "shape": "1024 x 4096 per GPU"}
        n3 = (1 << 20) // world
        c3 = time_fill("c3", rank * n3, n3, max(5, args.steps // 10), args.warmup, world)
        extra["c3"] = {"value": world * c3["variates_per_step"] / (allmax(c3["ms_per_step"], world) / 1e3),
                       "ms_per_step": c3["ms_per_step"], "shape": f"2^20 x 1024 box-wide, {n3} streams per GPU"}
        c4 = time_fill("c4", rank * (1 << 22), 1 << 22, max(5, args.steps // 10), args.warmup, world, checks=True)
        extra["c4"] = {"value": world * c4["variates_per_step"] / (allmax(c4["ms_per_step"], world) / 1e3),
                       "ms_per_step": c4["ms_per_step"], "shape": "2^22 x 256 per GPU, fused checksum + moments"}
        from paper_2405_19493_b200 import streams

        cen = streams.central_from_psum(c4["psum"], 256)
        xr = streams.xor_fold(c4["checksum"])
        if world > 1:
            from paper_2405_19493_b200 import dist as gzdist

            merged = gzdist.gather_moments(cen)
            xr = gzdist.gather_xor(xr)
        else:
            merged = tuple(cen.cpu().tolist())
        m = streams.summarize(*merged)
        extra["c4"]["moments"] = {"n": m.n, "mean": m.mean, "variance": m.variance, "excess_kurtosis": m.excess_kurtosis}
        extra["c4"]["xor_all_streams"] = "%016x" % (xr & ((1 << 64) - 1))
        del c4
        n5 = 65536 // world
        c5 = time_mutate(rank * n5, n5, 10, max(3, args.steps // 20), args.warmup, world)
        extra["c5"] = {"value": world * c5["variates_per_step"] / (allmax(c5["ms_per_step"], world) / 1e3),
                       "ms_per_step": c5["ms_per_step"],
                       "shape": f"65536 x 1024 genes box-wide ({n5} per GPU), 10 generations per step"}
        torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_reference(REF_SAMPLE_STREAMS, 3, 1)

    barrier(world)
    if rank == 0:
        tr = traffic_record("c2")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PRNG streams)",
            "config": {"workload": "config 2: polar x LCG48, 2^20 streams x 256 variates per GPU per step",
                       "streams_per_gpu": STREAMS_PER_GPU, "n_per": N_PER, "seed": "Lcg48(7 + stream id)",
                       "l2": "output 2 GiB per step > 126 MB L2 (no flush needed)", "parallelism": f"streams/{world}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": tr, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": kernel_bytes,
                         "compute_bounds": compute_bounds(r["variates_per_step"] / (r["ms_per_step"] / 1e3),
                                                          hbm_peak, clocks)},
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "configs": extra,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
