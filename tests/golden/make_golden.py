#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the UNMODIFIED reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/gz_numba \
        python tests/golden/make_golden.py

Everything here goes through the reference's own public API
(`gausszig.make_source/make_sampler/engine.fill_gaussians/fill_u64`,
`build_ziggurat_tables`, `tables_to_json`, `moments`); the seeding conventions
for the five BASELINE.json configs are the ones pinned in SURVEY.md section 8d
and DESIGN.md.  The output pins the CPU oracle (oracle/gz_oracle.c, checked by
tests/test_oracle_golden.py) and, directly, the CUDA engine
(tests/test_gpu_parity.py).  Full outputs are recorded as sha256 digests plus
per-stream xor checksums, final states and a few leading values.
"""
import hashlib
import json
import os
import platform
import random
import subprocess
import sys

import numpy as np

import gausszig
from gausszig import engine, make_sampler, make_source, moments
from gausszig.sources import GOLDEN_GAMMA, MASK64, Lcg48, SplitMix64, mix64
from gausszig.tables import build_ziggurat_tables, tables_to_json

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def xor64(a):
    return "%016x" % int(np.bitwise_xor.reduce(bits(a))) if len(a) else "%016x" % 0


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hexs(a):
    return ["%016x" % int(v) for v in bits(a)]


def src_state(src):
    return {"state": "%016x" % src.state,
            "gamma": "%016x" % getattr(src, "gamma", 0)}


def host_info():
    info = {"python": platform.python_version(), "numpy": np.__version__,
            "gausszig": gausszig.__version__}
    try:
        info["glibc"] = subprocess.run(["ldd", "--version"], capture_output=True,
                                       text=True).stdout.splitlines()[0]
    except Exception:  # pragma: no cover
        info["glibc"] = "unknown"
    try:
        flags = open("/proc/cpuinfo").read()
        info["cpu_fma"] = " fma " in flags
        info["cpu_avx2"] = " avx2 " in flags
        model = [l for l in flags.splitlines() if l.startswith("model name")]
        info["cpu_model"] = model[0].split(":", 1)[1].strip() if model else "unknown"
    except Exception:  # pragma: no cover
        pass
    try:
        import numba
        info["numba"] = numba.__version__
    except Exception:  # pragma: no cover
        pass
    return info


def fill(alg, src, n):
    smp = make_sampler(alg)
    buf = np.empty(n, dtype=np.float64)
    engine.fill_gaussians(smp, src, buf)
    return buf, smp


# ---- seeding conventions for the configs ----------

def sm_output_seed(master, i):
    """i-th (0-based) output of SplitMix64(master): mix64(master + (i+1)*gamma)."""
    return mix64((master + (i + 1) * GOLDEN_GAMMA) & MASK64)


def main():
    g = {"meta": host_info()}

    # tables (tables.py:107-131), JSON wire format (tables.py:156-183)
    g["tables"] = {str(n): tables_to_json(build_ziggurat_tables(n)) for n in (8, 16, 32, 64, 128, 256, 512, 1024)}

    # source digests (tests/test_sources.py:9-10) and first outputs
    d = {}
    for sid in ("lcg48", "splitmix"):
        s = make_source(sid, 12345)
        acc = 0
        for _ in range(10_000):
            acc ^= s.next_u64()
        d[sid + "_xor1e4_12345"] = "%016x" % acc
        s = make_source(sid, 0)
        d[sid + "_first8_seed0"] = ["%016x" % s.next_u64() for _ in range(8)]
    g["digests"] = d

    # fill_u64 (engine.py:224-232), tests/test_engine.py:31-40 shape
    g["u64"] = {}
    for sid in ("lcg48", "splitmix"):
        src = make_source(sid, 99)
        buf = np.empty(100_000, dtype=np.uint64)
        engine.fill_u64(src, buf)
        g["u64"][sid] = {"seed": 99, "n": 100_000, "sha256": sha(buf), "first": ["%016x" % int(v) for v in buf[:8]],
                         "xor": "%016x" % int(np.bitwise_xor.reduce(buf)), **src_state(src)}

    # the six pairings at seed 424242, n = 300 000 (tests/test_engine.py:16-28)
    g["pairings"] = []
    for sid in ("lcg48", "splitmix"):
        for alg in ("polar", "ziggurat", "modified-ziggurat"):
            src = make_source(sid, 424242)
            buf, smp = fill(alg, src, 300_000)
            rec = {"source": sid, "sampler": alg, "seed": 424242, "n": 300_000, "sha256": sha(buf),
                   "xor": xor64(buf), "first": hexs(buf[:16]), "last": hexs(buf[-4:]), **src_state(src)}
            if alg == "polar":
                rec["spare"] = None if smp.spare is None else "%016x" % int(bits(np.array([smp.spare]))[0])
            g["pairings"].append(rec)

    # small/edge cases with full outputs (n = 0, 1, odd sizes, many seeds)
    g["small"] = []
    rnd = random.Random(20240529)
    for sid in ("lcg48", "splitmix"):
        for alg in ("polar", "ziggurat", "modified-ziggurat"):
            for n in (0, 1, 2, 3, 31, 32, 33, 127, 128, 129, 1000):
                seed = rnd.getrandbits(64)
                src = make_source(sid, seed)
                buf, smp = fill(alg, src, n)
                rec = {"source": sid, "sampler": alg, "seed": "%x" % seed, "n": n, "out": hexs(buf),
                       **src_state(src)}
                if alg == "polar":
                    rec["spare"] = None if smp.spare is None else "%016x" % int(bits(np.array([smp.spare]))[0])
                g["small"].append(rec)

    # polar spare hand-off across odd batches (tests/test_engine.py:58-71)
    smp = make_sampler("polar")
    src = make_source("lcg48", 3)
    chunks = []
    for size in (101, 57, 42):
        buf = np.empty(size)
        engine.fill_gaussians(smp, src, buf)
        chunks.append(buf)
    allv = np.concatenate(chunks)
    g["polar_chunks"] = {"seed": 3, "source": "lcg48", "sizes": [101, 57, 42], "out": hexs(allv),
                         "spare": None if smp.spare is None else "%016x" % int(bits(np.array([smp.spare]))[0]),
                         **src_state(src)}

    # ---- configs ------------------------------------------------------------
    cfg = {}
    # C1: ziggurat x SplitMix64, 1024 streams seeded by SplitMix64(42)'s outputs, 4096 each
    out = np.empty((1024, 4096))
    states = []
    for i in range(1024):
        src = SplitMix64(sm_output_seed(42, i))
        buf, _ = fill("ziggurat", src, 4096)
        out[i] = buf
        states.append("%016x" % src.state)
    cfg["c1"] = {"sha256": sha(out), "xor": [xor64(out[i]) for i in range(1024)], "state": states,
                 "first": hexs(out[:4, 0]), "stream0_first8": hexs(out[0, :8])}

    def sample_ids(total, k, seed):
        r = random.Random(seed)
        ids = {0, 1, 2, 31, 32, 33, total // 2, total - 2, total - 1}
        while len(ids) < k:
            ids.add(r.randrange(total))
        return sorted(ids)

    # C2: polar x Lcg48(7 + s), 2^20 streams x 256
    recs = []
    for s in sample_ids(1 << 20, 48, 2):
        src = Lcg48(7 + s)
        buf, smp = fill("polar", src, 256)
        recs.append({"id": s, "xor": xor64(buf), "state": "%016x" % src.state, "first": hexs(buf[:4]),
                     "spare": None if smp.spare is None else "%016x" % int(bits(np.array([smp.spare]))[0])})
    cfg["c2"] = recs
    # C3: modified ziggurat x SplitMix64(mix64(1234 + (s+1) gamma)), 2^20 x 1024
    recs = []
    for s in sample_ids(1 << 20, 48, 3):
        src = SplitMix64(sm_output_seed(1234, s))
        buf, _ = fill("modified-ziggurat", src, 1024)
        recs.append({"id": s, "xor": xor64(buf), "state": "%016x" % src.state, "first": hexs(buf[:4])})
    cfg["c3"] = recs
    # C4: ziggurat x Lcg48(99 + gid), gid in [0, 2^25), 256 each; plus moments of a block
    recs = []
    for s in sample_ids(1 << 25, 48, 4) + [1 << 22, (1 << 22) - 1, 3 << 22]:
        src = Lcg48(99 + s)
        buf, _ = fill("ziggurat", src, 256)
        recs.append({"id": s, "xor": xor64(buf), "state": "%016x" % src.state, "first": hexs(buf[:4])})
    cfg["c4"] = recs
    blk = np.empty((4096, 256))
    for s in range(4096):
        blk[s], _ = fill("ziggurat", Lcg48(99 + s), 256)
    ms = moments(blk.reshape(-1).tolist())
    cfg["c4_moments_first4096"] = {"n": ms.n, "mean": ms.mean.hex(), "variance": ms.variance.hex(),
                                   "skewness": ms.skewness.hex(), "excess_kurtosis": ms.excess_kurtosis.hex(),
                                   "xor_all": xor64(blk.reshape(-1)), "sha256": sha(blk)}
    # C5: x[i,g] = -5 + 10*u over SplitMix64(2024) row-major; sigma_i = 10**(-3 + 3*u) from the
    # same stream after all 65536*1024 genes; x += sigma_i * z with the original ziggurat over
    # SplitMix64(i ^ 0xC0FFEE), generation t using variates [1024 t, 1024 (t+1)).
    n_ind, n_genes = 65536, 1024
    recs = []
    zig = make_sampler("ziggurat")
    for i in (0, 1, 2, 8191, 8192, 40000, 65535):
        x = np.empty(n_genes)
        for gidx in range(n_genes):
            idx = i * n_genes + gidx
            u = SplitMix64((2024 + idx * GOLDEN_GAMMA) & MASK64).next_f64_unit()
            x[gidx] = -5.0 + 10.0 * u
        u = SplitMix64((2024 + (n_ind * n_genes + i) * GOLDEN_GAMMA) & MASK64).next_f64_unit()
        sigma = 10.0 ** (-3.0 + 3.0 * u)
        rec = {"id": i, "x0_sha256": sha(x), "x0_first": hexs(x[:4]), "sigma": sigma.hex(), "gens": []}
        src = SplitMix64(i ^ 0xC0FFEE)
        smp = make_sampler("ziggurat")
        for t in range(3):
            for gidx in range(n_genes):
                x[gidx] = gausszig.gaussian_affine(src, smp, float(x[gidx]), sigma)
            rec["gens"].append({"sha256": sha(x), "xor": xor64(x), "first": hexs(x[:4]),
                                "state": "%016x" % src.state})
        recs.append(rec)
    cfg["c5"] = recs
    g["configs"] = cfg

    # statistical gates (stats.py) on a known deviate buffer
    from gausszig import stats as S
    st = {"edges10": [v.hex() for v in S.equal_probability_edges(10)],
          "edges100": [v.hex() for v in S.equal_probability_edges(100)],
          "normal_cdf": {repr(x): S.normal_cdf(x).hex() for x in (-3.0, -0.5, 0.0, 1.7)},
          "chi_square_sf": [[x, k, S.chi_square_sf(x, k).hex()] for x, k in
                            ((3.0, 4), (50.0, 40), (120.5, 99), (0.5, 1), (250.0, 199), (30.0, 7))]}
    buf, _ = fill("ziggurat", make_source("lcg48", 424242), 300_000)
    gr = S.chi_square_gof(buf, S.equal_probability_edges(100))
    kr = S.ks_test(buf)
    st["gof_zig_lcg_424242"] = {"statistic": gr.statistic.hex(), "dof": gr.dof, "p_value": gr.p_value.hex(),
                                "ks_d": kr.d_statistic.hex(), "n": kr.n}
    for sid in ("lcg48", "splitmix"):
        r = S.low_bits_chi_square(make_source(sid, 5), 4, 100_000)
        st["lowbits_" + sid] = {"seed": 5, "k": 4, "n": 100_000, "statistic": r.statistic.hex(), "dof": r.dof}
    g["stats"] = st

    # bench checksum witness (bench.py:209-216): xor fold of WITNESS_OPS deviates of one fresh stream
    from gausszig import bench as B
    wit = {}
    for seed in (0x5EEDBA5E, 60):
        for sid in ("lcg48", "splitmix"):
            for alg in ("polar", "ziggurat", "modified-ziggurat"):
                buf, _ = fill(alg, make_source(sid, seed), B.WITNESS_OPS)
                wit["%s/%s/%d" % (sid, alg, seed)] = "%016x" % B._checksum_fold(buf)
    g["bench_witness"] = wit

    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
