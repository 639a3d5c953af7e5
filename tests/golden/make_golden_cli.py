#!/usr/bin/env python3
"""Generate tests/golden/golden_cli.json from the UNMODIFIED reference package:
layer-occupancy runs (samplers.py:89-93, 138-142 sample_with_occupancy) and the
stdout of the reference CLI (cli.py) for `sample`, `tables` and `bits`.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/gz_numba \
        python tests/golden/make_golden_cli.py
"""
import contextlib
import io
import json
import os
import sys

import numpy as np

import math

from gausszig import ScriptedSource, ScriptExhausted, SplitMix64, bench, build_ziggurat_tables, cli, make_sampler, make_source
from gausszig.samplers import tail_sample
from gausszig.stats import regularized_beta

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_cli.json")

SAMPLE_ARGS = [
    ["sample", "--source", "lcg48", "--sampler", "polar", "--n", "25", "--seed", "7"],
    ["sample", "--source", "splitmix", "--sampler", "ziggurat", "--n", "40", "--seed", "0x1234"],
    ["sample", "--source", "splitmix", "--sampler", "modified-ziggurat", "--n", "33", "--seed", "99",
     "--mu", "1.5", "--sigma", "0.25"],
    ["sample", "--source", "lcg48", "--sampler", "ziggurat", "--n", "0"],
    ["tables", "--n", "64"],
    ["bits", "--source", "splitmix", "--k", "3", "--n", "20000", "--seed", "9"],
    ["bits", "--source", "lcg48", "--k", "5", "--n", "50000", "--seed", "11"],
    ["sample", "--source", "lcg48", "--sampler", "modified-ziggurat", "--n", "4"],
    ["verify", "--source", "lcg48", "--sampler", "modified-ziggurat", "--n", "20000"],
    ["tables", "--n", "6"],
]


def run_cli(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return {"argv": argv, "code": code, "stdout": out.getvalue()}


def main():
    g = {"occupancy": [], "cli": []}
    for sid in ("lcg48", "splitmix"):
        for alg in ("ziggurat", "modified-ziggurat"):
            for seed in (0x5EEDBA5E, 77):
                src = make_source(sid, seed)
                vals, counts = make_sampler(alg).sample_with_occupancy(src, 5000)
                buf = np.array(vals, dtype=np.float64)
                g["occupancy"].append({
                    "source": sid, "sampler": alg, "seed": seed, "n_calls": 5000, "counts": list(counts),
                    "xor": "%016x" % int(np.bitwise_xor.reduce(buf.view(np.uint64))),
                    "state": "%016x" % src.state})
    for argv in SAMPLE_ARGS:
        g["cli"].append(run_cli(argv))
    # bench.py / stats.py host helpers (student_t_quantile, confidence_interval,
    # percent_faster, regularized_beta)
    g["host_fns"] = {
        "t_quantile": [[c, d, bench.student_t_quantile(c, d).hex()]
                       for c in (0.5, 0.9, 0.95, 0.999) for d in (1, 2, 3, 9, 30, 200)],
        "ci": [[xs, lvl, [v.hex() for v in bench.confidence_interval(xs, lvl)]]
               for xs, lvl in (([1.0, 1.2, 0.9, 1.1], 0.999), ([3.25, 3.5, 3.0], 0.9))],
        "percent_faster": [[b, c, bench.percent_faster(b, c).hex()] for b, c in ((5.0, 3.0), (1.7, 2.9))],
        "beta": [[a, b, x, regularized_beta(a, b, x).hex()]
                 for a, b, x in ((0.5, 0.5, 0.3), (2.0, 3.0, 0.7), (15.0, 0.5, 0.99), (0.5, 7.0, 0.01))],
    }
    # scripted-source scenarios of the samplers (the shapes of test_samplers.py:135-179):
    # each entry = (sampler, words, n calls, spare in) -> values, cursor, spare out / exhaustion
    def uw(u):   # a word whose next_f64_unit is u on the 53-bit grid
        return round(u * (1 << 53)) << 11

    t128, t256 = build_ziggurat_tables(128), build_ziggurat_tables(256)
    sc = []
    m_w = (t128.ktab[1] + (1 << 56)) // 2
    fast5 = (5 << 56) | (t128.ktab[5] // 2)
    gen = SplitMix64(8088)
    fast_words = []
    while len(fast_words) < 200:
        u = gen.next_u64()
        i = (u >> 56) & 0x7F
        if (u & ((1 << 56) - 1)) < t128.ktab[i]:
            fast_words.append(u & ~(1 << 63))
    scen = [
        ("ziggurat", [fast5], 1, None),
        ("ziggurat", fast_words, 200, None),
        ("ziggurat", [w | (1 << 63) for w in fast_words], 200, None),
        ("ziggurat", [t128.ktab[0] + 7, uw(math.exp(-1.0)), uw(math.exp(-0.5))], 1, None),
        ("ziggurat", [(1 << 56) | m_w, 0], 1, None),
        ("ziggurat", [(1 << 56) | m_w, (1 << 64) - 1, fast5], 1, None),
        ("ziggurat", [(1 << 56) | m_w, (1 << 64) - 1], 1, None),
        ("modified-ziggurat", [(t256.ktab[7] // 2 << 9) | 7, (t256.ktab[9] // 2 << 9) | (1 << 8) | 9], 2, None),
        ("modified-ziggurat", [((t256.ktab[3] + (1 << 55)) // 2 << 9) | 3, uw(0.25), (5 << 9) | 5], 1, None),
        ("polar", [uw(0.75), uw(0.25)], 2, None),
        ("polar", [uw(0.99), uw(0.99), uw(0.5), uw(0.75), uw(0.6), uw(0.6)], 3, None),
        ("polar", [uw(0.5), uw(0.5), uw(0.9), uw(0.2)], 3, 0.125),
        ("polar", [uw(0.999), uw(0.999)], 1, None),
    ]
    for alg, words, n, spare in scen:
        smp = make_sampler(alg)
        if spare is not None:
            smp.spare = spare
        src = ScriptedSource(words)
        vals, exhausted = [], False
        try:
            for _ in range(n):
                vals.append(smp.next_gaussian(src).hex())
        except ScriptExhausted:
            exhausted = True
        sc.append({"sampler": alg, "words": ["%016x" % w for w in words], "n": n, "spare_in": spare,
                   "values": vals, "exhausted": exhausted, "cursor": src.cursor,
                   "spare_out": None if getattr(smp, "spare", None) is None else smp.spare.hex()})
    g["scripted"] = sc
    g["tail"] = [[r, ["%016x" % w for w in ws], tail_sample(ScriptedSource(ws), r).hex()]
                 for r, ws in ((1.0, [uw(math.exp(-0.5)), uw(math.exp(-1.0))]),
                               (3.4426198558966377, [uw(0.3), uw(0.001), uw(0.5), uw(0.9)]))]
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
