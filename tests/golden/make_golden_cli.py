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

from gausszig import bench, cli, make_sampler, make_source
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
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
