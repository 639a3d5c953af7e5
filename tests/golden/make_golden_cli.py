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

from gausszig import cli, make_sampler, make_source

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
    with open(OUT, "w") as f:
        json.dump(g, f, indent=0, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
