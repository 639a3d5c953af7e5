"""The gausszig-style CLI (paper_2405_19493_b200/cli.py) against the reference
CLI's own output (tests/golden/golden_cli.json, made by make_golden_cli.py from
the unmodified reference), and layer occupancy against the reference's
sample_with_occupancy.  CPU tests cover the oracle pin, argument errors and the
table command; `gpu` tests run the device paths."""
import contextlib
import io
import json

import numpy as np
import pytest

from oracle import gz_oracle as O
from paper_2405_19493_b200 import cli


def run(argv):
    out, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
        code = cli.main(argv)
    return code, out.getvalue(), err.getvalue()


def state_words(source, seed):
    from paper_2405_19493_b200 import make_source

    s = make_source(source, seed)
    return np.array([s.state] if source == "lcg48" else [s.state, s.gamma], dtype=np.uint64)


def test_oracle_occupancy_pinned_to_reference(golden_cli):
    for r in golden_cli["occupancy"]:
        vals, counts, st, status = O.occupancy(r["sampler"], r["source"], state_words(r["source"], r["seed"]),
                                               r["n_calls"])
        assert status == 0
        assert [int(c) for c in counts] == r["counts"]
        assert "%016x" % int(np.bitwise_xor.reduce(vals.view(np.uint64))) == r["xor"]
        assert "%016x" % int(st[0]) == r["state"]


@pytest.mark.parametrize("case", range(10))
def test_cli_host_only_commands(golden_cli, case):
    rec = golden_cli["cli"][case]
    if rec["argv"][0] == "tables" or rec["code"] == 2:
        code, out, _ = run(rec["argv"])
        assert code == rec["code"]
        assert out == rec["stdout"]


def test_cli_argument_errors():
    assert run(["verify", "--source", "lcg48"])[0] == 2
    assert run(["sample", "--sampler", "polar"])[0] == 2
    assert run(["verify", "--source", "splitmix", "--sampler", "polar", "--n", "10"])[0] == 2
    assert run(["sample", "--source", "splitmix", "--sampler", "polar", "--n", "-1"])[0] == 2
    assert run(["sample", "--source", "splitmix", "--sampler", "polar", "--sigma", "-1"])[0] == 2
    assert run(["bits", "--source", "scripted", "--k", "2"])[0] == 2
    assert run(["bench", "--source", "lcg48", "--sampler", "modified-ziggurat"])[0] == 2
    assert run(["tables", "--n", "12"])[0] == 2
    assert run(["tables", "--n", "32", "--out", "/nonexistent-dir/t.json"])[0] == 3


@pytest.mark.gpu
def test_device_occupancy_matches_reference(golden_cli):
    from paper_2405_19493_b200 import make_sampler, make_source

    for r in golden_cli["occupancy"]:
        src = make_source(r["source"], r["seed"])
        vals, counts = make_sampler(r["sampler"]).sample_with_occupancy(src, r["n_calls"])
        assert counts == r["counts"]
        buf = np.array(vals, dtype=np.float64)
        assert "%016x" % int(np.bitwise_xor.reduce(buf.view(np.uint64))) == r["xor"]
        assert "%016x" % src.state == r["state"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", range(10))
def test_cli_matches_reference_output(golden_cli, case):
    rec = golden_cli["cli"][case]
    code, out, _ = run(rec["argv"])
    assert code == rec["code"]
    assert out == rec["stdout"]


@pytest.mark.gpu
@pytest.mark.parametrize("source,sampler", [("splitmix", "ziggurat"), ("lcg48", "polar"),
                                            ("splitmix", "modified-ziggurat")])
def test_cli_verify_passes(source, sampler):
    code, out, _ = run(["verify", "--source", source, "--sampler", sampler, "--n", "200000", "--seed", "5"])
    doc = json.loads(out)
    assert code == 0 and doc["verdict"] == "pass"
    tests = [r["test"] for r in doc["reports"]]
    assert tests[:3] == ["moments", "ks", "chi_square_equal_prob_bins"]
    assert ("layer_occupancy" in tests) == (sampler != "polar")


@pytest.mark.gpu
def test_cli_bits_scripted(tmp_path):
    words = np.random.default_rng(3).integers(0, 2 ** 63, 5000, dtype=np.uint64)
    p = tmp_path / "w.txt"
    p.write_text("\n".join(hex(int(w)) for w in words))
    code, out, _ = run(["bits", "--source", "scripted", "--k", "4", "--script", str(p)])
    doc = json.loads(out)
    exp = np.bincount((words & np.uint64(15)).astype(np.int64), minlength=16).astype(np.float64)
    e = exp.sum() / 16
    assert doc["statistic"] == float(((exp - e) ** 2 / e).sum())
    assert code == (0 if doc["verdict"] == "pass" else 1)
    assert run(["bits", "--source", "scripted", "--k", "4", "--script", str(p), "--n", "6000"])[0] == 2


@pytest.mark.gpu
def test_device_moments_buffer():
    import torch

    from paper_2405_19493_b200 import verify

    x = np.random.default_rng(8).standard_normal(300_001) * 1.3 + 0.2
    m = verify.moments(torch.from_numpy(x).cuda())
    n = x.size
    mean = x.mean()
    d = x - mean
    m2, m3, m4 = (d ** 2).sum(), (d ** 3).sum(), (d ** 4).sum()
    assert m.n == n
    assert abs(m.mean - mean) < 1e-12
    assert abs(m.variance / (m2 / (n - 1)) - 1) < 1e-10
    assert abs(m.skewness - np.sqrt(n) * m3 / m2 ** 1.5) < 1e-8
    assert abs(m.excess_kurtosis - (n * m4 / m2 ** 2 - 3)) < 1e-8


@pytest.mark.gpu
def test_bench_cli_smoke():
    code, out, _ = run(["bench", "--profile", "smoke", "--format", "json", "--source", "splitmix"])
    docs = json.loads(out)
    assert code == 0 and len(docs) == 3
    assert all(d["engine_used"] == "cuda" and d["ns_per_op"] > 0 for d in docs)
    assert sum("percent_faster_vs_polar" in d for d in docs) == 2


@pytest.mark.gpu
def test_bench_single_layout_matches_witness(golden):
    """The reference's one-stream call shape on the GPU: same checksum witness."""
    from paper_2405_19493_b200 import benchmark

    r = benchmark.run_benchmark("ziggurat", "splitmix", benchmark.BenchConfig.single())
    assert r.ns_per_op > 0 and r.engine_used == "cuda"
    assert "%016x" % r.checksum == golden["bench_witness"]["splitmix/ziggurat/%d" % benchmark.DEFAULT_SEED]


def test_bench_and_stats_host_helpers_match_reference(golden_cli):
    from paper_2405_19493_b200 import benchmark, verify

    h = golden_cli["host_fns"]
    for c, d, v in h["t_quantile"]:
        assert abs(benchmark.student_t_quantile(c, d) - float.fromhex(v)) <= 1e-12 * max(1.0, abs(float.fromhex(v)))
    for xs, lvl, (lo, hi) in h["ci"]:
        a, b = benchmark.confidence_interval(xs, lvl)
        assert abs(a - float.fromhex(lo)) < 1e-12 and abs(b - float.fromhex(hi)) < 1e-12
    for b, c, v in h["percent_faster"]:
        assert benchmark.percent_faster(b, c) == float.fromhex(v)
    for a, b, x, v in h["beta"]:
        assert abs(verify.regularized_beta(a, b, x) - float.fromhex(v)) < 1e-14
    with pytest.raises(ValueError):
        benchmark.percent_faster(0.0, 1.0)
    with pytest.raises(ValueError):
        benchmark.confidence_interval([1.0], 0.9)
