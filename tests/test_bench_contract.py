"""bench.py's driver contract on the CPU: `--impl reference --gpus 2` outside a
torchrun environment re-launches itself with two ranks (torch.distributed.run,
rendezvous on 127.0.0.1); rank 0 alone times the CPU port of config 4 and prints
exactly one JSON line, the other rank exits 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_spawns_ranks_and_prints_one_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env.update(GZ_BENCH_REF_STREAMS="4096", GZ_BENCH_NUMBA_STREAMS="64", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["world_size"] == 2 and d["n_gpus"] == 2
    assert d["unit"] == "variates/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "variates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "config 4" in d["config"]["workload"]
