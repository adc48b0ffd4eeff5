"""The bench contract for the reference arm (the CPU oracle), checked on CPU.

`bench.py --impl reference` must print exactly one JSON line on stdout with the keys the
driver reads; under torchrun only rank 0 prints. A short `--ref-seconds` keeps it to ~2 s.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-seconds", "0.5", "--workload", "C1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    return out.stdout


def test_reference_arm_prints_one_json_line():
    lines = [l for l in _run({"RANK": "0"}).splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "plan evaluations/sec" and d["unit"] == "evals/s"
    assert d["higher_is_better"] is True and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the same `config` our arm writes (bench.run_config): the workload and its size only
    import workloads as W
    c, w = d["config"], W.WORKLOADS["C1"]
    assert set(c) == {"workload", "chains_per_config", "feasible_configs", "enumerated_configs",
                      "sa_proposals_per_step"}
    assert c["chains_per_config"] == w.chains and c["workload"].startswith("C1:")
    assert c["sa_proposals_per_step"] <= c["chains_per_config"] * c["feasible_configs"] * w.iterations


def test_reference_arm_nonzero_rank_is_silent():
    assert _run({"RANK": "1"}).strip() == ""
