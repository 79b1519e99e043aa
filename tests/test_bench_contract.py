"""The bench.py contract on the CPU side: `--impl reference` (the oracle on the host cores) prints one
JSON line with the required keys, on the same metric / config as the GPU arm; under torchrun only rank
0 prints.  (The GPU arm is exercised on the B200 box.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_line():
    lines = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"])
    assert len(lines) == 1
    d = lines[0]
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "C1"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_silent():
    assert _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0", "--gpus", "2"],
                env={"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_gpus_must_match_world_size():
    """--gpus N under a launcher with another WORLD_SIZE must fail loudly, not time another count."""
    e = dict(os.environ, RANK="0", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                        "--warmup", "0", "--gpus", "4"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
