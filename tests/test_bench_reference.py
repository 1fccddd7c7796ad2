"""The reference arm of bench.py (tier framing: the CPU oracle, timed as it stands) keeps the driver's
JSON contract on CPU: one line with impl=reference, the lam arm's metric/unit/workload, a cpu_baseline
describing this run (full steps on a process pool, measured) and an e2e object with zero transfer bytes."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--model", "tiny"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "publish->all-rollouts sync latency" and d["unit"] == "s"
    assert d["higher_is_better"] is False and d["value"] > 0
    assert d["config"]["workload"].startswith("tiny [chain]: ")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["measured"] == "full step" and cb["host"]["nproc"] >= 1
    # the timed region really held `steps` full steps (the driver compares steps x value with its clock)
    assert abs(d["consistency"]["steps_x_value_s"] - d["consistency"]["timed_wall_s"]) < 0.05 + 0.1 * d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0 and not [l for l in r.stdout.splitlines() if l.startswith("{")]
