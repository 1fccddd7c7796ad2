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


def test_nvlink_bound_chain_vs_multicast():
    """The publish->all lower bound bench.py divides by: in the chain every middle relay
    receives and forwards the image; with multicast (NEXT-2) node 0's GPU sends it once and no relay
    forwards — the per-GPU maximum is M either way, only the distribution differs."""
    sys.path.insert(0, ROOT)
    import bench
    P = 1000
    T = bench.topology("chain", 4, 0)
    ing, egr = bench.nvlink_bound(T, 4, P)
    assert [ing[d] for d in range(4)] == [0, 2 * P, 2 * P, 2 * P]
    assert [egr[d] for d in range(4)] == [2 * P, 2 * P, 2 * P, 0]
    ing, egr = bench.nvlink_bound(T, 4, P, multicast=True)
    assert [ing[d] for d in range(4)] == [0, 2 * P, 2 * P, 2 * P]
    assert [egr[d] for d in range(4)] == [2 * P, 0, 0, 0]
    T = bench.topology("colocated", 4, 2)          # FSDP-4 colocated: no hop, pulls gather instead
    ing, egr = bench.nvlink_bound(T, 4, P, pull_in={0: 7.0})
    assert ing[0] == 7.0 and max(egr.values()) == 0


def test_line_config_is_shared_by_both_arms():
    """The driver compares the two arms only on the same `config` object."""
    sys.path.insert(0, ROOT)
    import bench
    import argparse
    args = argparse.Namespace(model="7b", config="chain", tp=0, hop_mode="kernel")
    c1, c2 = bench.line_config(args, 1), bench.line_config(args, 1)
    assert c1 == c2 and c1["params"] == 7615616512 and c1["snapshot_bytes"] == 2 * 7615616512
    args.hop_mode = "mc"
    assert bench.line_config(args, 4)["parallelism"] == "chain N=4 hop=mc"
