"""bench.py contract pieces that run without a GPU: the SURVEY.md §8d bytes
model (fp32 and fp16 table storage), the N>1 plan choice (AutoShard-RL plan
files), and the reference arm's JSON line (CPU port + the reference's own
pieces) on a small workload."""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_nominal_bytes_match_survey_formulas(P):
    tables, B, _ = bench.build_workload(P, "cfg1")
    L = [1000 + 10 * i for i in range(len(tables))]
    U = [100 + i for i in range(len(tables))]
    s = 4
    T, SD = len(tables), sum(t.dim for t in tables)
    LD = sum(l * t.dim for l, t in zip(L, tables))
    UD = sum(u * t.dim for u, t in zip(U, tables))
    fwd, bwd, ph = bench.nominal_bytes(tables, B, L, U)
    assert fwd == s * (sum(L) + T * (B + 1) + LD + B * SD)  # SURVEY §8d FWD
    assert bwd == s * (sum(L) + T * (B + 1) + LD) + 2 * s * UD + 2 * s * sum(U)  # BWD
    assert sum(ph.values()) == fwd + bwd
    fwd2, bwd2, ph2 = bench.nominal_bytes(tables, B, L, U, wb=2)
    assert fwd - fwd2 == 2 * LD and bwd - bwd2 == 2 * 2 * UD
    assert sum(ph2.values()) == fwd2 + bwd2


def test_n_gpu_plan_prefers_autoshard_rl_file(P):
    tables, B, _ = bench.build_workload(P, "cfg4")
    task = P.ShardingTask(tables, 8, [int(180e9)] * 8)
    plan, name = bench.bench_plan(P, task, "cfg4", 8)
    path = os.path.join(ROOT, "plans", "cfg4_k8_autoshard_rl.assignment")
    if os.path.exists(path):
        assert name.startswith("autoshard-rl")
        assert plan.assignment == [int(x) for x in open(path).read().split()]
    else:
        assert name.startswith("lookup-greedy")
    assert plan.feasible(task)
    # no RL plan for this shard count -> lookup-greedy
    task3 = P.ShardingTask(tables, 3, [int(180e9)] * 3)
    plan3, name3 = bench.bench_plan(P, task3, "cfg4", 3)
    assert name3.startswith("lookup-greedy")
    assert plan3.assignment == P.greedy_shard(task3, P.HeuristicKind.kLookupGreedy).assignment


def test_reference_arm_json_line():
    env = dict(os.environ, ASB_REF_PIECES="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "cfg1",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    pieces = d["reference_pieces"]
    assert "unavailable" in pieces or (pieces["generate_workload_s"] >= 0 and pieces["threads"] == 1)
    assert np.isfinite(d["ms_per_step"])
