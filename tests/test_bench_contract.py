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
    task = bench.device_task(P, tables, 8)
    assert all(t.bytes_per_param == 4 for t in task.tables)  # fp32 device storage
    plan, name = bench.bench_plan(P, task, "cfg4", 8)
    path = os.path.join(ROOT, "plans", "cfg4_k8_autoshard_rl.assignment")
    assert name.startswith("autoshard-rl") and "fingerprint" in name
    assert plan.assignment == [int(x) for x in open(path).read().split()]
    assert plan.feasible(task)
    # a plan file made for another task is rejected (fingerprint)
    other = bench.device_task(P, tables, 8, weights="fp16")
    try:
        bench.bench_plan(P, other, "cfg4", 8)
        raise AssertionError("stale plan accepted")
    except P.StateError as e:
        assert "fingerprint" in str(e)
    # no RL plan for this shard count -> lookup-greedy
    task3 = bench.device_task(P, tables, 3)
    plan3, name3 = bench.bench_plan(P, task3, "cfg4", 3)
    assert name3.startswith("lookup-greedy")
    assert plan3.assignment == P.greedy_shard(task3, P.HeuristicKind.kLookupGreedy).assignment


def test_compulsory_bytes_below_nominal(P):
    tables, B, _ = bench.build_workload(P, "cfg2")
    L = [200000 + 10 * i for i in range(len(tables))]
    U = [1000 + i for i in range(len(tables))]
    _, _, nom = bench.nominal_bytes(tables, B, L, U)
    comp = bench.compulsory_bytes(tables, B, L, U, bench.sort_passes(tables))
    for k in ("fwd_segreduce", "bwd_segreduce_adagrad"):
        assert 0 < comp[k] < nom[k]


def test_sources_sha_is_stable():
    a, b = bench.sources_sha(), bench.sources_sha()
    assert a == b and len(a) == 16


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
    assert d["config"] == bench.common_config("cfg1", 10, 512)
    assert "reference" in d["data"]  # tables/streams from the reference build (oracle/_ref) when present


def test_reference_arm_never_imports_the_product():
    """The reference arm runs the oracle port on oracle-generated streams only."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'cfg1', '--steps', '1', "
            "'--warmup', '3']; runpy.run_path('bench.py', run_name='__main__'); "
            "assert not any(m.startswith('paper_2208_06399_b200') for m in sys.modules), 'product imported'")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=dict(os.environ, ASB_REF_PIECES="0"))
    assert r.returncode == 0, r.stderr[-2000:]
