"""GPU parity at the BASELINE sizes, element by element.

Every pooled row of every bag is compared with the fp64 oracle (OpenMP,
oracle.c orc_emb_forward_f64_rows) — BIT-EXACT, because the initial weights
live on the k*2^-12 grid (see test_gpu_parity.py for the argument). After one
backward (grad = pooled, loss 1/2|pooled|^2), EVERY updated row and its
momentum of the checked tables is compared with the fp64 restatement of exact
row-wise Adagrad (oracle.c orc_emb_backward_adagrad_f64), tolerance as in
test_gpu_parity.py: |dW| <= 1e-5*max(|ref|, |W_old|, |W_old - ref|) + 1e-7,
|dm| <= 1e-5*|ref| + 1e-7. Rows never looked up must stay untouched (probed).

Configs: cfg2 (50 tables, dim 128, B 65,536; all bags, 10 tables' rows),
cfg3 (100 tables, dims 32-256, B 65,536; all bags, 8 tables' rows), one
shard of the 8-GPU AutoShard-RL plan of cfg4 (all bags, ALL tables' rows) and
one shard of cfg5 (B 131,072; all bags, 8 tables' rows).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from helpers import fp_close, to_oracle_tables, weight_rows

pytestmark = pytest.mark.gpu

LR, EPS, SEED = 0.01, 1e-8, 7
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _workload(P, name):
    import sys

    sys.path.insert(0, ROOT)
    import bench

    return bench, bench.build_workload(P, name)


def _plan_shard(P, name, k, shard):
    bench, (tables, B, _) = _workload(P, name)
    task = bench.device_task(P, tables, k)
    plan, _ = P.load_plan(os.path.join(ROOT, "plans", f"{name}_k{k}_autoshard_rl.plan"), task)
    return [tables[i] for i in plan.shard_member_indices(task)[shard]], B


def _check_shard(P, oracle, torch, tables, B, bwd_tables, block_rows=8192):
    wl = P.generate_workload(0, tables, B)
    streams = [(wl.find(t.id).offsets, wl.find(t.id).indices) for t in tables]
    otabs = to_oracle_tables(tables)
    with P.EmbeddingShard(tables, B, weight_seed=SEED) as sh:
        sh.load(wl)
        sh.forward()
        torch.cuda.synchronize()
        pooled = sh.pooled_tensor()
        # ---- forward: every bag, bit-exact ----
        for b0 in range(0, B, block_rows):
            b1 = min(B, b0 + block_rows)
            ref = oracle.forward_f64(otabs, B, streams, wseed=SEED, rows=(b0, b1))
            got = pooled[b0:b1].cpu().numpy().astype(np.float64)
            if not np.array_equal(got, ref):
                bad = np.argwhere(got != ref)[0]
                raise AssertionError(f"pooled row {b0 + bad[0]} col {bad[1]}: {got[tuple(bad)]} != {ref[tuple(bad)]}")
        # ---- backward with grad = pooled; the gradient slabs of the checked
        # tables are read before the update (the pooled buffer is not modified) ----
        grads = {t: pooled[:, sh.cols[t]:sh.cols[t] + tables[t].dim].contiguous().cpu().numpy() for t in bwd_tables}
        sh.backward(None, LR, EPS)
        torch.cuda.synchronize()

        def oracle_bwd(t):
            return t, oracle.backward_adagrad_f64(otabs[t], B, *streams[t], grads[t], 0, LR, EPS, wseed=SEED)

        with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
            results = list(ex.map(oracle_bwd, bwd_tables))
        checked_rows = 0
        for t, r in results:
            tab = tables[t]
            if len(r["rows"]) == 0:
                continue
            w = sh.read_rows(t, r["rows"])
            w_old = weight_rows(SEED, tab.id, r["rows"], tab.dim).astype(np.float64)
            ok, worst = fp_close(w, r["w"], scale=np.maximum(np.abs(w_old), np.abs(w_old - r["w"])))
            assert ok, f"table {tab.id}: updated rows off by {worst:.3g}x tolerance"
            m = sh.read_momentum(t, r["rows"])
            ok, worst = fp_close(m, r["m"])
            assert ok, f"table {tab.id}: momentum off by {worst:.3g}x tolerance"
            checked_rows += len(r["rows"])
            touched = np.zeros(tab.hash_size, dtype=bool)
            touched[r["rows"]] = True
            probe = np.flatnonzero(~touched)[:: max(1, (tab.hash_size - len(r["rows"])) // 97)][:97]
            if len(probe):
                assert np.array_equal(sh.read_rows(t, probe), weight_rows(SEED, tab.id, probe, tab.dim)), \
                    f"table {tab.id}: a row never looked up changed"
        return checked_rows


def _sample_tables(tables, streams_len, n):
    """n table positions: the most-looked-up, the largest, and evenly spread others."""
    order = sorted(range(len(tables)), key=lambda t: -streams_len[t])
    pick = {order[0], max(range(len(tables)), key=lambda t: tables[t].hash_size)}
    for t in np.linspace(0, len(tables) - 1, n).astype(int):
        if len(pick) >= n:
            break
        pick.add(int(t))
    return sorted(pick)


def test_cfg2_full_batch_every_bag_and_row(P, oracle, cuda):
    bench, (tables, B, _) = _workload(P, "cfg2")
    lens = [t.pooling_mean for t in tables]
    rows = _check_shard(P, oracle, cuda, tables, B, _sample_tables(tables, lens, 10))
    assert rows > 100_000


def test_cfg3_full_batch_every_bag_and_row(P, oracle, cuda):
    bench, (tables, B, _) = _workload(P, "cfg3")
    lens = [t.pooling_mean for t in tables]
    rows = _check_shard(P, oracle, cuda, tables, B, _sample_tables(tables, lens, 8))
    assert rows > 10_000


def test_cfg4_plan_shard_all_tables(P, oracle, cuda):
    """Shard 0 of the 8-GPU AutoShard-RL plan of cfg 4 (116 tables, dims 16/32)."""
    tables, B = _plan_shard(P, "cfg4", 8, 0)
    rows = _check_shard(P, oracle, cuda, tables, B, list(range(len(tables))))
    assert rows > 1_000_000


def test_cfg5_plan_shard(P, oracle, cuda):
    """Shard 3 of the 8-GPU AutoShard-RL plan of cfg 5 (91 tables, dims 64-256,
    B = 131,072: 48.7 GB of fp32 tables)."""
    tables, B = _plan_shard(P, "cfg5", 8, 3)
    lens = [t.pooling_mean for t in tables]
    rows = _check_shard(P, oracle, cuda, tables, B, _sample_tables(tables, lens, 8), block_rows=4096)
    assert rows > 10_000
