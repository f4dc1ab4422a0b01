#!/usr/bin/env python
"""GPU-measured cost signal for the AutoShard-RL reward (rl.hpp:66).

The reference trainer scores a terminal plan with SIM-2 over per-table
marginals: shard cost = c0 + max(max w, (1-rho)*sum w + rho*max w)
(simcost.hpp:97-109, rl.hpp:161-167), with w = SIM-1 per table (rl.hpp:66).
This tool replaces the analytic pieces with B200 measurements through the GPU
cost hook (`measure_plan`: W/B/R fwd+bwd+row-wise-Adagrad steps, L2 flushed):

  m_t   = measured time of table t alone (a one-table shard),
  c0, rho fitted (least squares) to measured multi-table shards of random
          plans, with w_t = m_t - c0,

and writes them as a text file the plan producer (oracle/rl_plans.cpp,
MARGINALS=<file>) loads into TaskContext::marginal_w / sim.c0 / sim.rho.

  python tools/measure_marginals.py --pool 300 --dims 32 64 128 256 --out plans/cfg3_gpu_marginals.txt
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_06399_b200 as P  # noqa: E402


def sim2(w, c0, rho):
    w = np.asarray(w)
    return c0 + max(w.max(), (1 - rho) * w.sum() + rho * w.max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pool", type=int, default=300)
    ap.add_argument("--dims", type=int, nargs="*", default=[32, 64, 128, 256])
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--fit-tables", type=int, default=100, help="random shards are drawn from tables [0, n)")
    ap.add_argument("--fit-plans", type=int, default=8)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--out", required=True)
    args = ap.parse_args()

    pool = P.generate_pool(0, args.pool, P.GeneratorConfig(dim_choices=tuple(args.dims)))
    t0 = time.time()
    wl = P.generate_workload(0, pool, args.batch).pin()
    bench = P.BenchConfig(warmup=5, measure=10, trim=2)
    # per-table: every table its own shard
    n = len(pool)
    task = P.ShardingTask(pool, n, [1 << 40] * n)
    m = np.array(P.measure_plan(P.ShardingPlan(list(range(n))), task, wl, bench))
    t1 = time.time()
    # multi-table shards of random plans over the target tables
    tabs = pool[:args.fit_tables]
    ftask = P.ShardingTask(tabs, args.shards, [1 << 40] * args.shards)
    shards = []
    for s in range(args.fit_plans):
        plan = P.random_shard(ftask, 1000 + s)
        cost = P.measure_plan(plan, ftask, wl, bench)
        for k, members in enumerate(plan.shard_member_indices(ftask)):
            if members:
                shards.append((members, cost[k]))
    y = np.array([c for _, c in shards])
    best = None
    for c0 in np.linspace(0.0, float(m.min()), 201):
        w = m - c0
        S = np.array([w[mb].sum() for mb, _ in shards])
        X = np.array([w[mb].max() for mb, _ in shards])
        # y = c0 + S - rho * (S - X)  (the (1-rho) branch; rho in [0, 1))
        a = S - X
        r = y - c0 - S
        rho = float(np.clip(-(a @ r) / max(a @ a, 1e-30), 0.0, 0.999))
        pred = np.array([sim2(w[mb], c0, rho) for mb, _ in shards])
        err = float(np.sqrt(np.mean(((pred - y) / y) ** 2)))
        if best is None or err < best[0]:
            best = (err, float(c0), rho)
    err, c0, rho = best
    with open(args.out, "w") as f:
        f.write(f"# GPU-measured marginals (tools/measure_marginals.py): generate_pool(0,{args.pool}, dims "
                f"{args.dims}), batch {args.batch}, fwd+bwd W5/B10/R2 L2 flushed, one B200\n")
        f.write(f"# SIM-2 fit on {len(shards)} random shards of tables [0,{args.fit_tables}): rel. RMS error {err:.4f}\n")
        f.write(f"c0 {c0:.6f}\nrho {rho:.6f}\n")
        for t, v in zip(pool, m):
            f.write(f"{t.id} {v - c0:.6f}\n")
    summary = {"tables": n, "single_ms_min_median_max": [float(m.min()), float(np.median(m)), float(m.max())],
               "c0": c0, "rho": rho, "fit_rel_rms": err, "fit_shards": len(shards),
               "measure_s": round(t1 - t0, 1), "fit_s": round(time.time() - t1, 1)}
    print(json.dumps(summary))
    with open(os.path.splitext(args.out)[0] + ".json", "w") as f:
        json.dump({**summary, "single_ms": {int(t.id): float(v) for t, v in zip(pool, m)},
                   "shards": [{"members": [int(pool[i].id) for i in mb], "ms": c} for mb, c in shards]}, f, indent=1)


if __name__ == "__main__":
    main()
