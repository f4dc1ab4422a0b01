#!/usr/bin/env python
"""AutoShard-RL vs the heuristics on MEASURED B200 shard times, as mean +- sd
over training seeds (the paper's format).

Every plan's shards are timed with the same protocol (W/B/R fwd + bwd +
row-wise Adagrad steps, L2 flushed, one shard at a time on one GPU) through
subset contexts over ONE resident copy of the target's tables
(EmbeddingShard.subset / retarget = as_create_subset / as_retarget_subset).
Plans:
  size / dim / lookup greedy     planners.hpp:73-107 (deterministic)
  random-<s>                     planners.hpp:111-136, seeds 0..R-1
  measured-lpt                   the same LPT with each table's cost = its measured one-table time
  <group>-s<seed>                AutoShard-RL plans from the reference trainer (oracle/rl_plans*.cpp),
                                 one per training seed, every seed reported (no best-of-N)

  python tools/rl_seed_study.py --workload cfg3 --group rl-gpu='plans/rl_gpu/cfg3_rl_gpu_s*.assignment' \\
      --group rl-sim='plans/rl_sim/cfg3_rl_sim_s*.assignment' --out profiles/r2_rl_seed_study_cfg3.json
"""
import argparse
import glob
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_06399_b200 as P  # noqa: E402
import bench  # noqa: E402


def lpt(tables, cost, K, budget):
    """planners.hpp:73-107's greedy (largest first, least-loaded feasible shard)
    with the given per-table costs."""
    order = sorted(range(len(tables)), key=lambda i: (-cost[i], tables[i].id))
    load, used, a = [0.0] * K, [0] * K, [0] * len(tables)
    for i in order:
        fits = [k for k in range(K) if used[k] + tables[i].size_bytes() <= budget[k]] or list(range(K))
        k = min(fits, key=lambda k: (load[k], k))
        a[i] = k
        load[k] += cost[i]
        used[k] += tables[i].size_bytes()
    return P.ShardingPlan(a)


def mean_sd(xs):
    return {"mean": statistics.mean(xs), "sd": statistics.stdev(xs) if len(xs) > 1 else 0.0, "n": len(xs),
            "min": min(xs), "max": max(xs)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--random-seeds", type=int, default=5)
    ap.add_argument("--group", action="append", default=[], help="NAME=GLOB of .assignment files (one per seed)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--measure", type=int, default=10)
    ap.add_argument("--trim", type=int, default=2)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    tables, B, desc = bench.build_workload(P, args.workload)
    K = args.shards
    wl = P.generate_workload(0, tables, B).pin()
    total = sum(t.size_bytes() for t in tables)
    task = P.ShardingTask(tables, K, [int(1.6 * total / K)] * K)  # SPEC.md:620, as the trainer's task_of
    parent = P.EmbeddingShard(tables, B, weight_seed=0)
    sub = [None]
    cache = {}

    def shard_ms(positions):
        key = tuple(sorted(positions))
        if not key:
            return 0.0
        if key not in cache:
            if sub[0] is None:
                sub[0] = parent.subset(list(key))
            else:
                sub[0].retarget(list(key))
            sub[0].load(wl)
            cache[key] = sub[0].measure(args.warmup, args.measure, args.trim)
        return cache[key]

    t0 = time.time()
    single = [shard_ms([i]) for i in range(len(tables))]
    plans = {}
    for kind, name in [(P.HeuristicKind.kSizeGreedy, "size-greedy"), (P.HeuristicKind.kDimGreedy, "dim-greedy"),
                       (P.HeuristicKind.kLookupGreedy, "lookup-greedy")]:
        plans[name] = P.greedy_shard(task, kind)
    for s in range(args.random_seeds):
        plans[f"random-s{s}"] = P.random_shard(task, s)
    plans["measured-lpt"] = lpt(tables, single, K, task.mem_budget)
    groups = {"random": [f"random-s{s}" for s in range(args.random_seeds)]}
    for g in args.group:
        name, pat = g.split("=", 1)
        groups[name] = []
        for path in sorted(glob.glob(pat)):
            a = [int(x) for x in open(path).read().split()]
            if len(a) != len(tables) or max(a) >= K:
                raise SystemExit(f"{path}: not a {K}-shard plan of {len(tables)} tables")
            seed = os.path.basename(path).rsplit("_s", 1)[-1].split(".")[0]
            plans[f"{name}-s{seed}"] = P.ShardingPlan(a)
            groups[name].append(f"{name}-s{seed}")
    res = {}
    for name, plan in plans.items():
        costs = [shard_ms(m) for m in plan.shard_member_indices(task)]
        res[name] = {"shard_ms": costs, "max_ms": max(costs), "balance": P.degree_of_balance(costs),
                     "feasible": plan.feasible(task), "assignment": plan.assignment}
        print(f"{name:18s} max {max(costs):7.3f} ms  balance {res[name]['balance']:.3f}", flush=True)
    rnd = statistics.mean(res[k]["max_ms"] for k in groups["random"])
    lg = res["lookup-greedy"]["max_ms"]
    for v in res.values():
        v["speedup_vs_random_mean"] = rnd / v["max_ms"]
        v["speedup_vs_lookup_greedy"] = lg / v["max_ms"]
    summary = {}
    for name in ["size-greedy", "dim-greedy", "lookup-greedy", "measured-lpt"]:
        summary[name] = {k: res[name][k] for k in ("max_ms", "balance", "speedup_vs_random_mean",
                                                  "speedup_vs_lookup_greedy")}
    for g, members in groups.items():
        if members:
            summary[g] = {k: mean_sd([res[m][k] for m in members])
                          for k in ("max_ms", "balance", "speedup_vs_random_mean", "speedup_vs_lookup_greedy")}
    out = {"workload": args.workload, "desc": desc, "shards": K, "batch": B,
           "budget_rule": "1.6 x total / K (SPEC.md:620), bytes_per_param 2",
           "protocol": f"W={args.warmup} B={args.measure} R={args.trim}, L2 flushed, subset contexts over one "
                       f"resident copy of the tables, one shard at a time on 1 GPU",
           "single_table_ms": {t.id: c for t, c in zip(tables, single)},
           "random_max_ms_mean": rnd, "summary": summary, "plans": res, "wall_s": round(time.time() - t0, 1)}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    for k, v in summary.items():
        if isinstance(v["max_ms"], dict):
            print(f"{k:14s} max {v['max_ms']['mean']:.3f} +- {v['max_ms']['sd']:.3f} ms  balance "
                  f"{v['balance']['mean']:.3f} +- {v['balance']['sd']:.3f}  vs random "
                  f"{v['speedup_vs_random_mean']['mean']:.3f} +- {v['speedup_vs_random_mean']['sd']:.3f}  "
                  f"vs lookup-greedy {v['speedup_vs_lookup_greedy']['mean']:.3f} (n={v['max_ms']['n']})")
        else:
            print(f"{k:14s} max {v['max_ms']:.3f} ms  balance {v['balance']:.3f}  vs random "
                  f"{v['speedup_vs_random_mean']:.3f}  vs lookup-greedy {v['speedup_vs_lookup_greedy']:.3f}")
    if sub[0] is not None:
        sub[0].close()
    parent.close()


if __name__ == "__main__":
    main()
