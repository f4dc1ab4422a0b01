#!/usr/bin/env python
"""Sharding-plan study on MEASURED B200 shard times (§5).

For a BASELINE config, builds the comparison plans — size/dim/lookup greedy
(planners.hpp:73-107), random (planners.hpp:111-136, several seeds) and, when
present, an AutoShard-RL plan produced by the reference trainer
(oracle/rl_plans.cpp -> plans/<cfg>_autoshard_rl.assignment) — and measures
every shard of every plan with the GPU cost hook (`measure_plan`: W=5/B=10/R=2
fwd+bwd+row-wise Adagrad steps, L2 flushed). Shards run one at a time on one
GPU (the paper's per-device micro-benchmark). Reports max-shard ms (the C_k
objective), degree of balance and speedups.

  python tools/plan_study.py --workload cfg3 --out profiles/plan_study_cfg3.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2208_06399_b200 as P  # noqa: E402
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--random-seeds", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--measure", type=int, default=10)
    ap.add_argument("--trim", type=int, default=2)
    ap.add_argument("--weights", choices=["fp32", "fp16"], default="fp32")
    ap.add_argument("--plans", default="", help="comma list of plan names to measure (default: all)")
    args = ap.parse_args()

    tables, B, desc = bench.build_workload(P, args.workload)
    K = args.shards
    wl = P.generate_workload(0, tables, B).pin()
    total = sum(t.size_bytes() for t in tables)
    task = P.ShardingTask(tables, K, [int(1.6 * total / K)] * K)  # SPEC.md:620 budget rule
    plans = {}
    for kind, name in [(P.HeuristicKind.kSizeGreedy, "size-greedy"), (P.HeuristicKind.kDimGreedy, "dim-greedy"),
                       (P.HeuristicKind.kLookupGreedy, "lookup-greedy")]:
        plans[name] = P.greedy_shard(task, kind)
    for s in range(args.random_seeds):
        plans[f"random-{s}"] = P.random_shard(task, s)
    for tag, fname in (("autoshard-rl", f"{args.workload}_autoshard_rl"),
                       ("autoshard-rl", f"{args.workload}_k{K}_autoshard_rl"),
                       ("autoshard-rl-gpu", f"{args.workload}_autoshard_rl_gpu"),
                       ("autoshard-rl-gpu-1200", f"{args.workload}_autoshard_rl_gpu2")):
        rl = os.path.join(ROOT, "plans", fname + ".assignment")
        if os.path.exists(rl):
            a = [int(x) for x in open(rl).read().split()]
            if len(a) == len(tables) and max(a) < K:
                plans[tag] = P.ShardingPlan(a)
    # LPT greedy over GPU-MEASURED per-table costs (tools/measure_marginals.py), the
    # planners.hpp:73-107 algorithm with the analytic cost replaced by the measurement
    mj = os.path.join(ROOT, "plans", f"{args.workload}_gpu_marginals.json")
    if os.path.exists(mj):
        ms = json.load(open(mj))["single_ms"]
        if all(str(t.id) in ms for t in tables):
            order = sorted(range(len(tables)), key=lambda i: (-ms[str(tables[i].id)], tables[i].id))
            load, used, a = [0.0] * K, [0] * K, [0] * len(tables)
            for i in order:
                fits = [k for k in range(K) if used[k] + tables[i].size_bytes() <= task.mem_budget[k]] or list(range(K))
                k = min(fits, key=lambda k: (load[k], k))
                a[i] = k
                load[k] += ms[str(tables[i].id)]
                used[k] += tables[i].size_bytes()
            plans["measured-greedy"] = P.ShardingPlan(a)
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "plans", f"{args.workload}_autoshard_rl_s*.assignment")) +
                       glob.glob(os.path.join(ROOT, "plans", f"{args.workload}_k{K}_autoshard_rl_*.assignment"))):
        tag = "autoshard-rl-" + os.path.basename(path).split("_autoshard_rl_")[1].split(".")[0]  # seed / longer runs
        a = [int(x) for x in open(path).read().split()]
        if len(a) == len(tables) and max(a) < K:
            plans[tag] = P.ShardingPlan(a)
    if args.plans:
        keep = set(args.plans.split(","))
        plans = {k: v for k, v in plans.items() if k in keep or k.split("-")[0] in keep}
    bench_cfg = P.BenchConfig(warmup=args.warmup, measure=args.measure, trim=args.trim)
    res = {}
    for name, plan in plans.items():
        t0 = time.time()
        if args.weights == "fp32":
            costs = P.measure_plan(plan, task, wl, bench_cfg)
        else:  # same protocol shard by shard, fp16 table storage
            costs = []
            for members in plan.shard_member_indices(task):
                tabs = [tables[i] for i in members]
                with P.EmbeddingShard(tabs, B, weight_seed=0, weights=args.weights) as sh:
                    sh.load([(wl.find(t.id).offsets, wl.find(t.id).indices) for t in tabs])
                    costs.append(sh.measure(args.warmup, args.measure, args.trim))
        res[name] = {"assignment": plan.assignment, "shard_ms": costs, "max_ms": max(costs),
                     "balance": P.degree_of_balance(costs), "feasible": plan.feasible(task),
                     "wall_s": round(time.time() - t0, 1)}
        print(f"{name:14s} max {max(costs):7.3f} ms  balance {res[name]['balance']:.3f}  "
              f"shards {' '.join(f'{c:.3f}' for c in costs)}", flush=True)
    rnd = [res[k]["max_ms"] for k in res if k.startswith("random-")]
    rnd_mean = sum(rnd) / len(rnd) if rnd else None
    for k, v in res.items():
        v["speedup_vs_random_mean"] = rnd_mean / v["max_ms"] if rnd_mean else None
        v["speedup_vs_lookup_greedy"] = (res["lookup-greedy"]["max_ms"] / v["max_ms"]
                                         if "lookup-greedy" in res else None)
    out = {"workload": args.workload, "desc": desc, "shards": K, "batch": B, "weights": args.weights,
           "budget_rule": "1.6 x total / K (SPEC.md:620), bytes_per_param 2",
           "protocol": f"W={args.warmup} B={args.measure} R={args.trim}, L2 flushed, one shard at a time on 1 GPU",
           "random_max_ms_mean": rnd_mean, "plans": res}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps({k: {"max_ms": round(v["max_ms"], 3), "balance": round(v["balance"], 3),
                          "speedup_vs_random": v["speedup_vs_random_mean"] and round(v["speedup_vs_random_mean"], 3),
                          "speedup_vs_lookup_greedy": v["speedup_vs_lookup_greedy"] and round(v["speedup_vs_lookup_greedy"], 3)}
                      for k, v in res.items()}))


if __name__ == "__main__":
    main()
