#!/usr/bin/env python
"""Store the bench's AutoShard-RL plans as fingerprinted plan files.

The reference trainer (oracle/rl_plans.cpp) writes a bare assignment list;
bench.py consumes "autoshard-plan 1" files (as_plan_save / as_plan_load,
task fingerprint tables.hpp:417-441) made for the DEVICE task: fp32 bytes per
parameter and the per-GPU table budget of bench.device_task. A plan file made
for another pool, shard count or budget is rejected at load.

usage: python tools/make_bench_plans.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2208_06399_b200 as P  # noqa: E402

PLANS = [("cfg4", 2), ("cfg4", 4), ("cfg4", 8), ("cfg3", 8), ("cfg5", 8)]


def main():
    for wname, k in PLANS:
        src = os.path.join(ROOT, "plans", f"{wname}_k{k}_autoshard_rl.assignment")
        if not os.path.exists(src):
            src = os.path.join(ROOT, "plans", f"{wname}_autoshard_rl.assignment")
        a = [int(x) for x in open(src).read().split()]
        tables, _, _ = bench.build_workload(P, wname)
        task = bench.device_task(P, tables, k)
        plan = P.ShardingPlan(a)
        plan.validate(task)
        used = plan.mem_used(task)
        print(wname, k, "feasible" if plan.feasible(task) else "INFEASIBLE", [round(u / 1e9, 1) for u in used])
        dst = os.path.join(ROOT, "plans", f"{wname}_k{k}_autoshard_rl.plan")
        P.save_plan(dst, task, plan)
        back, _ = P.load_plan(dst, task)
        assert back.assignment == a
        print("  ->", os.path.relpath(dst, ROOT), "from", os.path.relpath(src, ROOT))


if __name__ == "__main__":
    main()
