#!/usr/bin/env python
"""Cross-check of the seed study's timing path: every shard of the
lookup-greedy cfg3 plan timed through a subset context on a resident parent
(as_create_subset / as_retarget_subset, what tools/rl_seed_study.py and the
RL hook use) and through a freshly created context per shard (as_measure_plan,
the reference-shaped hook). Same W/B/R, L2 flushed."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2208_06399_b200 as P  # noqa: E402
import bench  # noqa: E402

tables, B, _ = bench.build_workload(P, "cfg3")
wl = P.generate_workload(0, tables, B).pin()
total = sum(t.size_bytes() for t in tables)
task = P.ShardingTask(tables, 8, [int(1.6 * total / 8)] * 8)
plan = P.greedy_shard(task, P.HeuristicKind.kLookupGreedy)
fresh = P.measure_plan(plan, task, wl, P.BenchConfig(warmup=5, measure=10, trim=2))
sub_ms = []
with P.EmbeddingShard(tables, B) as parent:
    sub = None
    for m in plan.shard_member_indices(task):
        if sub is None:
            sub = parent.subset(m)
        else:
            sub.retarget(m)
        sub.load(wl)
        sub_ms.append(sub.measure(5, 10, 2))
    sub.close()
print(json.dumps({"fresh_ms": fresh, "subset_ms": sub_ms,
                  "ratio": [round(a / b, 4) for a, b in zip(sub_ms, fresh)]}))
