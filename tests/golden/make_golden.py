#!/usr/bin/env python
"""Regenerates tests/golden/golden.json and the small workload-file fixtures
from the UNMODIFIED reference compiled in place (oracle/_ref/libref.so, built
by oracle/Makefile from /root/reference/proj/include). Run in the container
that has /root/reference; the outputs are committed so tests need neither.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Oracle, Ref, Table, stream_hash  # noqa: E402


def plan_str(a):
    return "".join(map(str, a))


def main():
    r, o = Ref(), Oracle()
    g = {"source": "oracle/_ref/libref.so (reference headers compiled in place, -std=gnu++20 -O3 -ffp-contract=off)"}

    # cfg1
    pool1 = r.generate_pool(0, 10, dim_choices=(64,), pooling_mean_target=20.0)
    h1, w1 = r.generate_workload(0, pool1, 512)
    g["cfg1"] = {
        "pool": [vars(t) for t in pool1],
        "fingerprint_pool": f"{r.fingerprint_pool(pool1):016x}",
        "stream_hash": f"{stream_hash(o.fnv, [w1[t.id] for t in pool1]):016x}",
        "lookups": int(sum(len(w1[t.id][1]) for t in pool1)),
        "unique_rows": int(sum(len(np.unique(w1[t.id][1])) for t in pool1)),
        "table0_offsets_head": w1[pool1[0].id][0][:65].tolist(),
        "table0_indices_head": w1[pool1[0].id][1][:64].tolist(),
    }
    budget1 = [sum(t.dim * t.hash_size * t.bytes_per_param for t in pool1)] * 2
    g["cfg1"]["budget"] = budget1
    g["cfg1"]["plans"] = {k: plan_str(r.greedy_shard(pool1, budget1, i)) for i, k in
                          enumerate(["size", "dim", "lookup"])}
    g["cfg1"]["plans"]["random0"] = plan_str(r.random_shard(pool1, budget1, 0))
    g["cfg1"]["fingerprint_task"] = f"{r.fingerprint_task(pool1, budget1):016x}"
    # the reference's own cost hook (SIM measure_plan, exact and noisy)
    a = r.greedy_shard(pool1, budget1, 2)
    g["cfg1"]["sim_measure_plan_exact"] = r.measure_plan(pool1, budget1, a, h1, exact=True)
    g["cfg1"]["sim_measure_plan_noisy_seed0"] = r.measure_plan(pool1, budget1, a, h1, exact=False, seed=0)
    # tiny workload file written by the reference (format golden)
    small = r.generate_pool(4, 3, hash_size_min=50.0, hash_size_max=500.0, pooling_mean_target=3.0)
    hs, _ = r.generate_workload(9, small, 16)
    path = os.path.join(HERE, "ref_small.workload")
    r.lib.ref_save_workload_file(path.encode(), hs)
    g["small_workload"] = {"file": "ref_small.workload", "pool": [vars(t) for t in small], "seed": 9, "batch": 16}
    r.free_workload(hs)
    r.free_workload(h1)

    # cfg2: pool856[0:50], dim 128, B=65536
    pool856 = r.generate_pool(0, 856)
    g["pool856_fingerprint"] = f"{r.fingerprint_pool(pool856):016x}"
    p2 = [Table(t.id, 128, t.hash_size, t.pooling_mean, t.access_ratio, t.bytes_per_param) for t in pool856[:50]]
    h2, w2 = r.generate_workload(0, p2, 65536)
    budget2 = [sum(t.dim * t.hash_size * t.bytes_per_param for t in p2)] * 8
    g["cfg2"] = {
        "stream_hash": f"{stream_hash(o.fnv, [w2[t.id] for t in p2]):016x}",
        "lookups": int(sum(len(w2[t.id][1]) for t in p2)),
        "budget": budget2,
        "plans": {k: plan_str(r.greedy_shard(p2, budget2, i)) for i, k in enumerate(["size", "dim", "lookup"])},
    }
    g["cfg2"]["plans"]["random0"] = plan_str(r.random_shard(p2, budget2, 0))
    r.free_workload(h2)

    # canonical-build check
    h3, _ = r.generate_workload(0, pool856[:40], 4096)
    hh, nb = r.serialized_hash(pool856, h3)
    g["canonical"] = {"hash": f"{hh:016x}", "bytes": nb,
                      "what": "fnv1a64(save_pool(generate_pool(0,856)) || save_workload(generate_workload(0, first 40, 4096)))"}
    r.free_workload(h3)

    # SPEC.md:244 greedy fixture: costs [4,3,3,2,2] (lookup-greedy, dim 1), K=2 -> {4,2,2}, {3,3}
    spec = [Table(i, 1, 10, float(c), 1.0, 1) for i, c in enumerate([4, 3, 3, 2, 2])]
    g["spec_greedy"] = {"assignment": r.greedy_shard(spec, [10 ** 9, 10 ** 9], 2)}

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
