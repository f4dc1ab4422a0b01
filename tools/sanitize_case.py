#!/usr/bin/env python
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck) over every
kernel of the hot path (K1-K4 and the fixups, K2's packed and unpacked
passes): cfg 1, a long-bag / hot-row / empty-table case for narrow and wide
rows, fp16 storage, a backward with no forward, and subset contexts on a
parent's storage. Only this library's kernels run (no torch); results are checked
against the oracle so the sanitised runs are the correct path.

usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2208_06399_b200 as P  # noqa: E402
from helpers import to_oracle_tables  # noqa: E402
from oracle import Oracle  # noqa: E402


def streams_of(wl, tables):
    return [(wl.find(t.id).offsets, wl.find(t.id).indices) for t in tables]


def handmade(B, dim, chunk):
    rng = np.random.default_rng(0)
    hs = [5000, 70, 10, 1000]
    lens = [np.array([0, 20000, 1, 0, 0, chunk, chunk, 2 * chunk + 1] + [3] * (B - 8)),
            np.array([chunk - 1, 1, chunk + 1] + [0] * (B - 4) + [5000]),
            np.zeros(B, dtype=np.int64), rng.integers(0, 50, size=B)]
    st = []
    for t, ln in enumerate(lens):
        off = np.zeros(B + 1, dtype=np.int64)
        off[1:] = np.cumsum(ln)
        r = rng.integers(0, hs[t], size=int(off[-1])).astype(np.int64)
        r[: len(r) // 2] = 3 if t == 1 else 7
        st.append((off, r))
    return [P.TableDesc(id=10 + t, dim=dim, hash_size=h, pooling_mean=1.0) for t, h in enumerate(hs)], st


def run(tables, B, st, weights="fp32", fwd=True):
    o = Oracle()
    with P.EmbeddingShard(tables, B, weight_seed=3, weights=weights) as sh:
        sh.load(st)
        if fwd:
            sh.forward()
            got = sh.read_pooled()
            ref = o.forward_f64(to_oracle_tables(tables), B, st, wseed=3)
            assert np.array_equal(got.astype(np.float64), ref), "forward mismatch"
            sh.backward(None, 0.01, 1e-8)
        else:
            sh.step(0.01, 1e-8, want_loss=True)
            sh.load(st)
            import ctypes as C
            from paper_2208_06399_b200._capi import lib
            info = sh.info()
            # backward straight after a load, grad = the ctx's own pooled buffer
            P.errors.check(lib().as_backward_rowwise_adagrad(sh._h, C.c_void_p(info.pooled), 0.01, 1e-8, None))
        sh.features()
        sh.read_buffer(P.device.SORTED_ROWS)


def main():
    pool = P.generate_pool(0, 10, P.GeneratorConfig(dim_choices=(64,), pooling_mean_target=20.0))
    wl = P.generate_workload(0, pool, 512)
    run(pool, 512, streams_of(wl, pool))
    for dim, chunk in ((16, 32), (128, 256)):
        tables, st = handmade(64, dim, chunk)
        run(tables, 64, st)
    mixed = P.generate_pool(1, 6, P.GeneratorConfig(hash_size_max=5e4, pooling_mean_target=30.0))
    for t, d in zip(mixed, (8, 24, 64, 96, 256, 1024)):
        t.dim = d
    wl = P.generate_workload(2, mixed, 300)
    run(mixed, 300, streams_of(wl, mixed))
    half = [t for t in mixed if t.dim % 8 == 0]
    run(half, 300, streams_of(wl, half), weights="fp16")
    wl1 = P.generate_workload(0, pool, 512)  # keep the workload alive: the streams are views into it
    run(pool, 512, streams_of(wl1, pool), fwd=False)
    # subset contexts on a parent's storage, retargeted (the measured-cost hook)
    with P.EmbeddingShard(mixed, 300, weight_seed=3) as parent:
        sub = parent.subset([4, 1])
        for pos in ([4, 1], [0, 2, 5], [3]):
            sub.retarget(pos)
            sub.load(wl)
            sub.step(0.01, 1e-8, want_loss=True)
        sub.close()
    print("sanitize_case ok")


if __name__ == "__main__":
    main()
