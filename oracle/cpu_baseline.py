"""TEST INFRASTRUCTURE ONLY — the CPU baseline of bench.py.

Used by exactly two callers, as the baseline and never as the product:
``bench.py --impl reference`` (the reference arm) and the ``cpu_baseline`` leg
of bench.py's GPU arm. It never imports ``paper_2208_06399_b200``.

* Workloads are built with the REFERENCE's own generator (``oracle/_ref/libref.so``,
  the unmodified headers compiled in place: ``generate_pool`` tables.hpp:178-200,
  ``generate_workload`` tables.hpp:237-288), one table per call on a thread pool
  (subset stability, tests/test_tables.cpp:149-161, makes that bit-identical to
  one call over the whole pool). Without the reference build, the C restatement
  (``oracle/oracle.c``, pinned to the same goldens) generates them.
* The step is ``orc_cpu_step_f32`` (oracle/oracle.c): fp32 sum-pooled forward,
  row-bucketed radix sort, segment sum and exact row-wise Adagrad, OpenMP over
  every host thread in every phase. The reference has no embedding arithmetic
  (SURVEY.md §8c), so this port of the path is the CPU implementation timed.
* Every table of the workload is stepped — no sampling, no extrapolation. When
  host RAM cannot hold all dense tables at once, tables run in groups, one
  group resident at a time, and a step's time is the SUM of the groups'
  measured times (each group re-initialised outside the timed region).
* Timing protocol: W warm-up steps, K measured steps, sorted, R dropped at each
  end, mean (simcost.hpp:140-154).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import Oracle, Ref

WEIGHT_SEED = 0
LR, EPS = 0.01, 1e-8


def _gen(seed, n, **cfg):
    try:
        return Ref().generate_pool(seed, n, **cfg), "reference build (oracle/_ref/libref.so)"
    except RuntimeError:
        return Oracle().generate_pool(seed, n, **cfg), "oracle/oracle.c restatement"


def workload_tables(name):
    """(tables, batch, zipf, description) of a BASELINE config."""
    if name in ("cfg2", "cfg2u"):
        tables, src = _gen(0, 856)
        tables = tables[:50]
        for t in tables:
            t.dim = 128
            if name == "cfg2u":
                t.access_ratio = 1.0
        return tables, 65536, (1e-6 if name == "cfg2u" else 1.05), src
    if name == "cfg3":
        tables, src = _gen(0, 100, dim_choices=(32, 64, 128, 256))
        return tables, 65536, 1.05, src
    if name == "cfg4":
        tables, src = _gen(0, 856)
        return tables, 65536, 1.05, src
    if name == "cfg5":
        tables, src = _gen(0, 856, dim_choices=(64, 128, 192, 256))
        return tables, 131072, 1.05, src
    if name == "cfg1":
        tables, src = _gen(0, 10, dim_choices=(64,), pooling_mean_target=20.0)
        return tables, 512, 1.05, src
    raise ValueError(f"unknown workload {name}")


def generate_streams(tables, batch, zipf=1.05, threads=None):
    """{table_id: (offsets int64[B+1], indices int64[L])}, per table on a thread pool."""
    threads = threads or os.cpu_count() or 1
    try:
        ref = Ref()

        def one(t):
            h, d = ref.generate_workload(0, [t], batch, zipf)
            ref.free_workload(h)
            return d[t.id]
        src = "reference generate_workload (oracle/_ref/libref.so), per table"
    except RuntimeError:
        orc = Oracle()

        def one(t):
            return orc.generate_stream(0, t, batch, zipf)
        src = "oracle/oracle.c generate_stream (restatement), per table"
    with ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(one, tables))
    return {t.id: r for t, r in zip(tables, res)}, src


def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) * 1024
    except OSError:
        pass
    return 16 << 30


class CpuBaseline:
    """orc_cpu_step_f32 over ALL tables of a workload (grouped if RAM is short)."""

    def __init__(self, tables, streams, batch, threads=0, mem_fraction=0.6):
        self.o = Oracle()
        self.tables, self.B, self.threads = list(tables), int(batch), threads
        self.streams = streams
        budget = mem_fraction * mem_available()
        out_row = 4 * self.B  # bytes of one pooled column
        groups, cur, cur_b = [], [], 0
        for t in self.tables:
            L = len(streams[t.id][1])
            b = 4 * t.hash_size * (t.dim + 1) + out_row * t.dim + 16 * L
            if cur and cur_b + b > budget:
                groups.append(cur)
                cur, cur_b = [], 0
            cur.append(t)
            cur_b += b
        if cur:
            groups.append(cur)
        self.groups = groups
        self._resident = None
        self.cores = 1
        if len(groups) == 1:
            self._load(0)

    def _load(self, g):
        if self._resident == g:
            return
        self._state = None  # free the previous group first
        sub = self.groups[g]
        W = np.empty(sum(t.hash_size * t.dim for t in sub), dtype=np.float32)
        off = 0
        for t in sub:
            self.o.fill_weights(WEIGHT_SEED, t, W[off:off + t.hash_size * t.dim].reshape(t.hash_size, t.dim))
            off += t.hash_size * t.dim
        M = np.zeros(sum(t.hash_size for t in sub), dtype=np.float32)
        out = np.empty((self.B, sum(t.dim for t in sub)), dtype=np.float32)
        self._state = (sub, W, M, out, [self.streams[t.id] for t in sub])
        self._resident = g

    def step(self):
        """One full step over every table: seconds (sum over groups)."""
        total = 0.0
        for g in range(len(self.groups)):
            self._load(g)
            sub, W, M, out, st = self._state
            t0 = time.perf_counter()
            self.cores = self.o.cpu_step_f32([t.dim for t in sub], [t.hash_size for t in sub], self.B, st,
                                             W, M, out, LR, EPS, self.threads)
            total += time.perf_counter() - t0
        return total

    def run(self, warmup, steps, trim=None):
        """W/B/R protocol (simcost.hpp:140-154): -> (trimmed-mean s, all step times)."""
        for _ in range(warmup):
            self.step()
        ts = sorted(self.step() for _ in range(steps))
        r = trim if trim is not None else min(2, (steps - 1) // 2)
        kept = ts[r:len(ts) - r] if len(ts) - 2 * r >= 1 else ts
        return sum(kept) / len(kept), ts, r

    def describe(self):
        return (f"oracle/orc_cpu_step_f32 (fp32 fwd + row-bucketed radix sort + segment sum + row-wise Adagrad, "
                f"OpenMP over all phases) on all {len(self.tables)} tables, batch {self.B}"
                + (f", {len(self.groups)} resident groups (host RAM), step = sum of group times"
                   if len(self.groups) > 1 else ""))


def cpu_host():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model, "mem_available_gb": round(mem_available() / 1e9, 1)}
