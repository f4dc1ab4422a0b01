#!/usr/bin/env python
"""Benchmark of the B200 embedding-bag hot path (AutoShard, arXiv 2208.06399).

One "step" = one training pass of the multi-table pooled embedding bag over one
batch: K4 bag expansion -> sum-pooled forward -> (N>1: all-to-all of pooled
rows to the sample owners, loss 1/2|pooled|^2, all-to-all of the gradient back)
-> radix sort of the lookups by row -> segment-sum + exact row-wise Adagrad in
place. Metric: samples/s of the whole job (BASELINE.json).

  python bench.py                       # N=1, BASELINE cfg 2 (50 tables, dim 128, B=65536)
  torchrun --nproc-per-node N bench.py --gpus N   # cfg 4 (856 tables) sharded over N GPUs
  python bench.py --impl reference      # CPU baseline arm (oracle port, all host cores)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LR, EPS = 0.01, 1e-8
WEIGHT_SEED = 0
METRIC = "emb-bag fwd+bwd samples/s"


# ---------------------------------------------------------------------------
# workloads (all from the bit-exact reference generator)
# ---------------------------------------------------------------------------
def build_workload(P, name):
    if name == "cfg2":
        tables = P.generate_pool(0, 856)[:50]
        for t in tables:
            t.dim = 128
        return tables, 65536, "cfg2: generate_pool(0,856)[0:50], dim:=128, batch 65536, zipf 1.05"
    if name == "cfg2u":
        # SURVEY.md §8d uniform-access control: cfg2 with access_ratio = 1 and
        # zipf ~ 0, so gathered rows are nearly all distinct (DRAM-bound)
        tables = P.generate_pool(0, 856)[:50]
        for t in tables:
            t.dim = 128
            t.access_ratio = 1.0
        return tables, 65536, "cfg2u: cfg2 with access_ratio=1, zipf 1e-6 (uniform-access control)"
    if name == "cfg3":
        tables = P.generate_pool(0, 100, P.GeneratorConfig(dim_choices=(32, 64, 128, 256)))
        return tables, 65536, "cfg3: generate_pool(0,100,dims {32,64,128,256}), batch 65536"
    if name == "cfg4":
        return P.generate_pool(0, 856), 65536, "cfg4: generate_pool(0,856) dims {16,32}, batch 65536"
    if name == "cfg5":
        # unseen-table transfer: the AutoShard-RL plan is trained on tables 0..427 only
        return (P.generate_pool(0, 856, P.GeneratorConfig(dim_choices=(64, 128, 192, 256))), 131072,
                "cfg5: generate_pool(0,856,dims {64,128,192,256}), batch 131072 (RL trained on tables 0..427)")
    if name == "cfg1":
        tables = P.generate_pool(0, 10, P.GeneratorConfig(dim_choices=(64,), pooling_mean_target=20.0))
        return tables, 512, "cfg1: generate_pool(0,10,dim 64,pooling 20), batch 512"
    raise SystemExit(f"unknown workload {name}")


def same_workload_n1(wname):
    """N>1 runs use BASELINE cfg 4 while N=1 reports cfg 2 (the metric's
    single-GPU config): the committed N=1 line of THIS workload, so scaling can
    be read on one workload."""
    path = os.path.join(ROOT, "profiles", f"r1_bench_{wname}.json")
    try:
        d = json.load(open(path))
        return {"value": d["value"], "ms_per_step": d["ms_per_step"], "source": os.path.relpath(path, ROOT)}
    except Exception:
        return None


def bench_plan(P, task, wname, world):
    """The sharding plan of an N>1 run: the AutoShard-RL plan produced by the
    reference trainer for this config and shard count (plans/<cfg>_k<N>_autoshard_rl.assignment,
    oracle/rl_plans.cpp; BASELINE cfg 4 names the AutoShard-RL plan), else
    lookup-greedy (planners.hpp:73-107)."""
    for name in (f"{wname}_k{world}_autoshard_rl.assignment", f"{wname}_autoshard_rl.assignment"):
        path = os.path.join(ROOT, "plans", name)
        if os.path.exists(path):
            a = [int(x) for x in open(path).read().split()]
            if len(a) == len(task.tables) and max(a) < world:
                plan = P.ShardingPlan(a)
                if plan.feasible(task):
                    return plan, f"autoshard-rl (plans/{name}, reference trainer)"
    return P.greedy_shard(task, P.HeuristicKind.kLookupGreedy), "lookup-greedy (planners.hpp:73-107)"


def nominal_bytes(tables, B, L, U, wb=4):
    """SURVEY.md §8d algorithmic bytes (s = 4; weights wb = 4, or 2 for fp16
    storage): per-phase split that sums to FWD+BWD."""
    s = 4
    T = len(tables)
    SD = sum(t.dim for t in tables)
    LD = sum(l * t.dim for l, t in zip(L, tables))
    UD = sum(u * t.dim for u, t in zip(U, tables))
    Lt, Ut = sum(L), sum(U)
    phases = {
        "bag_expand": s * T * (B + 1),
        "fwd_segreduce": s * (Lt + B * SD) + wb * LD,
        "fwd_fixup": 0,
        "radix_sort": s * (Lt + T * (B + 1)),
        "bwd_segreduce_adagrad": s * LD + 2 * wb * UD + 2 * s * Ut,
        "bwd_fixup": 0,
    }
    fwd = s * (Lt + T * (B + 1) + B * SD) + wb * LD
    bwd = s * (Lt + T * (B + 1) + LD) + 2 * wb * UD + 2 * s * Ut
    return fwd, bwd, phases


def stream_stats(wl, tables):
    L, U = [], []
    for t in tables:
        idx = wl.find(t.id).indices
        L.append(int(len(idx)))
        U.append(int(np.count_nonzero(np.bincount(idx, minlength=1))) if len(idx) else 0)
    return L, U


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel, workload):
    """dram bytes/launch of `kernel` from the committed ncu --set full summary, if it matches."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(workload, {}).get(kernel)
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU baseline (oracle port; test infrastructure, only ever the checker/baseline)
# ---------------------------------------------------------------------------
class CpuSample:
    """oracle/orc_cpu_step_f32 (the CPU port of the path) on a prefix of the
    tables whose dense fp32 weights fit max_weight_bytes; times scale to the
    full workload by gathered bytes (sum L_t * dim_t)."""

    def __init__(self, tables, wl, B, max_weight_bytes=3 << 30, threads=0):
        from oracle import Oracle

        self.o = o = Oracle()
        sub, wb = [], 0
        for t in tables:
            b = t.hash_size * t.dim * 4
            if sub and wb + b > max_weight_bytes:
                continue
            sub.append(t)
            wb += b
            if wb > max_weight_bytes * 0.9:
                break
        self.W = np.empty(sum(t.hash_size * t.dim for t in sub), dtype=np.float32)
        off = 0
        for t in sub:
            o.fill_weights(WEIGHT_SEED, t, self.W[off:off + t.hash_size * t.dim].reshape(t.hash_size, t.dim))
            off += t.hash_size * t.dim
        self.M = np.zeros(sum(t.hash_size for t in sub), dtype=np.float32)
        self.out = np.empty((B, sum(t.dim for t in sub)), dtype=np.float32)
        self.streams = [(wl.find(t.id).offsets, wl.find(t.id).indices) for t in sub]
        self.dims = [t.dim for t in sub]
        self.hashes = [t.hash_size for t in sub]
        self.sub, self.tables, self.B, self.threads = sub, tables, B, threads
        ld_full = sum(len(wl.find(t.id).indices) * t.dim for t in tables)
        ld_sub = sum(len(s[1]) * t.dim for s, t in zip(self.streams, sub))
        self.scale = ld_full / max(1, ld_sub)
        self.cores = 1

    def step(self):
        t0 = time.perf_counter()
        self.cores = self.o.cpu_step_f32(self.dims, self.hashes, self.B, self.streams, self.W, self.M, self.out,
                                         LR, EPS, self.threads)
        return time.perf_counter() - t0

    def result(self, t_sample, n):
        sub = self.sub
        return {
            "value": round(self.B / (t_sample * self.scale), 2),
            "unit": "samples/s",
            "cores": self.cores,
            "kind": "port",
            "sample": (f"oracle/orc_cpu_step_f32 (fp32 fwd + radix-sort bwd + row-wise Adagrad, OpenMP) on "
                       f"{len(sub)}/{len(self.tables)} tables (ids {sub[0].id}..{sub[-1].id}), full batch {self.B}; "
                       f"median of {n} steps = {t_sample * 1e3:.1f} ms, scaled x{self.scale:.2f} by gathered bytes"),
            "host": cpu_host(),
        }


def cpu_sample(tables, wl, B, steps=3):
    cs = CpuSample(tables, wl, B)
    cs.step()  # warm-up
    t = statistics.median([cs.step() for _ in range(steps)])
    return cs.result(t, steps)


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
    return {"nproc": os.cpu_count(), "model": model}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="auto",
                    help="cfg1|cfg2|cfg2u|cfg3|cfg4 (auto: cfg2 at N=1, cfg4 at N>1)")
    ap.add_argument("--weights", choices=["fp32", "fp16"], default="fp32",
                    help="table storage (fp16 = bytes_per_param 2, as_create_ex AS_WEIGHTS_FP16; fp32 accumulation)")
    ap.add_argument("--plan-shard", type=int, default=-1,
                    help="N=1: run only this shard of the --plan-k GPU plan (AutoShard-RL if present)")
    ap.add_argument("--plan-k", type=int, default=8)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no clocks/e2e/cpu)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.profile_only:
        raise SystemExit("--warmup must be >= 3")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    wname = args.workload if args.workload != "auto" else ("cfg2" if world == 1 else "cfg4")

    if args.impl == "reference":
        return run_reference(args, world, rank, wname)

    import torch
    import torch.distributed as dist

    import paper_2208_06399_b200 as P

    # ASB_TEST_ONE_GPU=1 (functional test of the N>1 path on a 1-GPU box only):
    # every rank on cuda:0, gloo instead of NCCL. Never used for timings.
    one_gpu = os.environ.get("ASB_TEST_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    tables_all, B, wdesc = build_workload(P, wname)
    if world > 1:
        if B % world:
            raise SystemExit("batch must divide by the GPU count")
        budget = [int(180e9)] * world
        task = P.ShardingTask(tables_all, world, budget)
        plan, plan_name = bench_plan(P, task, wname, world)
        mine = [t for t, k in zip(tables_all, plan.assignment) if k == rank]
    elif args.plan_shard >= 0:
        # one shard of the K-GPU plan on this GPU (the per-GPU work of the K-GPU
        # run; the K-GPU box time is the max over its shards)
        task = P.ShardingTask(tables_all, args.plan_k, [int(180e9)] * args.plan_k)
        plan, plan_name = bench_plan(P, task, wname, args.plan_k)
        plan_name = f"shard {args.plan_shard} of {args.plan_k}: {plan_name}"
        mine = [t for t, k in zip(tables_all, plan.assignment) if k == args.plan_shard]
    else:
        plan_name = "single shard"
        mine = list(tables_all)

    zipf = 1e-6 if wname == "cfg2u" else 1.05
    wl = P.generate_workload(0, mine, B, zipf)  # subset-stable: identical to the full-pool streams
    wl.pin()
    L, U = stream_stats(wl, mine)
    shard = P.EmbeddingShard(mine, B, device=local, weight_seed=WEIGHT_SEED, weights=args.weights)
    shard.load(wl)
    stream = torch.cuda.current_stream()
    SD = shard.sum_dim
    pooled = shard.pooled_tensor()

    # N>1: table-wise shards; pooled rows go to their sample owners and the
    # gradient comes back with the inverse all-to-all (paper_2208_06399_b200.sharded)
    exchange = None
    if world > 1:
        from paper_2208_06399_b200.sharded import FusedPooledExchange, PooledExchange, a2a_layout

        lay = a2a_layout(task, plan, B)
        exch = None
        if os.environ.get("ASB_FUSED_A2A", "1") != "0":
            try:  # forward exchange fused into the forward kernel (peer stores, symmetric memory)
                exch = FusedPooledExchange(lay, rank, shard, device="cuda")
                exchange = "fused: pooled rows stored into the sample owners' symmetric-memory receive buffers by the " \
                           "forward kernel + device barrier; backward: NCCL all_to_all_single"
            except Exception as e:  # noqa: BLE001
                exchange = (f"NCCL all_to_all_single both ways (symmetric memory unavailable: "
                            f"{type(e).__name__}: {str(e).splitlines()[0][:160] if str(e) else ''})")
        if exch is None:
            exch = PooledExchange(lay, rank, device="cuda")
            exchange = exchange or "NCCL all_to_all_single both ways"

    xev = []  # (fwd a, fwd b, bwd a, bwd b) exchange events of the profiling pass

    def step(timed_exchange=False):
        if world > 1:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timed_exchange else None
            if isinstance(exch, FusedPooledExchange):
                recv = exch.forward(stream=stream)  # exchange inside K1/K4 + barrier
            else:
                shard.forward(pooled, stream=stream)
                if ev:
                    ev[0].record(stream)
                recv = exch.forward(pooled)
                if ev:
                    ev[1].record(stream)
            # dense part out of scope: loss 1/2|pooled|^2 -> dL/dpooled = pooled (recv)
            if ev:
                ev[2].record(stream)
            g = exch.backward(recv)
            if ev:
                ev[3].record(stream)
                xev.append(ev)
            shard.backward(g, LR, EPS, stream=stream)
        else:
            shard.forward(pooled, stream=stream)
            shard.backward(pooled, LR, EPS, stream=stream)

    props = torch.cuda.get_device_properties(local)
    l2 = getattr(props, "L2_cache_size", 126 << 20) or (126 << 20)
    flush_buf = torch.empty(2 * l2 // 4 + 1024, device="cuda", dtype=torch.float32)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    # ---- timed region: K steps, L2 flushed between steps (flush not timed) ----
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    shard.profile_read(reset=True)
    sampler = ClockSampler(local) if not args.profile_only else None
    if sampler:
        sampler.__enter__()
    barrier()
    for i in range(K):
        flush_buf.fill_(float(i))
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    barrier()
    if sampler:
        sampler.__exit__()
    _, launches = shard.profile_read(reset=True)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_local = sum(step_ms)
    tt = torch.tensor([t_local], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max = float(tt.item())  # ms over K steps, max over ranks
    ms_per_step = t_max / K
    value = B * K / (t_max / 1e3)

    # ---- per-kernel timing pass: events around each phase, phases serialized
    # (the sort's side-stream overlap off) so every kernel is timed alone ----
    shard.profile(True, serialize=True)
    for i in range(K):
        flush_buf.fill_(float(i))
        step(timed_exchange=True)
    torch.cuda.synchronize()
    exchange_stats = None
    if world > 1 and xev:
        # NCCL convention: busbw = (bytes one rank sends / t) * (G-1)/G; max t over ranks
        bwd_ms = sum(e[2].elapsed_time(e[3]) for e in xev) / len(xev)
        fwd_ms = (sum(e[0].elapsed_time(e[1]) for e in xev) / len(xev)
                  if not isinstance(exch, FusedPooledExchange) else None)
        tx = torch.tensor([bwd_ms, fwd_ms or 0.0], device="cuda", dtype=torch.float64)
        dist.all_reduce(tx, op=dist.ReduceOp.MAX)
        bwd_ms, fwd_max = float(tx[0]), float(tx[1])
        nbytes = 4 * B * max(lay.shard_dims)  # the largest owner's pooled block
        busbw = lambda ms: round(nbytes / (ms / 1e3) / 1e9 * (world - 1) / world, 1) if ms > 0 else None
        exchange_stats = {"bwd_a2a_ms": round(bwd_ms, 4), "bwd_busbw_gbs": busbw(bwd_ms),
                          "fwd_a2a_ms": round(fwd_max, 4) if fwd_ms is not None else "fused into K1/K4 (peer stores)",
                          "fwd_busbw_gbs": busbw(fwd_max) if fwd_ms is not None else None,
                          "bytes_per_rank_max": nbytes * (world - 1) // world}
    phase_ms, _ = shard.profile_read(reset=True)
    shard.profile(False)
    # shard time = this rank's own kernels (serialized phases, no exchange): the
    # paper's per-device cost C_k; max over ranks = max-shard time
    ts = torch.tensor([sum(phase_ms.values()) / K], device="cuda", dtype=torch.float64)
    shard_ms = [float(ts.item())]
    if world > 1:
        allt = [torch.zeros_like(ts) for _ in range(world)]
        dist.all_gather(allt, ts)
        shard_ms = [float(x.item()) for x in allt]
    fwd_b, bwd_b, phase_bytes = nominal_bytes(mine, B, L, U, wb=2 if args.weights == "fp16" else 4)
    peak, peak_kind = measured_peak_hbm()
    dom = max(phase_ms, key=phase_ms.get)
    dom_ms = phase_ms[dom] / K
    achieved = phase_bytes[dom] / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    traffic = (ncu_traffic(dom, wname) if world == 1 and args.weights == "fp32" and args.plan_shard < 0 else None)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "algorithmic_bytes_per_launch": phase_bytes[dom],
                "ms_per_launch": round(dom_ms, 4)}
    step_gbs = (fwd_b + bwd_b) / (ms_per_step / 1e3) / 1e9

    # ---- e2e through the public API: every step's int64 streams go host (pinned)
    # -> device. Pipelined like a training loop: batch i+1 is staged (H2D on the
    # copy engine) while batch i computes; commit = on-device pack + validation;
    # the loss of each step is read back (D2H) and the batch's validation checked ----
    e2e = None
    if not args.no_e2e and not args.profile_only:
        # bytes the staging pipeline copies host->device per step: int32 rows
        # and rebased int32 offsets (narrowed from the caller's int64 CSR on the
        # host), the per-batch table descriptors (~96 B each) and work maps
        info = shard.info()
        h2d = 4 * sum(L) + 4 * (len(mine) * B + 1) + 96 * len(mine) + 4 * int(info.n_chunks)
        d2h = 8 + 8

        def e2e_step():
            if world > 1:
                step()
                return torch.dot(exch.recv_buf, exch.recv_buf).mul_(0.5).item()
            return shard.step(LR, EPS, want_loss=True, stream=stream)

        shard.stage(wl)
        shard.commit(stream)
        for _ in range(2):  # warm-up of the pipelined loop
            shard.stage(wl)
            e2e_step()
            shard.commit(stream)
        shard.stage(wl)
        barrier()
        t0 = time.perf_counter()
        for i in range(K):
            loss = e2e_step()  # batch i (its H2D overlapped the previous step)
            shard.commit(stream)  # batch i+1 becomes current (waits for its copy)
            shard.stage(wl)  # batch i+2 -> copy engine, overlaps the next step
        shard.commit(stream)
        shard.check()  # drain: every copy issued in the region has landed
        barrier()
        te = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(B * K / float(te.item()), 1), "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": d2h, "ms_per_step": round(float(te.item()) * 1e3 / K, 3),
               "pipelined": "H2D of batch i+1 overlaps compute of batch i (as_stage_workload / as_commit_staged)",
               "loss_last": loss}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile_only:
        cpu = cpu_sample(mine, wl, B)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": round(value, 1),
            "unit": "samples/s",
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None,
            "dtype": "fp32" if args.weights == "fp32" else "fp32 (fp16 table storage)",
            "data": "synthetic (reference generator, bit-exact; weights: counter-hash grid init)",
            "config": {
                "workload": wname,
                "desc": wdesc,
                "tables": len(tables_all),
                "global_batch": B,
                "sum_dim": sum(t.dim for t in tables_all),
                "lookups": int(sum(L)) if world == 1 else None,
                "plan": plan_name,
                "weights": args.weights,
                "parallelism": "table-wise" if world > 1 else "single",
                "exchange": exchange,
                "step": "K4 bag-expand + fwd segreduce + fixup + radix sort + bwd segreduce/row-wise Adagrad + fixup"
                        + (" + pooled-row exchange both ways" if world > 1 else "") + "; grad = pooled (loss 1/2|pooled|^2)",
                "l2": "flushed (2x L2 fill) between timed steps, flush excluded from step time",
                "lr": LR,
                "eps": EPS,
            },
            "roofline": roofline,
            "step_roofline": {"bytes_fwd": fwd_b, "bytes_bwd": bwd_b, "achieved_gbs": round(step_gbs, 1),
                              "frac": round(step_gbs / peak, 4)},
            "phase_ms_per_step": {k: round(v / K, 4) for k, v in phase_ms.items()},
            "exchange_timing": exchange_stats,
            "same_workload_n1": same_workload_n1(wname) if world > 1 else None,
            "shard_ms_per_step": [round(x, 4) for x in shard_ms],
            "max_shard_ms": round(max(shard_ms), 4),
            "balance": round(min(shard_ms) / max(shard_ms), 4) if max(shard_ms) > 0 else 1.0,
            "gpu_launches": int(launches),
            "launches_per_step": launches / K,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": sampler.summary() if sampler else None,
            "step_ms_min_median_max": [round(min(step_ms), 4), round(statistics.median(step_ms), 4),
                                       round(max(step_ms), 4)],
        }
        print(json.dumps(line), flush=True)
    shard.close()
    if world > 1:
        dist.destroy_process_group()


def reference_pieces(P, tables, B, wl):
    """the reference's own CPU pieces on the path, timed single-threaded
    as the reference runs them (oracle/_ref/libref.so = the unmodified headers compiled
    in place), next to this repo's host equivalents on the same inputs."""
    try:
        from oracle import Ref, Table
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"}
    try:
        ref = Ref()
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)}
    otabs = [Table(t.id, t.dim, t.hash_size, t.pooling_mean, t.access_ratio, t.bytes_per_param) for t in tables]
    budgets = [sum(t.size_bytes() for t in tables)]
    out = {"threads": 1, "tables": len(tables), "batch": B}
    t0 = time.perf_counter()
    h, _ = ref.generate_workload(0, otabs, B)
    out["generate_workload_s"] = round(time.perf_counter() - t0, 3)
    t0 = time.perf_counter()
    ref.measure_plan(otabs, budgets, [0] * len(otabs), h)
    out["measure_plan_sim_s"] = round(time.perf_counter() - t0, 3)
    t0 = time.perf_counter()
    for k in (0, 1, 2):
        ref.greedy_shard(otabs, budgets, k)
    out["greedy_x3_s"] = round(time.perf_counter() - t0, 6)
    ref.free_workload(h)
    t0 = time.perf_counter()
    P.generate_workload(0, tables, B)
    out["ours_generate_workload_s"] = round(time.perf_counter() - t0, 3)
    out["ours_generate_workload_threads"] = os.cpu_count()
    return out


def run_reference(args, world, rank, wname):
    """CPU arm: the reference has no embedding arithmetic, so the
    reference-side implementation of the path is the oracle port (fp32, OpenMP,
    all host threads), timed on a bounded sample of the same workload."""
    if rank != 0:
        return
    import paper_2208_06399_b200 as P  # host generator only (no device calls)

    tables, B, wdesc = build_workload(P, wname)
    wl = P.generate_workload(0, tables, B)
    pieces = reference_pieces(P, tables, B, wl) if os.environ.get("ASB_REF_PIECES", "1") != "0" else None
    cs = CpuSample(tables, wl, B)
    for _ in range(args.warmup):
        cs.step()
    ts = [cs.step() for _ in range(args.steps)]
    cpu = cs.result(statistics.median(ts), len(ts))
    v = cpu["value"]
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 2),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(B / v * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic (reference generator, bit-exact)",
        "config": {"workload": wname, "desc": wdesc, "tables": len(tables), "global_batch": B},
        "cpu_baseline": cpu,
        "reference_pieces": pieces,
        "e2e": {"value": round(v, 2), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
