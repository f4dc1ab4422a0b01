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


def device_task(P, tables, K, weights="fp32"):
    """The ShardingTask the bench places tables with: bytes_per_param = the
    device's storage bytes (4 fp32 / 2 fp16, tables.hpp:30), per-GPU budget =
    HBM left for the tables after momentum, pooled buffers and workspaces."""
    import copy

    tabs = [copy.copy(t) for t in tables]
    for t in tabs:
        t.bytes_per_param = 4 if weights == "fp32" else 2
    return P.ShardingTask(tabs, K, [PLAN_BUDGET_BYTES] * K)


PLAN_BUDGET_BYTES = 160_000_000_000  # of the B200's 180 GB: tables; the rest is momentum, pooled rows, scratch


def bench_plan(P, task, wname, world):
    """The sharding plan of an N>1 run: the AutoShard-RL plan of the reference
    trainer for this config and shard count, stored as a fingerprinted plan
    file (plans/<cfg>_k<N>_autoshard_rl.plan, "autoshard-plan 1" format,
    loaded with as_plan_load which rejects a plan made for another task);
    else lookup-greedy (planners.hpp:73-107). Either must be feasible for the
    device task (fp32 bytes per parameter)."""
    path = os.path.join(ROOT, "plans", f"{wname}_k{world}_autoshard_rl.plan")
    if os.path.exists(path):
        plan, _ = P.load_plan(path, task)
        if not plan.feasible(task):
            raise SystemExit(f"{path}: plan does not fit the per-GPU budget")
        return plan, f"autoshard-rl ({os.path.relpath(path, ROOT)}, reference trainer, fingerprint checked)"
    plan = P.greedy_shard(task, P.HeuristicKind.kLookupGreedy)
    return plan, "lookup-greedy (planners.hpp:73-107)"


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


def common_config(wname, n_tables, B):
    """The `config` both arms print (identical by construction)."""
    return {"workload": wname, "tables": n_tables, "global_batch": B,
            "l2": "GPU arm: L2 flushed (2x L2 fill) between timed steps, flush not timed; "
                  "CPU arm: dense tables (>= 33 GB) far larger than the host caches"}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s, an earlier measurement on this pool)"


def sources_sha():
    """Identity of the native build: sha256 over the library's CUDA/C++ sources
    and the C-ABI header. An ncu summary carries the sha of the sources it was
    captured on; bench.py uses its DRAM bytes only when they match."""
    import hashlib

    h = hashlib.sha256()
    base = os.path.join(ROOT, "paper_2208_06399_b200", "csrc")
    files = []
    for dp, dn, fs in os.walk(base):
        dn[:] = sorted(d for d in dn if d != "build")
        files += [os.path.join(dp, f) for f in fs if f.endswith((".cu", ".cuh", ".hpp", ".cpp", ".h")) or f == "Makefile"]
    files.append(os.path.join(ROOT, "include", "autoshard_b200.h"))
    for path in sorted(files):
        h.update(os.path.relpath(path, ROOT).encode())
        with open(path, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel, workload, sha):
    """DRAM bytes (read + write) per launch of `kernel` from profiles/ncu_traffic.json
    (tools/ncu_summary.py over an `ncu --set full` capture) when the capture was
    taken on these sources; else (None, why)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f).get(workload)
    except Exception:
        return None, "no profiles/ncu_traffic.json"
    if not d or "kernels" not in d:
        return None, f"no ncu capture of {workload}"
    if d.get("sources_sha") != sha:
        return None, f"ncu capture of {workload} is from other sources ({d.get('sources_sha')} != {sha})"
    e = d["kernels"].get(kernel)
    if not e:
        return None, f"ncu capture of {workload} has no {kernel}"
    return float(e["dram_bytes_per_launch"]), f"profiles/{e['summary']} (sources {sha})"


def compulsory_bytes(tables, B, L, U, passes, wb=4):
    """Per-phase MINIMUM DRAM traffic: every distinct weight row, gradient row
    and index read or written once (the §8d nominal model counts every gather)."""
    s = 4
    T = len(tables)
    SD = sum(t.dim for t in tables)
    UD = sum(u * t.dim for u, t in zip(U, tables))
    Lt, Ut = sum(L), sum(U)
    return {
        "bag_expand": s * (T * (B + 1) + Lt),
        "fwd_segreduce": s * (2 * Lt + B * SD) + wb * UD,
        "fwd_fixup": 0,
        "radix_sort": s * Lt + sum(16 * l * p for l, p in zip(L, passes)),
        "bwd_segreduce_adagrad": s * (2 * Lt + B * SD) + 2 * wb * UD + 2 * s * Ut,
        "bwd_fixup": 0,
    }


def sort_passes(tables):
    return [max(1, (max(1, (t.hash_size - 1).bit_length()) + 7) // 8) for t in tables]


# ---------------------------------------------------------------------------
# CPU baseline (oracle/cpu_baseline.py: test infrastructure, the baseline only)
# ---------------------------------------------------------------------------
def cpu_baseline_leg(tables, wl, B, warmup=1, steps=3):
    """GPU arm's cpu_baseline: the CPU port on ALL of this run's tables and the
    same streams (bounded by steps, not by sampling tables)."""
    from oracle.cpu_baseline import CpuBaseline, cpu_host

    streams = {t.id: (wl.find(t.id).offsets, wl.find(t.id).indices) for t in tables}
    cb = CpuBaseline(tables, streams, B)
    mean, ts, r = cb.run(warmup, steps, trim=0)
    med = statistics.median(ts)
    return {"value": round(B / med, 2), "unit": "samples/s", "cores": cb.cores, "kind": "port",
            "sample": f"{cb.describe()}; {warmup} warm-up + median of {steps} steps = {med * 1e3:.1f} ms/step",
            "host": cpu_host()}


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
    ap.add_argument("--exchange", choices=["peer", "peer-fwd", "nccl"], default="peer",
                    help="N>1 pooled-row exchange: peer memory both ways (fused forward), fused forward + NCCL "
                         "backward, or NCCL both ways")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kjt", action="store_true",
                    help="N>1: also time e2e with the input-side KJT all-to-all (as_load_streams_exchanged): every "
                         "rank starts from ITS samples of ALL tables (PAPER.md:169)")
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
        task = device_task(P, tables_all, world, args.weights)
        plan, plan_name = bench_plan(P, task, wname, world)
        mine = [t for t, k in zip(tables_all, plan.assignment) if k == rank]
    elif args.plan_shard >= 0:
        # one shard of the K-GPU plan on this GPU (the per-GPU work of the K-GPU
        # run; the K-GPU box time is the max over its shards)
        task = device_task(P, tables_all, args.plan_k, args.weights)
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

    # N>1: table-wise shards through the C-ABI's sharded step (as_comm,
    # csrc/cuda/sharded.cu): pooled rows go to their sample owners (forward
    # exchange fused into the forward kernel's epilogues over peer memory, or
    # NCCL), the gradient comes back with the inverse exchange, K2/K3 run on
    # the table owner
    exchange = None
    comm = None
    if world > 1:
        from paper_2208_06399_b200.sharded import a2a_layout, connect

        lay = a2a_layout(task, plan, B)
        modes = {"peer": 0, "peer-fwd": 2, "nccl": 3}
        mode = modes[args.exchange] if not one_gpu else 0
        comm = connect(shard, lay, rank, world, mode=mode, use_nccl=not one_gpu, host_barrier=one_gpu)
        exchange = {
            0: "forward fused into K4/K1 epilogues (NVLink peer stores into the owners' receive buffers) + "
               "system-scope device barrier; backward: gradient blocks pushed to the table owners by copy engines "
               "over peer memory + barrier",
            2: "forward fused into K4/K1 epilogues (peer stores) + device barrier; backward: NCCL send/recv",
            3: "NCCL grouped send/recv both ways",
        }[mode] + f" (as_step_sharded; samples split {lay.row_start[1] - lay.row_start[0]}..{lay.rows(world - 1)} per rank)"

    def step():
        if world > 1:
            comm.step(LR, EPS, stream=stream)  # dense part out of scope: loss 1/2|recv|^2, grad = recv
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
        step()
    torch.cuda.synchronize()
    exchange_stats = None
    if world > 1:
        fwd_x, bwd_x = comm.profile_read(reset=True)
        tx = torch.tensor([fwd_x / K, bwd_x / K], device="cuda", dtype=torch.float64)
        dist.all_reduce(tx, op=dist.ReduceOp.MAX)
        ci = comm.info()
        nb = torch.tensor([float(ci.bytes_sent_fwd), float(ci.bytes_sent_bwd)], device="cuda", dtype=torch.float64)
        dist.all_reduce(nb, op=dist.ReduceOp.MAX)
        fwd_ms, bwd_ms = float(tx[0]), float(tx[1])
        # NCCL convention: busbw of a rank = bytes it sends to the others / t (max t, max bytes over ranks)
        busbw = lambda nbytes, ms: round(nbytes / (ms / 1e3) / 1e9, 1) if ms > 0 else None
        exchange_stats = {"fwd_exchange_ms": round(fwd_ms, 4), "bwd_exchange_ms": round(bwd_ms, 4),
                          "fwd_bytes_per_rank_max": int(nb[0]), "bwd_bytes_per_rank_max": int(nb[1]),
                          "fwd_busbw_gbs": busbw(float(nb[0]), fwd_ms) if mode & 1 else None,
                          "bwd_busbw_gbs": busbw(float(nb[1]), bwd_ms),
                          "note": ("fwd_exchange_ms of the fused forward is the device-barrier wait after K1 (the "
                                   "peer stores ride in K1/K4); it includes waiting for the slowest rank"
                                   if not mode & 1 else "NCCL send/recv time")}
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
    wbytes = 2 if args.weights == "fp16" else 4
    comp = compulsory_bytes(mine, B, L, U, sort_passes(mine), wb=wbytes)
    prof_key = wname if (world == 1 and args.plan_shard < 0) else f"{wname}_k{world if world > 1 else args.plan_k}s{rank if world > 1 else args.plan_shard}"
    if args.weights != "fp32":
        prof_key += "_fp16"
    traffic, traffic_src = ncu_traffic(dom, prof_key, sources_sha())
    gbs = lambda nbytes: nbytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    # roofline: HBM bytes the kernel actually moved (ncu DRAM read+write of this
    # build) over its live launch time; with no matching capture, its
    # compulsory bytes (a lower bound of the DRAM traffic). The §8d nominal
    # bytes count every gathered row and mostly hit L1/L2 at Zipf access:
    # reported against the MEASURED L2 random-gather ceiling instead.
    row_bytes = min(512, max(16, 1 << (max(t.dim for t in mine) * wbytes - 1).bit_length())) if mine else 512
    l2_peak = hbm_gather = None
    if os.environ.get("ASB_BENCH_PROBE", "1") != "0":
        try:
            l2_peak = P.probe_gather_bw(min(64 << 20, int(l2 // 2)), row_bytes, device=local)
            hbm_gather = P.probe_gather_bw(8 << 30, row_bytes, device=local)
        except Exception:  # noqa: BLE001
            l2_peak = hbm_gather = None
    hbm_bytes = traffic if traffic is not None else comp[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(gbs(hbm_bytes), 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(gbs(hbm_bytes) / peak, 4),
                "traffic": traffic,
                "achieved_basis": ("ncu DRAM bytes per launch, " + traffic_src) if traffic is not None else
                                  f"compulsory bytes per launch ({traffic_src})",
                "ms_per_launch": round(dom_ms, 4),
                "compulsory_bytes_per_launch": comp[dom],
                "algorithmic_bytes_per_launch": phase_bytes[dom],
                "nominal_gbs": round(gbs(phase_bytes[dom]), 1),
                "l2_gather_peak_gbs": round(l2_peak, 1) if l2_peak else None,
                "hbm_gather_peak_gbs": round(hbm_gather, 1) if hbm_gather else None,
                "gather_row_bytes": row_bytes,
                "l2_frac": round(gbs(phase_bytes[dom]) / l2_peak, 4) if l2_peak else None}
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
                return comm.step(LR, EPS, want_loss=True, stream=stream)
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

    # ---- e2e with the input-side exchange (opt-in): each rank's loader holds
    # its samples of EVERY table; the indices reach the table owners through
    # as_load_streams_exchanged (NCCL), then the sharded step ----
    e2e_kjt = None
    if args.kjt and world > 1 and not one_gpu and not args.profile_only:
        try:
            from paper_2208_06399_b200.sharded import local_batch

            wl_all = P.generate_workload(0, tables_all, B, zipf)
            full = [(wl_all.find(t.id).offsets, wl_all.find(t.id).indices) for t in tables_all]
            local = local_batch(full, lay.row_start, rank)
            del full, wl_all
            owner = list(plan.assignment)
            h2d_k = sum(4 * (len(o) - 1) + 4 * len(i) for o, i in local)
            for _ in range(2):
                comm.load_exchanged(tables_all, owner, local, stream=stream)
                comm.step(LR, EPS, want_loss=True, stream=stream)
            barrier()
            t0 = time.perf_counter()
            for _ in range(K):
                comm.load_exchanged(tables_all, owner, local, stream=stream)
                loss_k = comm.step(LR, EPS, want_loss=True, stream=stream)
            barrier()
            te = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e_kjt = {"value": round(B * K / float(te.item()), 1), "unit": "samples/s",
                       "h2d_bytes_per_step": int(h2d_k), "d2h_bytes_per_step": 16,
                       "ms_per_step": round(float(te.item()) * 1e3 / K, 3), "loss_last": loss_k,
                       "path": "local mini-batch of all tables -> validate, pack, H2D, NCCL grouped send/recv, "
                               "on-device assembly (as_load_streams_exchanged) -> as_step_sharded; not pipelined"}
        except Exception as e:  # noqa: BLE001  (reported, never silently replaced)
            e2e_kjt = {"error": f"{type(e).__name__}: {e}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile_only:
        cpu = cpu_baseline_leg(mine, wl, B)

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
            "config": common_config(wname, len(tables_all), B),
            "setup": {
                "desc": wdesc,
                "sum_dim": sum(t.dim for t in tables_all),
                "lookups": int(sum(L)) if world == 1 else None,
                "plan": plan_name,
                "weights": args.weights,
                "parallelism": "table-wise" if world > 1 else "single",
                "exchange": exchange,
                "step": "K4 bag-expand + fwd segreduce + fixup + radix sort + bwd segreduce/row-wise Adagrad + fixup"
                        + (" + pooled-row exchange both ways" if world > 1 else "") + "; grad = pooled (loss 1/2|pooled|^2)",
                "lr": LR,
                "eps": EPS,
                "sources_sha": sources_sha(),
            },
            "roofline": roofline,
            "step_roofline": {"bytes_fwd": fwd_b, "bytes_bwd": bwd_b, "achieved_gbs": round(step_gbs, 1),
                              "frac": round(step_gbs / peak, 4)},
            "phase_ms_per_step": {k: round(v / K, 4) for k, v in phase_ms.items()},
            "exchange_timing": exchange_stats,
            "shard_ms_per_step": [round(x, 4) for x in shard_ms],
            "max_shard_ms": round(max(shard_ms), 4),
            "balance": round(min(shard_ms) / max(shard_ms), 4) if max(shard_ms) > 0 else 1.0,
            "gpu_launches": int(launches),
            "launches_per_step": launches / K,
            "e2e": e2e,
            "e2e_kjt": e2e_kjt,
            "cpu_baseline": cpu,
            "clocks": sampler.summary() if sampler else None,
            "step_ms_min_median_max": [round(min(step_ms), 4), round(statistics.median(step_ms), 4),
                                       round(max(step_ms), 4)],
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    shard.close()
    if world > 1:
        dist.destroy_process_group()


def reference_pieces(tables, B, streams_src):
    """the reference's own CPU pieces on the path, single-threaded
    as the reference runs them (oracle/_ref/libref.so = the unmodified headers
    compiled in place)."""
    try:
        from oracle import Ref
        ref = Ref()
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"}
    budgets = [sum(t.dim * t.hash_size * t.bytes_per_param for t in tables)]
    out = {"threads": 1, "tables": len(tables), "batch": B}
    t0 = time.perf_counter()
    h, _ = ref.generate_workload(0, tables, B)
    out["generate_workload_s"] = round(time.perf_counter() - t0, 3)
    t0 = time.perf_counter()
    ref.measure_plan(tables, budgets, [0] * len(tables), h)
    out["measure_plan_sim_s"] = round(time.perf_counter() - t0, 3)
    t0 = time.perf_counter()
    for k in (0, 1, 2):
        ref.greedy_shard(tables, budgets, k)
    out["greedy_x3_s"] = round(time.perf_counter() - t0, 6)
    ref.free_workload(h)
    return out


def run_reference(args, world, rank, wname):
    """Reference arm: the reference has no embedding arithmetic,
    so the CPU implementation of the path is the oracle port, stepped over
    EVERY table of the workload on all host threads, with the W/B/R protocol
    (simcost.hpp:140-154). Tables and streams come from the reference's own
    generator (oracle/_ref); nothing of paper_2208_06399_b200 is imported."""
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuBaseline, cpu_host, generate_streams, workload_tables

    tables, B, zipf, tsrc = workload_tables(wname)
    t0 = time.perf_counter()
    streams, ssrc = generate_streams(tables, B, zipf)
    gen_s = time.perf_counter() - t0
    pieces = (reference_pieces(tables, B, ssrc) if wname in ("cfg1", "cfg2") and os.environ.get("ASB_REF_PIECES", "1") != "0"
              else None)
    cb = CpuBaseline(tables, streams, B)
    trim = min(2, (args.steps - 1) // 2)
    mean, ts, r = cb.run(args.warmup, args.steps, trim=trim)
    v = B / mean
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 2),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(mean * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": f"synthetic (tables: {tsrc}; streams: {ssrc})",
        "config": common_config(wname, len(tables), B),
        "cpu_baseline": {"value": round(v, 2), "unit": "samples/s", "cores": cb.cores, "kind": "port",
                         "sample": f"{cb.describe()}; W={args.warmup}, B={args.steps}, R={r}: trimmed mean "
                                   f"{mean * 1e3:.1f} ms/step (min {ts[0] * 1e3:.1f}, max {ts[-1] * 1e3:.1f})",
                         "host": cpu_host()},
        "step_s_sorted": [round(x, 4) for x in ts],
        "generate_s": round(gen_s, 2),
        "reference_pieces": pieces,
        "e2e": {"value": round(v, 2), "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
