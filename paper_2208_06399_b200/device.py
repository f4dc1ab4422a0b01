"""The device hot path (L2): one shard of tables on one B200, and the GPU
``measure_plan`` that replaces the simulator (autoshard/simcost.hpp:60-204).

Everything here drives ``libautoshard_b200.so`` through the C-ABI; device
buffers handed in (pooled output, gradients) may be torch CUDA tensors or raw
device pointers. There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from ._capi import BenchConfigC, CtxInfoC, lib
from .errors import check
from .tables import ShardingPlan, ShardingTask, TableDesc, Workload, specs_to_c

# as_read_buffer selectors
POOLED, BAG_IDS, SORTED_ROWS, SORTED_BAGS, GLOBAL_ROWS = 0, 1, 2, 3, 4


def _ptr(x) -> Optional[int]:
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_cuda or not x.is_contiguous():
            raise ValueError("device buffers must be contiguous CUDA tensors")
        return x.data_ptr()
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


@dataclass
class BenchConfig:
    """simcost.hpp:163-171 plus the GPU knobs (L2 flush, Adagrad lr/eps, weight seed)."""

    warmup: int = 5
    measure: int = 10
    trim: int = 2
    exact: bool = False  # kept for signature parity; the GPU protocol is always measured
    seed: int = 0
    flush_l2: bool = True
    lr: float = 0.01
    eps: float = 1e-8

    def _c(self):
        return BenchConfigC(self.warmup, self.measure, self.trim, int(self.flush_l2), self.seed, self.lr, self.eps)


class EmbeddingShard:
    """One shard (a list of tables) resident on one device (``as_ctx``)."""

    def __init__(self, tables: Sequence[TableDesc], batch_size: int, device: int = 0, weight_seed: int = 0,
                 weights: str = "fp32"):
        """weights: "fp32" or "fp16" (as_create_ex AS_WEIGHTS_FP16: bytes_per_param 2 storage,
        fp32 accumulation and update)."""
        self.tables = list(tables)
        self.batch_size = int(batch_size)
        self.device = int(device)
        if weights not in ("fp32", "fp16"):
            raise ValueError(f"weights must be 'fp32' or 'fp16', got {weights!r}")
        self.weights = weights
        h = C.c_void_p()
        check(lib().as_create_ex(self.device, specs_to_c(self.tables), len(self.tables), self.batch_size,
                                 weight_seed, 1 if weights == "fp16" else 0, C.byref(h)))
        self._h = h
        self.sum_dim = sum(t.dim for t in self.tables)
        self.cols = np.cumsum([0] + [t.dim for t in self.tables])[:-1].tolist()

    def subset(self, positions: Sequence[int]) -> "EmbeddingShard":
        """A shard over some of this shard's tables (positions in its table
        order) on THIS shard's weight and momentum storage (as_create_subset):
        nothing is copied, steps through it update this shard's rows. Keep this
        shard alive while the subset is in use."""
        pos = [int(p) for p in positions]
        arr = (C.c_int32 * max(1, len(pos)))(*pos)
        h = C.c_void_p()
        check(lib().as_create_subset(self._h, arr, len(pos), C.byref(h)))
        sub = EmbeddingShard.__new__(EmbeddingShard)
        sub.tables = [self.tables[p] for p in pos]
        sub.batch_size, sub.device, sub.weights = self.batch_size, self.device, self.weights
        sub._h = h
        sub._parent = self  # storage owner
        import weakref

        self._subsets = getattr(self, "_subsets", []) + [weakref.ref(sub)]
        sub.sum_dim = sum(t.dim for t in sub.tables)
        sub.cols = np.cumsum([0] + [t.dim for t in sub.tables])[:-1].tolist()
        return sub

    def retarget(self, positions: Sequence[int]) -> None:
        """Subset shards only: switch to another subset of the same parent's
        tables (as_retarget_subset); load streams again afterwards."""
        pos = [int(p) for p in positions]
        arr = (C.c_int32 * max(1, len(pos)))(*pos)
        check(lib().as_retarget_subset(self._h, arr, len(pos)))
        self.tables = [self._parent.tables[p] for p in pos]
        self.sum_dim = sum(t.dim for t in self.tables)
        self.cols = np.cumsum([0] + [t.dim for t in self.tables])[:-1].tolist()

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        # communicators built on this shard (sharded.ShardComm) and subset
        # shards on its storage go first
        for c in list(getattr(self, "_comms", [])) + list(getattr(self, "_subsets", [])):
            c = c()
            if c is not None:
                c.close()
        if getattr(self, "_h", None) is not None and self._h.value:
            check(lib().as_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- data --------------------------------------------------------------
    def load(self, streams, stream=None) -> None:
        """streams: per table (in this shard's order) a pair (offsets int64[B+1], indices int64[L])."""
        if isinstance(streams, Workload):
            check(lib().as_load_workload(self._h, streams.handle, _stream(stream)))
            return
        st = [(np.ascontiguousarray(o, dtype=np.int64), np.ascontiguousarray(i, dtype=np.int64)) for o, i in streams]
        if len(st) != len(self.tables):
            raise ValueError(f"expected {len(self.tables)} streams, got {len(st)}")
        n = max(1, len(st))
        po = (C.c_void_p * n)(*[o.ctypes.data for o, _ in st])
        pi = (C.c_void_p * n)(*[i.ctypes.data for _, i in st])
        ni = (C.c_int64 * n)(*[len(i) for _, i in st])
        check(lib().as_load_streams(self._h, po, pi, ni, _stream(stream)))
        self._keep = st

    def stage(self, streams) -> None:
        """Asynchronously copy the next batch to the device (see as_stage_streams)."""
        # the native staging job reads the host arrays until the matching commit:
        # keep them (the Workload object or the converted arrays) alive until then
        if isinstance(streams, Workload):
            check(lib().as_stage_workload(self._h, streams.handle))
            self._staged_keep = getattr(self, "_staged_keep", [])[-1:] + [streams]
            return
        st = [(np.ascontiguousarray(o, dtype=np.int64), np.ascontiguousarray(i, dtype=np.int64)) for o, i in streams]
        if len(st) != len(self.tables):
            raise ValueError(f"expected {len(self.tables)} streams, got {len(st)}")
        n = max(1, len(st))
        po = (C.c_void_p * n)(*[o.ctypes.data for o, _ in st])
        pi = (C.c_void_p * n)(*[i.ctypes.data for _, i in st])
        ni = (C.c_int64 * n)(*[len(i) for _, i in st])
        check(lib().as_stage_streams(self._h, po, pi, ni))
        self._staged_keep = getattr(self, "_staged_keep", [])[-1:] + [st]

    def commit(self, stream=None) -> None:
        """Pack + validate the oldest staged batch on `stream`; it becomes current."""
        check(lib().as_commit_staged(self._h, _stream(stream)))

    def check(self) -> None:
        """Report OffsetError / IndexError of the last committed batch (synchronises)."""
        check(lib().as_check_batch(self._h))

    # -- compute -----------------------------------------------------------
    def forward(self, out=None, stream=None) -> None:
        check(lib().as_forward(self._h, _ptr(out), _stream(stream)))

    def set_peer_outputs(self, bases, rows) -> None:
        """Fused forward exchange (as_set_peer_outputs[_v]): pooled row b goes to
        bases[q] for the peer q whose sample range holds b. rows: rows per peer
        (int, even split) or the row_start list (len(bases) + 1 entries, uneven
        splits); bases=[] restores the local output."""
        n = len(bases)
        arr = (C.c_void_p * max(1, n))(*[int(b) for b in bases])
        if isinstance(rows, int):
            check(lib().as_set_peer_outputs(self._h, n, arr, int(rows) if n else 0))
        else:
            st = (C.c_int64 * (n + 1))(*[int(x) for x in rows]) if n else None
            check(lib().as_set_peer_outputs_v(self._h, n, arr, st))

    def backward(self, grad=None, lr: float = 0.01, eps: float = 1e-8, stream=None) -> None:
        check(lib().as_backward_rowwise_adagrad(self._h, _ptr(grad), lr, eps, _stream(stream)))

    def step(self, lr: float = 0.01, eps: float = 1e-8, want_loss: bool = False, stream=None) -> Optional[float]:
        loss = C.c_double()
        check(lib().as_step(self._h, lr, eps, C.byref(loss) if want_loss else None, _stream(stream)))
        return loss.value if want_loss else None

    def measure(self, warmup=5, measure=10, trim=2, flush_l2=True, lr=0.01, eps=1e-8) -> float:
        ms = C.c_double()
        check(lib().as_measure(self._h, warmup, measure, trim, int(flush_l2), lr, eps, C.byref(ms)))
        return ms.value

    # -- profiling ---------------------------------------------------------
    PHASES = ("bag_expand", "fwd_segreduce", "fwd_fixup", "radix_sort", "bwd_segreduce_adagrad", "bwd_fixup")

    def profile(self, enable: bool = True, serialize: bool = False) -> None:
        """Per-phase event timing; serialize=True runs the sort inside the backward (no overlap)."""
        check(lib().as_profile_enable(self._h, (2 if serialize else 1) if enable else 0))

    def profile_read(self, reset: bool = True):
        """-> ({phase: ms accumulated}, kernel launches) since the last reset."""
        ms = (C.c_double * len(self.PHASES))()
        n = C.c_int64()
        check(lib().as_profile_read(self._h, ms, C.byref(n), int(reset)))
        return dict(zip(self.PHASES, list(ms))), n.value

    def features(self, stream=None) -> np.ndarray:
        """[n_tables, 21] raw cost-model features (extract_features, tables.hpp:344-386) on the GPU."""
        out = np.zeros((max(1, len(self.tables)), 21), dtype=np.float64)
        check(lib().as_table_features(self._h, out.ctypes.data_as(C.POINTER(C.c_double)), _stream(stream)))
        return out[: len(self.tables)]

    # -- introspection / readback -------------------------------------------
    def info(self) -> CtxInfoC:
        i = CtxInfoC()
        check(lib().as_ctx_info_get(self._h, C.byref(i)))
        return i

    def read_pooled(self) -> np.ndarray:
        a = np.empty((self.batch_size, self.sum_dim), dtype=np.float32)
        check(lib().as_read_buffer(self._h, POOLED, a.ctypes.data, a.nbytes))
        return a

    def read_buffer(self, what: int) -> np.ndarray:
        n = self.info().n_lookups
        a = np.empty(n, dtype=np.int32)
        check(lib().as_read_buffer(self._h, what, a.ctypes.data, a.nbytes))
        return a

    def read_rows(self, t: int, rows) -> np.ndarray:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((len(r), self.tables[t].dim), dtype=np.float32)
        check(lib().as_read_rows(self._h, t, r.ctypes.data_as(C.POINTER(C.c_int64)), len(r),
                                 out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def read_momentum(self, t: int, rows) -> np.ndarray:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(len(r), dtype=np.float32)
        check(lib().as_read_momentum(self._h, t, r.ctypes.data_as(C.POINTER(C.c_int64)), len(r),
                                     out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def write_table(self, t: int, weights=None, momentum=None) -> None:
        pw = pm = None
        if weights is not None:
            weights = np.ascontiguousarray(weights, dtype=np.float32)
            pw = weights.ctypes.data_as(C.POINTER(C.c_float))
        if momentum is not None:
            momentum = np.ascontiguousarray(momentum, dtype=np.float32)
            pm = momentum.ctypes.data_as(C.POINTER(C.c_float))
        check(lib().as_write_table(self._h, t, pw, pm))

    def pooled_tensor(self):
        """torch view of the shard's device pooled buffer [B, sum_dim] (no copy)."""
        import torch

        info = self.info()

        class _CAI:
            __cuda_array_interface__ = {
                "shape": (self.batch_size, self.sum_dim),
                "typestr": "<f4",
                "data": (int(info.pooled), False),
                "version": 3,
                "strides": None,
            }

        return torch.as_tensor(_CAI(), device=f"cuda:{self.device}")


def probe_gather_bw(footprint_bytes: int, row_bytes: int, device: int = 0) -> float:
    """GB/s of random row gathers over a device buffer (as_probe_gather_bw): the
    measured gather ceiling bench.py reports the seg_reduce kernels against."""
    g = C.c_double()
    check(lib().as_probe_gather_bw(int(device), int(footprint_bytes), int(row_bytes), C.byref(g)))
    return g.value


def measure_plan(plan: ShardingPlan, task: ShardingTask, wl: Workload, bench: Optional[BenchConfig] = None,
                 devices: Optional[Sequence[int]] = None) -> List[float]:
    """measure_plan (simcost.hpp:194-204) on real kernels: per-shard ms."""
    bench = bench or BenchConfig()
    plan.validate(task)
    a = (C.c_int32 * max(1, len(plan.assignment)))(*plan.assignment)
    devs = list(devices) if devices else [0]
    d = (C.c_int32 * len(devs))(*devs)
    out = (C.c_double * task.num_shards)()
    bc = bench._c()
    check(lib().as_measure_plan(specs_to_c(task.tables), len(task.tables), task.num_shards, a, wl.handle, d,
                                len(devs), C.byref(bc), out))
    return list(out)
