"""L1 host types and the synthetic generator (autoshard/tables.hpp,
autoshard/workload_io.hpp), backed by the C++ host library through the C-ABI.

Names and semantics follow the reference: ``TableDesc``, ``GeneratorConfig``,
``generate_pool``, ``generate_workload``, ``Workload``/``TableStream``,
``ShardingTask``, ``ShardingPlan``, ``fingerprint``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._capi import GeneratorConfigC, TableSpecC, lib
from .errors import ConfigError, check


@dataclass
class TableDesc:
    """tables.hpp:24-38."""

    id: int = 0
    dim: int = 16
    hash_size: int = 1
    pooling_mean: float = 0.0
    access_ratio: float = 1.0
    bytes_per_param: int = 2

    def size_bytes(self) -> int:
        return int(self.dim) * int(self.hash_size) * int(self.bytes_per_param)

    def size_gb(self) -> float:
        return self.size_bytes() / (1024.0 ** 3)


def specs_to_c(tables: Sequence[TableDesc]):
    arr = (TableSpecC * max(1, len(tables)))()
    for i, t in enumerate(tables):
        arr[i] = TableSpecC(int(t.id), int(t.dim), int(t.hash_size), float(t.pooling_mean),
                            float(t.access_ratio), int(t.bytes_per_param), 0)
    return arr


def specs_from_c(arr, n) -> List[TableDesc]:
    return [TableDesc(arr[i].id, arr[i].dim, arr[i].hash_size, arr[i].pooling_mean,
                      arr[i].access_ratio, arr[i].bytes_per_param) for i in range(n)]


@dataclass
class GeneratorConfig:
    """tables.hpp:149-174."""

    hash_size_min: float = 1e3
    hash_size_max: float = 1e7
    pooling_mean_target: float = 15.0
    pooling_shape: float = 2.0
    pooling_cap: float = 193.0
    dim_choices: Sequence[int] = (16, 32)
    access_ratio_min: float = 1e-3
    access_ratio_max: float = 1.0
    bytes_per_param: int = 2

    def _c(self):
        dims = (C.c_int32 * max(1, len(self.dim_choices)))(*self.dim_choices)
        c = GeneratorConfigC(self.hash_size_min, self.hash_size_max, self.pooling_mean_target,
                             self.pooling_shape, self.pooling_cap, dims, len(self.dim_choices),
                             self.access_ratio_min, self.access_ratio_max, self.bytes_per_param)
        return c, dims


def generate_pool(seed: int, n_tables: int, cfg: Optional[GeneratorConfig] = None) -> List[TableDesc]:
    """generate_pool, tables.hpp:178-200 (bit-exact)."""
    if n_tables < 1:
        raise ConfigError("generate_pool: n_tables must be >= 1")
    c, keep = (cfg or GeneratorConfig())._c()
    out = (TableSpecC * n_tables)()
    check(lib().as_generate_pool(seed, n_tables, C.byref(c), out))
    del keep
    return specs_from_c(out, n_tables)


@dataclass
class TableStream:
    """tables.hpp:43-47 (numpy views into the library-owned buffers)."""

    table_id: int
    indices: np.ndarray
    offsets: np.ndarray


class Workload:
    """tables.hpp:49-60. Owns an ``as_workload`` handle; per_table arrays are
    zero-copy int64 views valid for the lifetime of this object."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        L = lib()
        self.batch_size = int(L.as_workload_batch_size(self._h))
        n = L.as_workload_num_tables(self._h)
        self.per_table: List[TableStream] = []
        for i in range(n):
            tid = C.c_int32()
            po, pi = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
            ni = C.c_int64()
            check(L.as_workload_stream(self._h, i, C.byref(tid), C.byref(po), C.byref(pi), C.byref(ni)))
            off = np.ctypeslib.as_array(po, shape=(self.batch_size + 1,))
            idx = (np.ctypeslib.as_array(pi, shape=(ni.value,)) if ni.value
                   else np.zeros(0, dtype=np.int64))
            self.per_table.append(TableStream(tid.value, idx, off))
        self._ids = [s.table_id for s in self.per_table]

    @property
    def handle(self):
        return self._h

    def find(self, table_id: int) -> Optional[TableStream]:
        import bisect

        k = bisect.bisect_left(self._ids, table_id)
        if k < len(self._ids) and self._ids[k] == table_id:
            return self.per_table[k]
        return None

    def pin(self) -> "Workload":
        """Page-lock the stream buffers for full-rate host->device loads."""
        check(lib().as_workload_pin(self._h))
        return self

    def save(self, path: str, tables: Sequence[TableDesc]) -> None:
        check(lib().as_workload_save(self._h, specs_to_c(tables), path.encode()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().as_workload_destroy(h)
            except Exception:
                pass
            self._h = None

    @staticmethod
    def from_arrays(batch_size: int, streams) -> "Workload":
        """streams: iterable of (table_id, offsets, indices), ascending ids."""
        streams = [(int(t), np.ascontiguousarray(o, dtype=np.int64), np.ascontiguousarray(i, dtype=np.int64))
                   for t, o, i in streams]
        n = len(streams)
        ids = (C.c_int32 * max(1, n))(*[s[0] for s in streams])
        po = (C.c_void_p * max(1, n))(*[s[1].ctypes.data for s in streams])
        pi = (C.c_void_p * max(1, n))(*[s[2].ctypes.data for s in streams])
        ni = (C.c_int64 * max(1, n))(*[len(s[2]) for s in streams])
        h = C.c_void_p()
        check(lib().as_workload_from_arrays(batch_size, n, ids, po, pi, ni, C.byref(h)))
        return Workload(h)


def generate_workload(seed: int, tables: Sequence[TableDesc], batch_size: int,
                      zipf_exponent: float = 1.05, n_threads: int = 0) -> Workload:
    """generate_workload, tables.hpp:237-288 (bit-exact; parallel over tables)."""
    h = C.c_void_p()
    check(lib().as_generate_workload(seed, specs_to_c(tables), len(tables), batch_size, zipf_exponent,
                                     n_threads, C.byref(h)))
    return Workload(h)


def load_workload(path: str):
    """load_workload_file, workload_io.hpp:247-258 -> (Workload, tables)."""
    n = C.c_int32()
    h = C.c_void_p()
    check(lib().as_workload_load(path.encode(), C.byref(h), None, 0, C.byref(n)))
    lib().as_workload_destroy(h)
    arr = (TableSpecC * max(1, n.value))()
    h = C.c_void_p()
    check(lib().as_workload_load(path.encode(), C.byref(h), arr, n.value, C.byref(n)))
    return Workload(h), specs_from_c(arr, n.value)


def save_pool(path: str, tables: Sequence[TableDesc]) -> None:
    check(lib().as_pool_save(specs_to_c(tables), len(tables), path.encode()))


def load_pool(path: str) -> List[TableDesc]:
    n = C.c_int32()
    check(lib().as_pool_load(path.encode(), None, 0, C.byref(n)))
    arr = (TableSpecC * max(1, n.value))()
    check(lib().as_pool_load(path.encode(), arr, n.value, C.byref(n)))
    return specs_from_c(arr, n.value)


def fingerprint(obj) -> int:
    """fingerprint(pool) / fingerprint(ShardingTask), tables.hpp:435-441."""
    if isinstance(obj, ShardingTask):
        b = np.asarray(obj.mem_budget, dtype=np.int64)
        return int(lib().as_fingerprint_task(specs_to_c(obj.tables), len(obj.tables), obj.num_shards,
                                             b.ctypes.data_as(C.POINTER(C.c_int64))))
    tables = list(obj)
    return int(lib().as_fingerprint_pool(specs_to_c(tables), len(tables)))


@dataclass
class ShardingTask:
    """tables.hpp:63-90."""

    tables: List[TableDesc] = field(default_factory=list)
    num_shards: int = 1
    mem_budget: List[int] = field(default_factory=list)

    @staticmethod
    def default_num_shards(n_tables: int) -> int:
        return (n_tables + 9) // 10

    def total_bytes(self) -> int:
        return sum(t.size_bytes() for t in self.tables)

    def total_budget(self) -> int:
        return int(sum(self.mem_budget))

    def validate(self) -> None:
        if self.num_shards < 1:
            raise ConfigError("task: num_shards must be >= 1")
        if len(self.mem_budget) != self.num_shards:
            raise ConfigError("task: mem_budget size must equal num_shards")
        if any(b <= 0 for b in self.mem_budget):
            raise ConfigError("task: all memory budgets must be > 0")


@dataclass
class ShardingPlan:
    """tables.hpp:93-143 (assignment is positional against task.tables)."""

    assignment: List[int] = field(default_factory=list)

    def _a(self):
        return (C.c_int32 * max(1, len(self.assignment)))(*self.assignment)

    def validate(self, task: ShardingTask) -> None:
        if len(self.assignment) != len(task.tables):
            raise ConfigError(f"plan: assignment length {len(self.assignment)} does not match task table "
                              f"count {len(task.tables)}")
        check(lib().as_plan_validate(len(self.assignment), task.num_shards, self._a()))

    def shard_members(self, task: ShardingTask) -> List[List[int]]:
        self.validate(task)
        m = [[] for _ in range(task.num_shards)]
        for i, k in enumerate(self.assignment):
            m[k].append(task.tables[i].id)
        return m

    def shard_member_indices(self, task: ShardingTask) -> List[List[int]]:
        self.validate(task)
        m = [[] for _ in range(task.num_shards)]
        for i, k in enumerate(self.assignment):
            m[k].append(i)
        return m

    def mem_used(self, task: ShardingTask) -> List[int]:
        self.validate(task)
        used = (C.c_int64 * task.num_shards)()
        check(lib().as_plan_mem_used(specs_to_c(task.tables), len(task.tables), task.num_shards, self._a(), used))
        return list(used)

    def feasible(self, task: ShardingTask) -> bool:
        return all(u <= b for u, b in zip(self.mem_used(task), task.mem_budget))
