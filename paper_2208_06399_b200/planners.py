"""Planners (autoshard/planners.hpp:20-144) and the plan file,
backed by the C++ host library."""
from __future__ import annotations

import ctypes as C
import enum
from typing import Optional, Sequence, Tuple

import numpy as np

from ._capi import lib
from .errors import ConfigError, check
from .tables import ShardingPlan, ShardingTask, TableDesc, specs_to_c


class HeuristicKind(enum.IntEnum):
    """planners.hpp:20."""

    kSizeGreedy = 0
    kDimGreedy = 1
    kLookupGreedy = 2
    kRandom = 3


def heuristic_name(k: HeuristicKind) -> str:
    return {0: "size-greedy", 1: "dim-greedy", 2: "lookup-greedy", 3: "rand"}[int(k)]


def heuristic_cost(t: TableDesc, kind: HeuristicKind) -> float:
    out = C.c_double()
    check(lib().as_heuristic_cost(specs_to_c([t]), int(kind), C.byref(out)))
    return out.value


def _budgets(task: ShardingTask):
    task.validate()
    b = np.asarray(task.mem_budget, dtype=np.int64)
    return b, b.ctypes.data_as(C.POINTER(C.c_int64))


def greedy_shard(task: ShardingTask, kind: HeuristicKind) -> ShardingPlan:
    """planners.hpp:73-107."""
    if int(kind) == int(HeuristicKind.kRandom):
        raise ConfigError("greedy_shard: use random_shard for kind=rand")
    b, pb = _budgets(task)
    out = (C.c_int32 * max(1, len(task.tables)))()
    check(lib().as_greedy_shard(specs_to_c(task.tables), len(task.tables), task.num_shards, pb, int(kind), out))
    return ShardingPlan(list(out)[: len(task.tables)])


def random_shard(task: ShardingTask, seed: int) -> ShardingPlan:
    """planners.hpp:111-136."""
    b, pb = _budgets(task)
    out = (C.c_int32 * max(1, len(task.tables)))()
    check(lib().as_random_shard(specs_to_c(task.tables), len(task.tables), task.num_shards, pb, seed, out))
    return ShardingPlan(list(out)[: len(task.tables)])


def degree_of_balance(costs: Sequence[float]) -> float:
    """planners.hpp:139-144."""
    c = np.asarray(costs, dtype=np.float64)
    if c.size == 0:
        raise ConfigError("degree_of_balance: empty cost vector")
    out = C.c_double()
    check(lib().as_degree_of_balance(c.ctypes.data_as(C.POINTER(C.c_double)), len(c), C.byref(out)))
    return out.value


def speedup_over(costs_baseline: Sequence[float], costs: Sequence[float]) -> float:
    """Speedup of a plan over a baseline plan: max(C_base) / max(C)."""
    return max(costs_baseline) / max(costs)


def save_plan(path: str, task: ShardingTask, plan: ShardingPlan,
              costs: Optional[Sequence[float]] = None) -> None:
    b, pb = _budgets(task)
    a = (C.c_int32 * max(1, len(plan.assignment)))(*plan.assignment)
    pc = None
    if costs is not None:
        cc = np.asarray(costs, dtype=np.float64)
        pc = cc.ctypes.data_as(C.POINTER(C.c_double))
    check(lib().as_plan_save(path.encode(), specs_to_c(task.tables), len(task.tables), task.num_shards, pb, a, pc))


def load_plan(path: str, task: ShardingTask) -> Tuple[ShardingPlan, Optional[list]]:
    b, pb = _budgets(task)
    a = (C.c_int32 * max(1, len(task.tables)))()
    costs = (C.c_double * task.num_shards)()
    has = C.c_int32()
    check(lib().as_plan_load(path.encode(), specs_to_c(task.tables), len(task.tables), task.num_shards, pb, a,
                             costs, C.byref(has)))
    return ShardingPlan(list(a)[: len(task.tables)]), (list(costs) if has.value else None)
