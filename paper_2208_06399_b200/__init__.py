"""B200-native AutoShard embedding-bag hot path (arXiv 2208.06399).

Host mirror of the reference's interface for this path (autoshard/tables.hpp,
planners.hpp, simcost.hpp) over the C-ABI in include/autoshard_b200.h, whose
device side is hand-written sm_100a CUDA. Importing this package loads the
native library and raises if it has not been built.
"""
from ._capi import LIB_PATH, lib
from .device import BenchConfig, EmbeddingShard, measure_plan, probe_gather_bw
from .errors import (ConfigError, CudaError, Error, GuardError, IndexError_, InfeasibleError, LookupError_,
                     NcclError, OffsetError, ParseError, ShapeError, StateError)
from .planners import (HeuristicKind, degree_of_balance, greedy_shard, heuristic_cost, heuristic_name, load_plan,
                       random_shard, save_plan, speedup_over)
from .tables import (GeneratorConfig, ShardingPlan, ShardingTask, TableDesc, TableStream, Workload, fingerprint,
                     generate_pool, generate_workload, load_pool, load_workload, save_pool)

lib()  # fail loudly at import if the native library is missing

__all__ = [
    "LIB_PATH", "BenchConfig", "EmbeddingShard", "measure_plan", "ConfigError", "CudaError", "Error", "GuardError",
    "IndexError_", "InfeasibleError", "LookupError_", "NcclError", "OffsetError", "ParseError", "ShapeError",
    "StateError", "HeuristicKind", "degree_of_balance", "greedy_shard", "heuristic_cost", "heuristic_name",
    "load_plan", "random_shard", "save_plan", "speedup_over", "GeneratorConfig", "ShardingPlan", "ShardingTask",
    "TableDesc", "TableStream", "Workload", "fingerprint", "generate_pool", "generate_workload", "load_pool",
    "load_workload", "save_pool",
]
