// Drop-in demonstration: code written against the reference's C++ types
// (autoshard/tables.hpp, simcost.hpp) swaps the simulated cost hook for the
// measured B200 one by changing one call. Built by tests/cpp/Makefile against
// the reference headers (where mounted) and libautoshard_b200.so.
//
//   usage: dropin_example            -> prints per-shard costs (SIM and GPU)
#define AUTOSHARD_B200_REFERENCE_ERRORS 1
#include <cstdio>
#include <memory>

#include "autoshard/planners.hpp"
#include "autoshard/simcost.hpp"
#include "autoshard/tables.hpp"
#include "autoshard_b200.hpp"

int main() {
  using namespace autoshard;
  GeneratorConfig cfg;
  cfg.dim_choices = {64};
  cfg.pooling_mean_target = 20.0;
  const auto pool = generate_pool(0, 10, cfg);       // BASELINE cfg 1
  const Workload wl = generate_workload(0, pool, 512);
  ShardingTask task;
  task.tables = pool;
  task.num_shards = 2;
  task.mem_budget.assign(2, task.total_bytes());
  const ShardingPlan plan = greedy_shard(task, HeuristicKind::kLookupGreedy);
  BenchConfig bench;  // W=5, B=10, R=2

  const auto sim = measure_plan(plan, task, wl, SimParams{}, bench);  // reference: simulator
  std::printf("sim  ms: %.4f %.4f  balance %.3f\n", sim[0], sim[1], degree_of_balance(sim));
  try {
    const auto gpu = gpu::measure_plan(plan, task, wl, bench);  // drop-in: measured on the B200
    std::printf("gpu  ms: %.4f %.4f  balance %.3f\n", gpu[0], gpu[1], degree_of_balance(gpu));
  } catch (const gpu::Error& e) {
    std::printf("gpu  unavailable (%s)\n", e.what());
    return e.code == AS_CUDA ? 0 : 1;
  }
  return 0;
}
