// PLAN-PRODUCING INFRASTRUCTURE (not the product). Drives the UNMODIFIED
// reference AutoShard-RL trainer (autoshard/rl_train.hpp:400-547, compiled in
// place from /root/reference/proj/include by oracle/Makefile) to produce the
// "AutoShard-RL" plans that the GPU cost hook then measures (SURVEY.md §2.3:
// rl/rl_train are kept as the oracle build, not re-implemented).
//
// Unseen-table transfer: training tasks are random subsets of
// pool tables [n_target, n_pool); the target task is tables [0, n_target)
// (e.g. BASELINE cfg 3 = generate_pool(0, 100, dims {32,64,128,256})).
//
// usage: rl_plans <n_pool> <n_target> <K> <batch> <max_updates> <max_seconds> <out_prefix> [dims...]
// writes <out_prefix>.assignment (one line, n_target shard ids) and
// <out_prefix>.ckpt (the reference checkpoint, ASHCKPT1).
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "autoshard/planners.hpp"
#include "autoshard/rl_train.hpp"
#include "autoshard/tables.hpp"

using namespace autoshard;

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s n_pool n_target K batch max_updates max_seconds out_prefix [dims...]\n", argv[0]);
    return 2;
  }
  const int n_pool = std::atoi(argv[1]), n_target = std::atoi(argv[2]), K = std::atoi(argv[3]);
  const long long batch = std::atoll(argv[4]);
  const int max_updates = std::atoi(argv[5]);
  const double max_seconds = std::atof(argv[6]);
  const std::string out = argv[7];
  GeneratorConfig gcfg;
  if (argc > 8) {
    gcfg.dim_choices.clear();
    for (int i = 8; i < argc; ++i) gcfg.dim_choices.push_back(std::atoi(argv[i]));
  }
  const auto pool = generate_pool(0, n_pool, gcfg);
  const Workload wl = generate_workload(0, pool, batch);
  const std::vector<TableDesc> target(pool.begin(), pool.begin() + n_target);
  const std::vector<TableDesc> train_pool(pool.begin() + n_target, pool.end());
  const NormStats norm = compute_norm_stats(train_pool, wl);
  const FeatureMask mask{};
  const SimParams sim{};

  auto task_of = [&](std::vector<TableDesc> tabs) {
    ShardingTask t;
    t.tables = std::move(tabs);
    t.num_shards = K;
    const long long per = (long long)(1.6 * (double)t.total_bytes() / K);
    t.mem_budget.assign(K, per);
    return t;
  };
  // training tasks: random subsets (n_target tables) of the unseen-for-target tables
  std::vector<rl::TaskContext> train_tasks, test_tasks;
  Rng rng(derive_seed(0, "rl-plans-tasks"));
  const int n_train = 8;
  for (int i = 0; i < n_train; ++i) {
    std::vector<TableDesc> tabs(train_pool);
    rng.shuffle(tabs.begin(), tabs.end());
    tabs.resize(std::min<size_t>(tabs.size(), (size_t)n_target));
    train_tasks.push_back(rl::make_task_context(i, task_of(tabs), wl, norm, mask, sim));
  }
  test_tasks.push_back(rl::make_task_context(1000, task_of(target), wl, norm, mask, sim));

  rl::TrainConfig cfg;
  cfg.max_updates = max_updates;
  cfg.max_seconds = max_seconds;
  cfg.eval_every = 10;
  const auto t0 = std::chrono::steady_clock::now();
  const auto res = rl::train(train_tasks, test_tasks, norm, mask, sim, batch, fingerprint(pool), cfg, &std::cerr);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  rl::save_checkpoint_file(out + ".ckpt", res.checkpoint);

  const ShardingTask ttask = task_of(target);
  const ShardingPlan plan = rl::shard_with_checkpoint(res.checkpoint, ttask, wl);
  std::ofstream os(out + ".assignment");
  for (size_t i = 0; i < plan.assignment.size(); ++i) os << (i ? " " : "") << plan.assignment[i];
  os << "\n";
  const auto sim_costs = measure_plan(plan, ttask, wl, sim, BenchConfig{.exact = true});
  const auto greedy = greedy_shard(ttask, HeuristicKind::kLookupGreedy);
  const auto g_costs = measure_plan(greedy, ttask, wl, sim, BenchConfig{.exact = true});
  std::printf("updates %d  seconds %.1f  best_train_balance %.4f  test_balance %.4f  sim_balance_rl %.4f  "
              "sim_balance_lookup_greedy %.4f\n",
              res.updates, secs, res.best_train_balance, res.final_test_balance, degree_of_balance(sim_costs),
              degree_of_balance(g_costs));
  return 0;
}
