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
//
// RL_SEED=s: TrainConfig::seed (model init and actor streams). RL_SEEDS=a,b,..:
// one trainer per seed in parallel threads (outputs <out_prefix>_s<seed>.*).
//
// TRAIN_RANGE=a:b: train on subsets of pool tables [a, b) instead of
// [n_target, n_pool) — BASELINE cfg 5 (856 tables, 50% unseen): n_pool =
// n_target = 856, TRAIN_RANGE=0:428.
//
// GPU_REWARD=1 (rl_plans_gpu build): every per-shard cost
// of the environment is measured on the B200 (see the hook below); checkpoint
// selection then runs on a validation task drawn from the training pool.
// VALIDATION=1: the same validation task with the SIM reward (the matched
// control), instead of selecting on the target task.
//
// MARGINALS=<file>: train against B200-MEASURED costs
// instead of the analytic SIM (tools/measure_marginals.py writes the file:
// c0, rho and per-table marginals w_t = measured one-table time - c0). Every
// task context gets marginal_w[t] = w_t (the env's terminal reward and the
// cost-model bootstrap, rl.hpp:161-167 / rl_train.hpp:387-389), and the SIM
// the trainer still evaluates directly (checkpoint selection through
// measure_plan, rl_train.hpp:231) is CALIBRATED to the same measurements: c0
// and rho from the file, a / b / cache_floor of SIM-1 (simcost.hpp:60-78)
// least-squares fitted to the w_t on this workload.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <sstream>
#include <unordered_set>
#include <fstream>
#include <iostream>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "autoshard/common.hpp"
#include "autoshard/costmodel.hpp"
#include "autoshard/netcore.hpp"
#include "autoshard/planners.hpp"
#include "autoshard/simcost.hpp"
#include "autoshard/tables.hpp"

#ifdef ASB_GPU_REWARD
// GPU_REWARD=1 (the rl_plans_gpu build): the per-shard costs
// the RL environment asks for are MEASURED on the B200 through the product's
// hook (autoshard::gpu::ShardCostService: subset contexts over one resident
// pool, W/B/R protocol, cached by membership). The three call sites — the
// terminal reward (rl.hpp:166), checkpoint selection (rl_train.hpp:231) and
// the cost-model bootstrap (rl_train.hpp:389) — are redirected at compile
// time; the reference headers are unmodified (INTEGRATION.md shows the
// one-line change a maintainer would make at each site instead). Task
// contexts carry table handles in marginal_w (task index * 2^16 + position),
// so the hooks know which tables form each shard.
#define AUTOSHARD_B200_REFERENCE_ERRORS 1
#include <mutex>

#include "autoshard_b200.hpp"
namespace autoshard {
struct GpuHook {
  gpu::ShardCostService* svc = nullptr;
  std::mutex mu;  // one measurement at a time (parallel trainers share the GPU)
  std::vector<std::vector<int>> task_ids;  // per encoded task: table ids by position
};
inline GpuHook& gpu_hook() {
  static GpuHook h;
  return h;
}
// off while a thread applies a checkpoint (shard_with_checkpoint builds a
// fresh SIM context and ignores the episode's reward)
inline thread_local bool gpu_hook_off = false;
inline int32_t gpu_decode(double w) {
  const long long v = std::llround(w);
  const GpuHook& h = gpu_hook();
  return h.svc->position(h.task_ids.at(static_cast<size_t>(v >> 16)).at(static_cast<size_t>(v & 0xffff)));
}
inline double gpu_shard_cost_from_marginals(const std::vector<double>& w, const SimParams& p) {
  if (!gpu_hook().svc || gpu_hook_off) return shard_cost_from_marginals(w, p);
  std::vector<int32_t> pos;
  for (double x : w) pos.push_back(gpu_decode(x));
  std::lock_guard<std::mutex> lk(gpu_hook().mu);
  return gpu_hook().svc->cost(std::move(pos));
}
inline std::vector<double> gpu_costs_from_marginals(const std::vector<std::vector<double>>& g, const SimParams& p,
                                                    const BenchConfig& b) {
  if (!gpu_hook().svc || gpu_hook_off) return measure_costs_from_marginals(g, p, b);
  std::vector<double> c;
  for (const auto& w : g) c.push_back(gpu_shard_cost_from_marginals(w, p));
  return c;
}
inline std::vector<double> gpu_measure_plan(const ShardingPlan& plan, const ShardingTask& task, const Workload& wl,
                                            const SimParams& p, const BenchConfig& b) {
  if (!gpu_hook().svc || gpu_hook_off) return measure_plan(plan, task, wl, p, b);
  std::lock_guard<std::mutex> lk(gpu_hook().mu);
  return gpu_hook().svc->plan_costs(plan, task);
}
}  // namespace autoshard
#define measure_costs_from_marginals gpu_costs_from_marginals
#define shard_cost_from_marginals gpu_shard_cost_from_marginals
#define measure_plan gpu_measure_plan
#endif
#include "autoshard/rl.hpp"
#include "autoshard/rl_train.hpp"
#ifdef ASB_GPU_REWARD
#undef measure_costs_from_marginals
#undef shard_cost_from_marginals
#undef measure_plan
#endif

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
  int tr_lo = n_target, tr_hi = n_pool;
  if (const char* r = std::getenv("TRAIN_RANGE")) std::sscanf(r, "%d:%d", &tr_lo, &tr_hi);
  if (tr_lo < 0 || tr_hi > n_pool || tr_lo >= tr_hi) {
    std::fprintf(stderr, "bad TRAIN_RANGE %d:%d\n", tr_lo, tr_hi);
    return 2;
  }
  const std::vector<TableDesc> train_pool(pool.begin() + tr_lo, pool.begin() + tr_hi);
  const NormStats norm = compute_norm_stats(train_pool, wl);
  const FeatureMask mask{};
  SimParams sim{};
  std::map<int, double> measured;  // table id -> GPU marginal (ms)
  if (const char* mf = std::getenv("MARGINALS")) {
    std::ifstream is(mf);
    if (!is) {
      std::fprintf(stderr, "cannot read MARGINALS=%s\n", mf);
      return 2;
    }
    std::string line;
    while (std::getline(is, line)) {
      if (line.empty() || line[0] == '#') continue;
      std::istringstream ls(line);
      std::string k;
      double v;
      ls >> k >> v;
      if (k == "c0") sim.c0 = v;
      else if (k == "rho") sim.rho = v;
      else measured[std::atoi(k.c_str())] = v;
    }
    // fit SIM-1's a, b, cache_floor to the measured marginals of the pool
    double best = 1e300, ba = sim.a, bb = sim.b, bf = sim.cache_floor;
    std::vector<double> x1, x2, y;
    std::vector<double> L, u, dim, lh;
    for (const auto& t : pool) {
      auto it = measured.find(t.id);
      if (it == measured.end()) continue;
      const TableStream* s = wl.find(t.id);
      std::unordered_set<std::int64_t> d(s->indices.begin(), s->indices.end());
      L.push_back((double)s->indices.size());
      u.push_back(s->indices.empty() ? 0.0 : std::min(1.0, (double)d.size() / (double)s->indices.size()));
      dim.push_back(t.dim);
      lh.push_back(std::log10(1.0 + (double)t.hash_size));
      y.push_back(it->second);
    }
    for (int g = 1; g <= 100; ++g) {
      const double f = g / 100.0;
      double s11 = 0, s12 = 0, s22 = 0, r1 = 0, r2 = 0;
      std::vector<double> a1(y.size()), a2(y.size());
      for (size_t i = 0; i < y.size(); ++i) {
        a1[i] = L[i] * dim[i] * (f + (1 - f) * u[i]);
        a2[i] = dim[i] * lh[i];
        // relative least squares: weight 1/y^2
        const double wgt = 1.0 / std::max(1e-9, y[i] * y[i]);
        s11 += wgt * a1[i] * a1[i]; s12 += wgt * a1[i] * a2[i]; s22 += wgt * a2[i] * a2[i];
        r1 += wgt * a1[i] * y[i]; r2 += wgt * a2[i] * y[i];
      }
      const double det = s11 * s22 - s12 * s12;
      double a = det != 0 ? (r1 * s22 - r2 * s12) / det : 0, b = det != 0 ? (s11 * r2 - s12 * r1) / det : 0;
      if (a < 0) { a = 0; b = r2 / s22; }
      if (b < 0) { b = 0; a = r1 / s11; }
      double err = 0;
      for (size_t i = 0; i < y.size(); ++i) {
        const double e = (a * a1[i] + b * a2[i] - y[i]) / std::max(1e-9, y[i]);
        err += e * e;
      }
      if (err < best) { best = err; ba = a; bb = b; bf = f; }
    }
    sim.a = ba;
    sim.b = bb;
    sim.cache_floor = bf;
    std::fprintf(stderr, "MARGINALS %s: %zu tables, c0 %.5f rho %.4f; SIM-1 fit a %.4g b %.4g cache_floor %.2f rel.RMS %.4f\n",
                 mf, measured.size(), sim.c0, sim.rho, sim.a, sim.b, sim.cache_floor,
                 std::sqrt(best / std::max<size_t>(1, y.size())));
  }
  auto with_measured = [&](rl::TaskContext ctx) {
    if (!measured.empty())
      for (size_t i = 0; i < ctx.task.tables.size(); ++i) {
        auto it = measured.find(ctx.task.tables[i].id);
        if (it != measured.end()) ctx.marginal_w[i] = it->second;
      }
    return ctx;
  };

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
    train_tasks.push_back(with_measured(rl::make_task_context(i, task_of(tabs), wl, norm, mask, sim)));
  }
#ifdef ASB_GPU_REWARD
  std::unique_ptr<gpu::ShardCostService> svc;
  std::unique_ptr<Workload> gwl;
  if (const char* g = std::getenv("GPU_REWARD"); g && std::atoi(g) != 0) {
    // measured costs at GPU_BATCH (default 16384; the features stay on the
    // trainer's batch); selection on a VALIDATION task drawn from the training
    // pool, never on the target task the plan is evaluated on
    const long long gb = std::getenv("GPU_BATCH") ? std::atoll(std::getenv("GPU_BATCH")) : 16384;
    int w = 2, b = 5, r = 1;
    if (const char* e = std::getenv("GPU_WBR")) std::sscanf(e, "%d,%d,%d", &w, &b, &r);
    gwl = std::make_unique<Workload>(gb == batch ? wl : generate_workload(0, train_pool, gb));
    svc = std::make_unique<gpu::ShardCostService>(0, train_pool, *gwl, w, b, r, true);
    std::vector<TableDesc> vt(train_pool);
    Rng vr(derive_seed(0, "rl-plans-validation"));
    vr.shuffle(vt.begin(), vt.end());
    vt.resize(std::min<size_t>(vt.size(), (size_t)n_target));
    test_tasks.push_back(rl::make_task_context(1000, task_of(vt), wl, norm, mask, sim));
    auto& hook = gpu_hook();
    int k = 0;
    for (auto* v : {&train_tasks, &test_tasks})
      for (auto& c : *v) {
        std::vector<int> ids;
        for (size_t i = 0; i < c.task.tables.size(); ++i) {
          ids.push_back(c.task.tables[i].id);
          c.marginal_w[i] = (double)k * 65536.0 + (double)i;
        }
        hook.task_ids.push_back(std::move(ids));
        ++k;
      }
    hook.svc = svc.get();
    std::fprintf(stderr, "GPU_REWARD: %zu pool tables resident, measurement batch %lld, W/B/R %d/%d/%d\n",
                 train_pool.size(), gb, w, b, r);
  } else
#endif
  if (const char* v = std::getenv("VALIDATION"); v && std::atoi(v) != 0) {
    // checkpoint selection on a validation task from the training pool (the
    // same draw as the GPU_REWARD path), not on the target task
    std::vector<TableDesc> vt(train_pool);
    Rng vr(derive_seed(0, "rl-plans-validation"));
    vr.shuffle(vt.begin(), vt.end());
    vt.resize(std::min<size_t>(vt.size(), (size_t)n_target));
    test_tasks.push_back(with_measured(rl::make_task_context(1000, task_of(vt), wl, norm, mask, sim)));
  } else {
    test_tasks.push_back(with_measured(rl::make_task_context(1000, task_of(target), wl, norm, mask, sim)));
  }

  // RL_SEEDS=a,b,...: one trainer per seed, in parallel threads sharing the
  // task set (and, with GPU_REWARD, the measured-cost service and its cache);
  // outputs <out>_s<seed>.{ckpt,assignment,log}. Default: RL_SEED (or 0) -> <out>.*
  std::vector<std::uint64_t> seeds;
  bool multi = false;
  if (const char* ss = std::getenv("RL_SEEDS")) {
    multi = true;
    std::stringstream st(ss);
    std::string tok;
    while (std::getline(st, tok, ',')) seeds.push_back(std::strtoull(tok.c_str(), nullptr, 10));
  } else {
    seeds.push_back(std::getenv("RL_SEED") ? std::strtoull(std::getenv("RL_SEED"), nullptr, 10) : 0);  // TrainConfig::seed
  }
  const ShardingTask ttask = task_of(target);
  auto run_seed = [&](std::uint64_t seed) {
    rl::TrainConfig cfg;
    cfg.max_updates = max_updates;
    cfg.seed = seed;
    cfg.max_seconds = max_seconds;
    cfg.eval_every = 10;
    const std::string o = multi ? out + "_s" + std::to_string(seed) : out;
    std::ofstream logf;
    std::ostream* log = &std::cerr;
    if (multi) {
      logf.open(o + ".log");
      log = &logf;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const auto res = rl::train(train_tasks, test_tasks, norm, mask, sim, batch, fingerprint(pool), cfg, log);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rl::save_checkpoint_file(o + ".ckpt", res.checkpoint);
#ifdef ASB_GPU_REWARD
    gpu_hook_off = true;
#endif
    const ShardingPlan plan = rl::shard_with_checkpoint(res.checkpoint, ttask, wl);
    std::ofstream os(o + ".assignment");
    for (size_t i = 0; i < plan.assignment.size(); ++i) os << (i ? " " : "") << plan.assignment[i];
    os << "\n";
    std::ostringstream line;
    line << "seed " << seed << "  updates " << res.updates << "  seconds " << secs << "  best_train_balance "
         << res.best_train_balance << "  test_balance " << res.final_test_balance;
    return std::make_pair(plan, line.str());
  };
  std::vector<std::pair<ShardingPlan, std::string>> results(seeds.size());
  {
    std::vector<std::thread> th;
    for (size_t i = 0; i < seeds.size(); ++i) th.emplace_back([&, i] { results[i] = run_seed(seeds[i]); });
    for (auto& t : th) t.join();
  }
#ifdef ASB_GPU_REWARD
  if (svc) {
    std::fprintf(stderr, "GPU_REWARD: %zu shards measured, %zu cache hits\n", svc->measured(), svc->hits());
    gpu_hook().svc = nullptr;
  }
#endif
  const auto greedy = greedy_shard(ttask, HeuristicKind::kLookupGreedy);
  const auto g_costs = measure_plan(greedy, ttask, wl, sim, BenchConfig{.exact = true});
  for (auto& r : results) {
    const auto sim_costs = measure_plan(r.first, ttask, wl, sim, BenchConfig{.exact = true});
    std::printf("%s  sim_balance_rl %.4f  sim_balance_lookup_greedy %.4f\n", r.second.c_str(),
                degree_of_balance(sim_costs), degree_of_balance(g_costs));
  }
  return 0;
}
