// autoshard_b200.hpp — C++ face of the B200 hot path, shaped like the
// reference's own interface so it drops into code written against
// /root/reference/proj/include/autoshard (header-only, over the C-ABI in
// autoshard_b200.h; link with -lautoshard_b200).
//
//   autoshard::measure_plan(plan, task, wl, sim, bench)        simcost.hpp:194
//     -> autoshard::gpu::measure_plan(plan, task, wl, bench)   measured B200 ms per shard
//
// The templates are duck-typed on the reference types (TableDesc, ShardingTask,
// ShardingPlan, Workload/TableStream, BenchConfig: tables.hpp:24-143,
// simcost.hpp:163-171), so this header does not include the reference. Define
// AUTOSHARD_B200_REFERENCE_ERRORS after including "autoshard/common.hpp" to
// get the reference's exception classes (common.hpp:15-50) instead of
// autoshard::gpu::Error.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <unordered_map>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

#include "autoshard_b200.h"

namespace autoshard {
namespace gpu {

struct Error : std::runtime_error {
  as_status code;
  Error(as_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(as_status s, const std::string& msg) {
#ifdef AUTOSHARD_B200_REFERENCE_ERRORS
  switch (s) {
    case AS_CONFIG: throw ::autoshard::ConfigError(msg);
    case AS_PARSE: throw ::autoshard::ParseError(msg);
    case AS_OFFSET: throw ::autoshard::OffsetError(msg);
    case AS_INDEX: throw ::autoshard::IndexError(msg);
    case AS_INFEASIBLE: throw ::autoshard::InfeasibleError(msg);
    case AS_SHAPE: throw ::autoshard::ShapeError(msg);
    case AS_LOOKUP: throw ::autoshard::LookupError(msg);
    case AS_GUARD: throw ::autoshard::GuardError(msg);
    case AS_STATE: throw ::autoshard::StateError(msg);
    default: break;
  }
#endif
  throw Error(s, msg);
}

[[noreturn]] inline void throw_status(as_status s) { raise(s, as_last_error()); }

inline void check(as_status s) {
  if (s != AS_OK) throw_status(s);
}

template <class TableDescT>
as_table_spec to_spec(const TableDescT& t) {
  as_table_spec s{};
  s.id = t.id;
  s.dim = t.dim;
  s.hash_size = t.hash_size;
  s.pooling_mean = t.pooling_mean;
  s.access_ratio = t.access_ratio;
  s.bytes_per_param = t.bytes_per_param;
  return s;
}

template <class Tables>
std::vector<as_table_spec> to_specs(const Tables& tables) {
  std::vector<as_table_spec> v;
  v.reserve(tables.size());
  for (const auto& t : tables) v.push_back(to_spec(t));
  return v;
}

// Owning handle of an as_workload built from a reference Workload's streams
// (only the tables listed are copied).
class WorkloadView {
 public:
  template <class WorkloadT, class Tables>
  WorkloadView(const WorkloadT& wl, const Tables& tables) {
    std::vector<std::pair<int, const void*>> want;
    for (const auto& t : tables) {
      const auto* s = wl.find(t.id);
      if (!s) throw_missing(t.id);
      want.push_back({t.id, s});
    }
    std::sort(want.begin(), want.end(), [](auto& a, auto& b) { return a.first < b.first; });
    want.erase(std::unique(want.begin(), want.end(), [](auto& a, auto& b) { return a.first == b.first; }),
               want.end());
    std::vector<int32_t> ids;
    std::vector<const int64_t*> off, idx;
    std::vector<int64_t> n;
    using Stream = std::remove_pointer_t<decltype(wl.find(0))>;
    for (auto& w : want) {
      const auto* s = static_cast<const Stream*>(w.second);
      ids.push_back(w.first);
      off.push_back(s->offsets.data());
      idx.push_back(s->indices.data());
      n.push_back(static_cast<int64_t>(s->indices.size()));
    }
    as_workload* h = nullptr;
    check(as_workload_from_arrays(wl.batch_size, static_cast<int32_t>(ids.size()), ids.data(), off.data(),
                                  idx.data(), n.data(), &h));
    h_.reset(h);
  }
  const as_workload* get() const { return h_.get(); }
  as_workload* get() { return h_.get(); }

 private:
  [[noreturn]] static void throw_missing(int id) {
    raise(AS_LOOKUP, "measure_plan: table " + std::to_string(id) + " absent from workload");
  }
  struct Del {
    void operator()(as_workload* w) const { as_workload_destroy(w); }
  };
  std::unique_ptr<as_workload, Del> h_;
};

struct GpuBenchConfig {
  std::vector<int32_t> devices{0};  // shard k runs on devices[k % size]
  bool flush_l2 = true;
  float lr = 0.01f, eps = 1e-8f;
  uint64_t weight_seed = 0;
};

// measure_plan (simcost.hpp:194-204) with the simulator replaced by the
// micro-benchmark of the real kernels: per shard, W warm-up and B measured
// fwd+bwd steps (L2 flushed before each), trimmed mean of B-2R, in ms.
template <class Plan, class Task, class WorkloadT, class Bench>
std::vector<double> measure_plan(const Plan& plan, const Task& task, const WorkloadT& wl, const Bench& bench,
                                 const GpuBenchConfig& gpu = {}) {
  const auto specs = to_specs(task.tables);
  if (plan.assignment.size() != specs.size())
    raise(AS_CONFIG, "plan: assignment length " + std::to_string(plan.assignment.size()) +
                         " does not match task table count " + std::to_string(specs.size()));
  WorkloadView view(wl, task.tables);
  as_bench_config bc{};
  bc.warmup = bench.warmup;
  bc.measure = bench.measure;
  bc.trim = bench.trim;
  bc.flush_l2 = gpu.flush_l2 ? 1 : 0;
  bc.seed = gpu.weight_seed;
  bc.lr = gpu.lr;
  bc.eps = gpu.eps;
  std::vector<int32_t> a(plan.assignment.begin(), plan.assignment.end());
  std::vector<double> costs(static_cast<size_t>(task.num_shards), 0.0);
  check(as_measure_plan(specs.data(), static_cast<int32_t>(specs.size()), task.num_shards, a.data(), view.get(),
                        gpu.devices.data(), static_cast<int32_t>(gpu.devices.size()), &bc, costs.data()));
  return costs;
}

// One shard resident on one device (RAII over as_ctx).
class Shard {
 public:
  // flags: 0 (fp32 tables) or AS_WEIGHTS_FP16 (bytes_per_param 2 storage)
  template <class Tables>
  Shard(int device, const Tables& tables, int64_t batch, uint64_t weight_seed = 0, int32_t flags = 0) {
    const auto specs = to_specs(tables);
    as_ctx* c = nullptr;
    check(as_create_ex(device, specs.data(), static_cast<int32_t>(specs.size()), batch, weight_seed, flags, &c));
    ctx_.reset(c);
  }
  template <class WorkloadT, class Tables>
  void load(const WorkloadT& wl, const Tables& tables, void* stream = nullptr) {
    WorkloadView v(wl, tables);
    check(as_load_workload(ctx_.get(), v.get(), stream));
  }
  void forward(float* out = nullptr, void* stream = nullptr) { check(as_forward(ctx_.get(), out, stream)); }
  // fused forward exchange: pooled row b -> peer_bases[b / rows_per_peer] (as_set_peer_outputs)
  void set_peer_outputs(const std::vector<float*>& peer_bases, int64_t rows_per_peer) {
    check(as_set_peer_outputs(ctx_.get(), static_cast<int>(peer_bases.size()), peer_bases.data(), rows_per_peer));
  }
  void backward(const float* grad, float lr, float eps, void* stream = nullptr) {
    check(as_backward_rowwise_adagrad(ctx_.get(), grad, lr, eps, stream));
  }
  double step(float lr, float eps, void* stream = nullptr) {
    double loss = 0.0;
    check(as_step(ctx_.get(), lr, eps, &loss, stream));
    return loss;
  }
  double measure(int warmup, int measure, int trim, bool flush = true, float lr = 0.01f, float eps = 1e-8f) {
    double ms = 0.0;
    check(as_measure(ctx_.get(), warmup, measure, trim, flush ? 1 : 0, lr, eps, &ms));
    return ms;
  }
  as_ctx_info info() const {
    as_ctx_info i{};
    check(as_ctx_info_get(ctx_.get(), &i));
    return i;
  }
  as_ctx* get() { return ctx_.get(); }
  const as_ctx* get() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(as_ctx* c) const { as_destroy(c); }
  };
  std::unique_ptr<as_ctx, Del> ctx_;
};

// Measured cost of candidate shards over one resident pool of tables. The
// pool's weights live in one parent context; a candidate shard is a subset
// context on that storage (as_create_subset: no copy, no init), loaded with
// its tables' streams and timed with the W/B/R protocol (simcost.hpp:140-154).
// Costs are cached by membership. This is the measured replacement of the
// per-shard costs the reference's RL environment asks for: the terminal
// reward (rl.hpp:161-167), checkpoint selection (rl_train.hpp:231) and the
// cost-model bootstrap (rl_train.hpp:383-392). Not thread-safe: one caller
// at a time (parallel trainers serialise on a mutex, oracle/rl_plans.cpp).
class ShardCostService {
 public:
  template <class Tables, class WorkloadT>
  ShardCostService(int device, const Tables& pool, const WorkloadT& wl, int warmup = 2, int measure = 5, int trim = 1,
                   bool flush_l2 = true, uint64_t weight_seed = 0)
      : parent_(device, pool, wl.batch_size, weight_seed),
        view_(wl, pool),
        warmup_(warmup),
        measure_(measure),
        trim_(trim),
        flush_(flush_l2) {
    int i = 0;
    for (const auto& t : pool) pos_of_[t.id] = i++;
    check(as_workload_pin(view_.get()));
  }
  // position of a table id in the pool (LookupError-like AS_LOOKUP if absent)
  int position(int table_id) const {
    auto it = pos_of_.find(table_id);
    if (it == pos_of_.end()) raise(AS_LOOKUP, "shard cost: table " + std::to_string(table_id) + " not in the pool");
    return it->second;
  }
  // ms per fwd+bwd step of the shard made of these pool positions (0 for an empty shard)
  double cost(std::vector<int32_t> positions) {
    if (positions.empty()) return 0.0;
    std::sort(positions.begin(), positions.end());
    auto it = cache_.find(positions);
    if (it != cache_.end()) {
      ++hits_;
      return it->second;
    }
    if (!sub_) {
      as_ctx* sub = nullptr;
      check(as_create_subset(parent_.get(), positions.data(), static_cast<int32_t>(positions.size()), &sub));
      sub_.reset(sub);
    } else {
      check(as_retarget_subset(sub_.get(), positions.data(), static_cast<int32_t>(positions.size())));
    }
    check(as_load_workload(sub_.get(), view_.get(), nullptr));
    double ms = 0.0;
    check(as_measure(sub_.get(), warmup_, measure_, trim_, flush_ ? 1 : 0, 0.01f, 1e-8f, &ms));
    cache_.emplace(std::move(positions), ms);
    ++measured_;
    return ms;
  }
  template <class Tables>
  double cost_of_tables(const Tables& tables) {
    std::vector<int32_t> p;
    for (const auto& t : tables) p.push_back(position(t.id));
    return cost(std::move(p));
  }
  // per-shard ms of a plan over a task drawn from the pool (measure_plan's shape)
  template <class Plan, class Task>
  std::vector<double> plan_costs(const Plan& plan, const Task& task) {
    std::vector<std::vector<int32_t>> members(static_cast<size_t>(task.num_shards));
    for (size_t i = 0; i < plan.assignment.size(); ++i)
      members.at(static_cast<size_t>(plan.assignment[i])).push_back(position(task.tables[i].id));
    std::vector<double> c;
    for (auto& m : members) c.push_back(cost(std::move(m)));
    return c;
  }
  size_t measured() const { return measured_; }
  size_t hits() const { return hits_; }

 private:
  struct CtxDel {
    void operator()(as_ctx* c) const { as_destroy(c); }
  };
  Shard parent_;
  std::unique_ptr<as_ctx, CtxDel> sub_;  // one subset context, retargeted per shard
  WorkloadView view_;
  int warmup_, measure_, trim_;
  bool flush_;
  std::unordered_map<int, int> pos_of_;
  std::map<std::vector<int32_t>, double> cache_;
  size_t measured_ = 0, hits_ = 0;
};

}  // namespace gpu
}  // namespace autoshard
