// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/autoshard (compiled in place by
// oracle/Makefile into oracle/_ref/libref.so; no reference source is copied
// into this repo). It lets tests/ and tests/golden/make_golden.py call the
// real reference generator, planners and SIM cost hook through ctypes, so the
// C restatement in oracle/oracle.c and the product host library can be pinned
// against it bit-for-bit.
//
// Build flags follow SURVEY.md §8c: -std=gnu++20 -O3 -ffp-contract=off
// -include memory (planners.hpp:153 lacks <memory>).

#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "autoshard/common.hpp"
#include "autoshard/planners.hpp"
#include "autoshard/simcost.hpp"
#include "autoshard/tables.hpp"
#include "autoshard/workload_io.hpp"

namespace {

// Same layout as as_table_spec in include/autoshard_b200.h.
struct RefTable {
  int32_t id;
  int32_t dim;
  int64_t hash_size;
  double pooling_mean;
  double access_ratio;
  int32_t bytes_per_param;
  int32_t _pad;
};

autoshard::TableDesc to_desc(const RefTable& r) {
  autoshard::TableDesc t;
  t.id = r.id;
  t.dim = r.dim;
  t.hash_size = r.hash_size;
  t.pooling_mean = r.pooling_mean;
  t.access_ratio = r.access_ratio;
  t.bytes_per_param = r.bytes_per_param;
  return t;
}

RefTable from_desc(const autoshard::TableDesc& t) {
  RefTable r{};
  r.id = t.id;
  r.dim = t.dim;
  r.hash_size = t.hash_size;
  r.pooling_mean = t.pooling_mean;
  r.access_ratio = t.access_ratio;
  r.bytes_per_param = t.bytes_per_param;
  return r;
}

std::vector<autoshard::TableDesc> to_descs(const RefTable* t, int n) {
  std::vector<autoshard::TableDesc> v;
  for (int i = 0; i < n; ++i) v.push_back(to_desc(t[i]));
  return v;
}

thread_local std::string g_err;

int code_of(const std::exception& e) {
  if (dynamic_cast<const autoshard::OffsetError*>(&e)) return 3;
  if (dynamic_cast<const autoshard::IndexError*>(&e)) return 4;
  if (dynamic_cast<const autoshard::ParseError*>(&e)) return 2;
  if (dynamic_cast<const autoshard::ConfigError*>(&e)) return 1;
  if (dynamic_cast<const autoshard::InfeasibleError*>(&e)) return 5;
  if (dynamic_cast<const autoshard::ShapeError*>(&e)) return 6;
  if (dynamic_cast<const autoshard::LookupError*>(&e)) return 7;
  if (dynamic_cast<const autoshard::GuardError*>(&e)) return 8;
  if (dynamic_cast<const autoshard::StateError*>(&e)) return 9;
  return 99;
}

struct RefWorkload {
  autoshard::Workload wl;
  std::vector<autoshard::TableDesc> tables;
};

}  // namespace

#define REF_TRY(body)               \
  try {                             \
    body;                           \
    return 0;                       \
  } catch (const std::exception& e) { \
    g_err = e.what();               \
    return code_of(e);              \
  }

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate_pool(uint64_t seed, int n, double hash_min, double hash_max,
                      double pooling_target, double pooling_shape,
                      double pooling_cap, const int* dims, int n_dims,
                      double access_min, double access_max, int bpp,
                      RefTable* out) {
  REF_TRY({
    autoshard::GeneratorConfig cfg;
    cfg.hash_size_min = hash_min;
    cfg.hash_size_max = hash_max;
    cfg.pooling_mean_target = pooling_target;
    cfg.pooling_shape = pooling_shape;
    cfg.pooling_cap = pooling_cap;
    cfg.dim_choices.assign(dims, dims + n_dims);
    cfg.access_ratio_min = access_min;
    cfg.access_ratio_max = access_max;
    cfg.bytes_per_param = bpp;
    auto pool = autoshard::generate_pool(seed, n, cfg);
    for (int i = 0; i < n; ++i) out[i] = from_desc(pool[i]);
  })
}

int ref_generate_workload(uint64_t seed, const RefTable* tables, int n,
                          int64_t batch, double zipf, void** handle) {
  REF_TRY({
    auto* w = new RefWorkload;
    w->tables = to_descs(tables, n);
    w->wl = autoshard::generate_workload(seed, w->tables, batch, zipf);
    *handle = w;
  })
}

// Table i (ascending id) of a generated workload; pointers stay valid until
// ref_workload_free.
int ref_workload_table(void* handle, int i, int* table_id,
                       const int64_t** offsets, int64_t* n_offsets,
                       const int64_t** indices, int64_t* n_indices) {
  auto* w = static_cast<RefWorkload*>(handle);
  const auto& s = w->wl.per_table.at(static_cast<size_t>(i));
  *table_id = s.table_id;
  *offsets = s.offsets.data();
  *n_offsets = static_cast<int64_t>(s.offsets.size());
  *indices = s.indices.data();
  *n_indices = static_cast<int64_t>(s.indices.size());
  return 0;
}

void ref_workload_free(void* handle) { delete static_cast<RefWorkload*>(handle); }

uint64_t ref_fnv1a64(const void* p, uint64_t n, uint64_t h) {
  return autoshard::fnv1a64(p, static_cast<size_t>(n), h);
}

uint64_t ref_fingerprint_pool(const RefTable* t, int n) {
  return autoshard::fingerprint(to_descs(t, n));
}

uint64_t ref_fingerprint_task(const RefTable* t, int n, int k,
                              const int64_t* budgets) {
  autoshard::ShardingTask task;
  task.tables = to_descs(t, n);
  task.num_shards = k;
  task.mem_budget.assign(budgets, budgets + k);
  return autoshard::fingerprint(task);
}

// fnv1a64 over save_pool(pool) bytes followed by save_workload(wl, tables)
// bytes (the SURVEY.md §8c canonical-build check).
int ref_serialized_hash(const RefTable* pool, int n_pool, void* handle,
                        uint64_t* hash, uint64_t* nbytes) {
  REF_TRY({
    auto* w = static_cast<RefWorkload*>(handle);
    std::ostringstream os;
    autoshard::save_pool(os, to_descs(pool, n_pool));
    autoshard::save_workload(os, w->wl, w->tables);
    const std::string s = os.str();
    *hash = autoshard::fnv1a64(s.data(), s.size());
    *nbytes = s.size();
  })
}

int ref_save_workload_file(const char* path, void* handle) {
  REF_TRY({
    auto* w = static_cast<RefWorkload*>(handle);
    autoshard::save_workload_file(path, w->wl, w->tables);
  })
}

int ref_load_workload_file(const char* path, void** handle) {
  REF_TRY({
    auto lw = autoshard::load_workload_file(path);
    auto* w = new RefWorkload;
    w->wl = std::move(lw.workload);
    w->tables = std::move(lw.tables);
    *handle = w;
  })
}

// kind: 0 size, 1 dim, 2 lookup (HeuristicKind order, planners.hpp:20).
int ref_greedy_shard(const RefTable* t, int n, int k, const int64_t* budgets,
                     int kind, int* assignment) {
  REF_TRY({
    autoshard::ShardingTask task;
    task.tables = to_descs(t, n);
    task.num_shards = k;
    task.mem_budget.assign(budgets, budgets + k);
    auto plan = autoshard::greedy_shard(
        task, static_cast<autoshard::HeuristicKind>(kind));
    for (int i = 0; i < n; ++i) assignment[i] = plan.assignment[i];
  })
}

int ref_random_shard(const RefTable* t, int n, int k, const int64_t* budgets,
                     uint64_t seed, int* assignment) {
  REF_TRY({
    autoshard::ShardingTask task;
    task.tables = to_descs(t, n);
    task.num_shards = k;
    task.mem_budget.assign(budgets, budgets + k);
    auto plan = autoshard::random_shard(task, seed);
    for (int i = 0; i < n; ++i) assignment[i] = plan.assignment[i];
  })
}

int ref_degree_of_balance(const double* c, int n, double* out) {
  REF_TRY({ *out = autoshard::degree_of_balance(std::vector<double>(c, c + n)); })
}

// SIM measure_plan with default SimParams (simcost.hpp:194) — the reference's
// own CPU "cost of the path", timed by bench.py --impl reference beside the
// embedding-bag port.
int ref_measure_plan(const RefTable* t, int n, int k, const int64_t* budgets,
                     const int* assignment, void* handle, int warmup,
                     int measure, int trim, int exact, uint64_t seed,
                     double* costs) {
  REF_TRY({
    auto* w = static_cast<RefWorkload*>(handle);
    autoshard::ShardingTask task;
    task.tables = to_descs(t, n);
    task.num_shards = k;
    task.mem_budget.assign(budgets, budgets + k);
    autoshard::ShardingPlan plan;
    plan.assignment.assign(assignment, assignment + n);
    autoshard::BenchConfig bc;
    bc.warmup = warmup;
    bc.measure = measure;
    bc.trim = trim;
    bc.exact = exact != 0;
    bc.seed = seed;
    auto v = autoshard::measure_plan(plan, task, w->wl, autoshard::SimParams{}, bc);
    for (int i = 0; i < k; ++i) costs[i] = v[i];
  })
}

// extract_features raw vectors (tables.hpp:344-386), identity norm stats.
int ref_extract_features(const RefTable* t, int n, void* handle, double* out) {
  REF_TRY({
    auto* w = static_cast<RefWorkload*>(handle);
    autoshard::NormStats ns;
    for (int i = 0; i < n; ++i) {
      const auto f = autoshard::extract_features(to_desc(t[i]), w->wl, ns);
      for (int k = 0; k < autoshard::kNumFeatures; ++k) out[i * autoshard::kNumFeatures + k] = f.raw[k];
    }
  })
}

}  // extern "C"
