// Plans and planners: ShardingTask/ShardingPlan checks (tables.hpp:63-143),
// heuristic greedy and random sharding (planners.hpp:32-144), and the plan
// file of SPEC.md:291 ("version, task fingerprint, assignment array, and the
// evaluator's per-shard costs if available"; the reference CLI that would
// write it is absent, so the concrete text layout is defined here).
#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <sstream>

#include "host.hpp"

namespace asb {

void validate_task(int k, const int64_t* budgets) {
  if (k < 1) fail(AS_CONFIG, "task: num_shards must be >= 1");
  for (int i = 0; i < k; ++i)
    if (budgets[i] <= 0) fail(AS_CONFIG, "task: all memory budgets must be > 0");
}

void validate_plan(int n, int k, const int32_t* a) {
  for (int i = 0; i < n; ++i)
    if (a[i] < 0 || a[i] >= k)
      fail(AS_CONFIG, "plan: table index " + std::to_string(i) + " assigned to invalid shard " +
                          std::to_string(a[i]));
}

double heuristic_cost(const as_table_spec& t, int kind) {
  switch (kind) {
    case 0: return static_cast<double>(t.dim) * static_cast<double>(t.hash_size);
    case 1: return static_cast<double>(t.dim);
    case 2: return static_cast<double>(t.dim) * t.pooling_mean;  // declared pooling (planners.hpp:39)
    case 3: fail(AS_CONFIG, "heuristic_cost: rand has no cost function");
    default: fail(AS_CONFIG, "heuristic_cost: unknown kind " + std::to_string(kind));
  }
}

namespace {
void check_aggregate(const as_table_spec* t, int n, int k, const int64_t* budgets) {
  int64_t total = 0, budget = 0;
  for (int i = 0; i < n; ++i) total += size_bytes(t[i]);
  for (int i = 0; i < k; ++i) budget += budgets[i];
  if (total > budget)
    fail(AS_INFEASIBLE, "task infeasible: total table bytes " + std::to_string(total) +
                            " exceed total budget " + std::to_string(budget) + " by " +
                            std::to_string(total - budget));
}
int most_free(const std::vector<int64_t>& f) {
  return static_cast<int>(std::max_element(f.begin(), f.end()) - f.begin());  // first max
}
}  // namespace

void greedy_shard(const as_table_spec* t, int n, int k, const int64_t* budgets, int kind,
                  int32_t* out) {
  if (kind == 3) fail(AS_CONFIG, "greedy_shard: use random_shard for kind=rand");
  validate_task(k, budgets);
  check_aggregate(t, n, k, budgets);
  std::vector<double> cost(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) cost[i] = heuristic_cost(t[i], kind);
  std::vector<int> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int x, int y) {
    if (cost[x] != cost[y]) return cost[x] > cost[y];
    return t[x].id < t[y].id;
  });
  std::vector<double> load(static_cast<size_t>(k), 0.0);
  std::vector<int64_t> free_b(budgets, budgets + k);
  for (int i : order) {
    const int64_t sz = size_bytes(t[i]);
    int pick = -1;
    for (int s = 0; s < k; ++s)
      if (free_b[s] >= sz && (pick < 0 || load[s] < load[pick])) pick = s;
    if (pick < 0) pick = most_free(free_b);
    out[i] = pick;
    load[pick] += cost[i];
    free_b[pick] -= sz;
  }
}

void random_shard(const as_table_spec* t, int n, int k, const int64_t* budgets, uint64_t seed,
                  int32_t* out) {
  validate_task(k, budgets);
  check_aggregate(t, n, k, budgets);
  Stream64 r(derive_seed(seed, "random-shard"));
  std::vector<int64_t> free_b(budgets, budgets + k);
  for (int i = 0; i < n; ++i) {
    const int64_t sz = size_bytes(t[i]);
    int pick = -1;
    for (int attempt = 0; attempt < 16 && pick < 0; ++attempt) {
      const int s = static_cast<int>(r.below(static_cast<uint64_t>(k)));
      if (free_b[s] >= sz) pick = s;
    }
    if (pick < 0) pick = most_free(free_b);
    out[i] = pick;
    free_b[pick] -= sz;
  }
}

double degree_of_balance(const double* c, int n) {
  if (n < 1) fail(AS_CONFIG, "degree_of_balance: empty cost vector");
  const auto mm = std::minmax_element(c, c + n);
  if (*mm.second <= 0.0) return 1.0;
  return *mm.first / *mm.second;
}

// ---- plan file --------------------------------------------------------------
//   autoshard-plan 1
//   fingerprint <16 hex digits of fingerprint(ShardingTask)>
//   num_shards <K>
//   tables <N>
//   assignment <a_0> ... <a_{N-1}>
//   costs <c_0> ... <c_{K-1}>      (optional, %.17g ms)
//   end
void save_plan(const std::string& path, const as_table_spec* t, int n, int k,
               const int64_t* budgets, const int32_t* a, const double* costs) {
  validate_task(k, budgets);
  validate_plan(n, k, a);
  std::ofstream os(path);
  if (!os) fail(AS_PARSE, "cannot open for writing: " + path);
  char fp[32];
  std::snprintf(fp, sizeof fp, "%016" PRIx64, fingerprint_task(t, n, k, budgets));
  os << "autoshard-plan 1\nfingerprint " << fp << "\nnum_shards " << k << "\ntables " << n
     << "\nassignment";
  for (int i = 0; i < n; ++i) os << ' ' << a[i];
  os << "\n";
  if (costs) {
    os << "costs";
    char buf[40];
    for (int i = 0; i < k; ++i) {
      std::snprintf(buf, sizeof buf, "%.17g", costs[i]);
      os << ' ' << buf;
    }
    os << "\n";
  }
  os << "end\n";
  if (!os) fail(AS_PARSE, "failed writing plan file " + path);
}

bool load_plan(const std::string& path, const as_table_spec* t, int n, int k,
               const int64_t* budgets, int32_t* a, double* costs) {
  std::ifstream is(path);
  if (!is) fail(AS_PARSE, "cannot open: " + path);
  std::string line, tag;
  auto next = [&](const char* what) {
    if (!std::getline(is, line)) fail(AS_PARSE, std::string("truncated plan file while reading ") + what);
    if (!line.empty() && line.back() == '\r') line.pop_back();
    return std::istringstream(line);
  };
  if (next("magic").str() != "autoshard-plan 1") fail(AS_PARSE, "bad plan magic/version: '" + line + "'");
  std::string fp;
  { auto s = next("fingerprint"); if (!(s >> tag >> fp) || tag != "fingerprint") fail(AS_PARSE, "malformed fingerprint line"); }
  int kk = 0, nn = 0;
  { auto s = next("num_shards"); if (!(s >> tag >> kk) || tag != "num_shards") fail(AS_PARSE, "malformed num_shards line"); }
  { auto s = next("tables"); if (!(s >> tag >> nn) || tag != "tables") fail(AS_PARSE, "malformed tables line"); }
  if (kk != k || nn != n)
    fail(AS_STATE, "plan file is for " + std::to_string(nn) + " tables / " + std::to_string(kk) +
                       " shards, task has " + std::to_string(n) + " / " + std::to_string(k));
  char want[32];
  std::snprintf(want, sizeof want, "%016" PRIx64, fingerprint_task(t, n, k, budgets));
  if (fp != want) fail(AS_STATE, "plan fingerprint " + fp + " does not match task fingerprint " + want);
  {
    auto s = next("assignment");
    if (!(s >> tag) || tag != "assignment") fail(AS_PARSE, "malformed assignment line");
    for (int i = 0; i < n; ++i)
      if (!(s >> a[i])) fail(AS_PARSE, "assignment line too short");
  }
  validate_plan(n, k, a);
  bool has_costs = false;
  auto s = next("costs/end");
  s >> tag;
  if (tag == "costs") {
    for (int i = 0; i < k; ++i) {
      double v;
      if (!(s >> v)) fail(AS_PARSE, "costs line too short");
      if (costs) costs[i] = v;
    }
    has_costs = true;
    auto e = next("end");
    e >> tag;
  }
  if (tag != "end") fail(AS_PARSE, "missing end in plan file");
  return has_costs;
}

}  // namespace asb
