// Bit-exact synthetic table pool and lookup streams.
// Semantics: autoshard/rng.hpp:15-131, autoshard/tables.hpp:149-288.
// Pinned by tests/test_host.py against the reference built in place and the
// SURVEY.md §8c golden hashes.
//
// B200-side differences from the reference: tables are generated in parallel
// (each table has its own seeded stream, tables.hpp:260-261, so this is still
// bit-exact), largest expected streams first.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <thread>

#include "host.hpp"

namespace asb {

uint64_t fnv1a64(const void* p, size_t n, uint64_t h) {
  const auto* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 0x100000001b3ull;
  return h;
}

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

uint64_t derive_seed(uint64_t master, const char* stream, uint64_t index) {
  const uint64_t name = fnv1a64(stream, std::strlen(stream));
  const uint64_t inner = splitmix64(name + 0x9e3779b97f4a7c15ull * (index + 1));
  return splitmix64(master ^ inner);
}

double Stream64::log_uniform(double lo, double hi) {
  const double a = std::log(lo);
  const double b = std::log(hi);
  return std::exp(a + (b - a) * unit());
}

uint64_t Stream64::below(uint64_t n) {
  if (n == 0) fail(AS_CONFIG, "Rng::below: n must be positive");
  constexpr uint64_t kMax = std::numeric_limits<uint64_t>::max();
  const uint64_t limit = kMax - kMax % n;
  for (;;) {
    const uint64_t x = eng_();
    if (x < limit) return x % n;
  }
}

double Stream64::lomax(double alpha, double lambda) {
  if (lambda <= 0.0) return 0.0;  // consumes no draw
  const double u = unit();
  return lambda * (std::pow(1.0 - u, -1.0 / alpha) - 1.0);
}

// --- Zipf by rejection-inversion ------------------------------------------
namespace {
inline double log1p_over_x(double x) {
  return std::fabs(x) > 1e-8 ? std::log1p(x) / x : 1.0 - x / 2.0 + x * x / 3.0;
}
inline double expm1_over_x(double x) {
  return std::fabs(x) > 1e-8 ? std::expm1(x) / x : 1.0 + x / 2.0 + x * x / 6.0;
}
}  // namespace

double ZipfRanks::big_h(double x) const {
  const double lx = std::log(x);
  return expm1_over_x((1.0 - s_) * lx) * lx;
}
double ZipfRanks::small_h(double x) const { return std::exp(-s_ * std::log(x)); }
double ZipfRanks::big_h_inv(double x) const {
  double t = x * (1.0 - s_);
  if (t < -1.0) t = -1.0;
  return std::exp(log1p_over_x(t) * x);
}

ZipfRanks::ZipfRanks(uint64_t n, double s) : n_(n), s_(s) {
  if (n == 0) fail(AS_CONFIG, "ZipfSampler: n must be positive");
  if (s <= 0.0) fail(AS_CONFIG, "ZipfSampler: exponent must be positive");
  lo_ = big_h(1.5) - 1.0;
  hi_ = big_h(static_cast<double>(n) + 0.5);
  cut_ = 2.0 - big_h_inv(big_h(2.5) - small_h(2.0));
}

uint64_t ZipfRanks::draw(Stream64& r) const {
  if (n_ == 1) return 1;
  const double nd = static_cast<double>(n_);
  for (;;) {
    const double u = hi_ + r.unit() * (lo_ - hi_);
    const double x = big_h_inv(u);
    double k = std::floor(x + 0.5);
    k = k < 1.0 ? 1.0 : (k > nd ? nd : k);
    if (k - x <= cut_ || u >= big_h(k + 0.5) - small_h(k)) return static_cast<uint64_t>(k);
  }
}

// --- pool ------------------------------------------------------------------
void GenConfig::validate() const {
  if (hash_size_min < 1.0 || hash_size_max < hash_size_min)
    fail(AS_CONFIG, "generator: hash_size range empty or inverted");
  if (dim_choices.empty()) fail(AS_CONFIG, "generator: dim_choices must be non-empty");
  if (access_ratio_min <= 0.0 || access_ratio_max < access_ratio_min || access_ratio_max > 1.0)
    fail(AS_CONFIG, "generator: access_ratio range empty or inverted");
  if (pooling_mean_target < 0.0 || pooling_shape <= 1.0 || pooling_cap <= 0.0)
    fail(AS_CONFIG, "generator: bad pooling parameters");
  if (bytes_per_param < 1) fail(AS_CONFIG, "generator: bytes_per_param must be >= 1");
}

std::vector<as_table_spec> generate_pool(uint64_t seed, int n, const GenConfig& cfg) {
  cfg.validate();
  if (n < 1) fail(AS_CONFIG, "generate_pool: n_tables must be >= 1");
  const double lambda = cfg.pooling_mean_target * (cfg.pooling_shape - 1.0);
  std::vector<as_table_spec> pool(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    Stream64 r(derive_seed(seed, "pool-table", static_cast<uint64_t>(i)));
    as_table_spec& t = pool[static_cast<size_t>(i)];
    std::memset(&t, 0, sizeof t);
    t.id = i;
    // draw order: hash, pooling, dim, access (tables.hpp:189-195)
    const long long h = std::llround(r.log_uniform(cfg.hash_size_min, cfg.hash_size_max));
    t.hash_size = std::max<long long>(h, 1);
    t.pooling_mean = std::min(r.lomax(cfg.pooling_shape, lambda), cfg.pooling_cap);
    t.dim = cfg.dim_choices[r.below(cfg.dim_choices.size())];
    t.access_ratio = r.log_uniform(cfg.access_ratio_min, cfg.access_ratio_max);
    t.bytes_per_param = cfg.bytes_per_param;
  }
  return pool;
}

// --- streams ---------------------------------------------------------------
HostStream generate_stream(uint64_t seed, const as_table_spec& t, int64_t batch, double zipf) {
  if (t.hash_size < 1)
    fail(AS_CONFIG, "generate_workload: table " + std::to_string(t.id) + " has invalid hash_size");
  Stream64 r(derive_seed(seed, "workload-table", static_cast<uint64_t>(t.id)));
  HostStream s;
  s.table_id = t.id;
  const int64_t hash = t.hash_size;
  const int64_t accessible =
      std::clamp<int64_t>(static_cast<int64_t>(std::ceil(t.access_ratio * static_cast<double>(hash))),
                          1, hash);
  // Warm-row permutation j -> (a*j + b) mod hash with gcd(a, hash) = 1
  // (tables.hpp:210-230).
  int64_t a = 1, b = 0;
  if (hash != 1) {
    do {
      a = 1 + static_cast<int64_t>(r.below(static_cast<uint64_t>(hash - 1)));
    } while (std::gcd(a, hash) != 1);
    b = static_cast<int64_t>(r.below(static_cast<uint64_t>(hash)));
  }
  const ZipfRanks zipf_ranks(static_cast<uint64_t>(accessible), zipf);
  s.offsets.resize(static_cast<size_t>(batch) + 1);
  s.offsets[0] = 0;
  // Expected length pooling_mean * batch; reserve a little above it.
  s.indices.reserve(static_cast<size_t>(t.pooling_mean * 1.1 * static_cast<double>(batch)) + 16);
  const double lam = 2.0 * t.pooling_mean;
  for (int64_t q = 0; q < batch; ++q) {
    const double x = r.lomax(3.0, lam);
    const double fl = std::floor(x);
    int64_t cnt = static_cast<int64_t>(fl);
    if (r.unit() < x - fl) ++cnt;  // stochastic rounding, one draw per bag
    for (int64_t j = 0; j < cnt; ++j) {
      const int64_t slot = static_cast<int64_t>(zipf_ranks.draw(r)) - 1;
      s.indices.push_back((a * slot + b) % hash);
    }
    s.offsets[static_cast<size_t>(q) + 1] = static_cast<int64_t>(s.indices.size());
  }
  return s;
}

void generate_workload(uint64_t seed, const std::vector<as_table_spec>& tables, int64_t batch,
                       double zipf, int n_threads, HostWorkload* out) {
  if (batch < 1) fail(AS_CONFIG, "generate_workload: batch_size must be >= 1");
  std::vector<as_table_spec> sorted(tables);
  for (const auto& t : sorted)
    if (t.hash_size < 1)
      fail(AS_CONFIG, "generate_workload: table " + std::to_string(t.id) + " has invalid hash_size");
  std::sort(sorted.begin(), sorted.end(),
            [](const as_table_spec& x, const as_table_spec& y) { return x.id < y.id; });
  out->batch_size = batch;
  out->per_table.assign(sorted.size(), HostStream{});
  // Largest expected streams first for load balance across threads.
  std::vector<size_t> order(sorted.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    return sorted[x].pooling_mean > sorted[y].pooling_mean;
  });
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned nt = n_threads > 0 ? static_cast<unsigned>(n_threads) : hw;
  nt = std::min<unsigned>(nt, static_cast<unsigned>(std::max<size_t>(1, sorted.size())));
  std::atomic<size_t> next{0};
  std::vector<std::exception_ptr> errs(nt);
  auto worker = [&](unsigned w) {
    try {
      for (size_t k; (k = next.fetch_add(1)) < order.size();) {
        const size_t i = order[k];
        out->per_table[i] = generate_stream(seed, sorted[i], batch, zipf);
      }
    } catch (...) {
      errs[w] = std::current_exception();
    }
  };
  if (nt <= 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (unsigned w = 0; w < nt; ++w) th.emplace_back(worker, w);
    for (auto& x : th) x.join();
  }
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

int HostWorkload::find(int32_t table_id) const {
  auto it = std::lower_bound(per_table.begin(), per_table.end(), table_id,
                             [](const HostStream& s, int32_t id) { return s.table_id < id; });
  if (it == per_table.end() || it->table_id != table_id) return -1;
  return static_cast<int>(it - per_table.begin());
}

// --- fingerprints (tables.hpp:417-441) -------------------------------------
namespace {
uint64_t mix_table(const as_table_spec& t, uint64_t h) {
  h = fnv1a64(&t.id, sizeof t.id, h);
  h = fnv1a64(&t.dim, sizeof t.dim, h);
  h = fnv1a64(&t.hash_size, sizeof t.hash_size, h);
  h = fnv1a64(&t.pooling_mean, sizeof t.pooling_mean, h);
  h = fnv1a64(&t.access_ratio, sizeof t.access_ratio, h);
  h = fnv1a64(&t.bytes_per_param, sizeof t.bytes_per_param, h);
  return h;
}
}  // namespace

uint64_t fingerprint_pool(const as_table_spec* t, int n) {
  uint64_t h = fnv1a64("pool", 4);
  for (int i = 0; i < n; ++i) h = mix_table(t[i], h);
  return h;
}

uint64_t fingerprint_task(const as_table_spec* t, int n, int k, const int64_t* budgets) {
  uint64_t h = fnv1a64("task", 4);
  h = fingerprint_pool(t, n) ^ h;
  h = fnv1a64(&k, sizeof k, h);
  for (int i = 0; i < k; ++i) h = fnv1a64(&budgets[i], sizeof(int64_t), h);
  return h;
}

}  // namespace asb
