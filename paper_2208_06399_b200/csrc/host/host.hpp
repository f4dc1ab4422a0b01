// Host-side (C++) half of the B200 AutoShard hot path: the L1 types, the
// bit-exact synthetic generator, planners and file formats that sit above the
// C-ABI (include/autoshard_b200.h). Reference semantics are cited per
// function; nothing here touches the GPU except workload pinning.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "autoshard_b200.h"

namespace asb {

// Carries an as_status across C++ frames; the C-ABI layer converts it back
// (exception taxonomy of common.hpp:15-50).
struct Error : std::runtime_error {
  as_status code;
  Error(as_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(as_status c, const std::string& m) { throw Error(c, m); }

// ---- seeds and hashing (common.hpp:52-80) --------------------------------
uint64_t fnv1a64(const void* p, size_t n, uint64_t h = 0xcbf29ce484222325ull);
uint64_t splitmix64(uint64_t x);
uint64_t derive_seed(uint64_t master, const char* stream, uint64_t index = 0);

// ---- random streams (rng.hpp:15-131) -------------------------------------
// std::mt19937_64 is specified bit-exactly by the standard; the transforms are
// written out by hand (the std distributions are not portable) and the build
// uses -ffp-contract=off so double arithmetic rounds like the reference's
// canonical build.
class Stream64 {
 public:
  explicit Stream64(uint64_t seed) : eng_(seed) {}
  double unit() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  double log_uniform(double lo, double hi);
  uint64_t below(uint64_t n);
  double lomax(double alpha, double lambda);

 private:
  std::mt19937_64 eng_;
};

// Zipf(n, s) over ranks 1..n, rejection-inversion (rng.hpp:85-131).
class ZipfRanks {
 public:
  ZipfRanks(uint64_t n, double s);
  uint64_t draw(Stream64& r) const;

 private:
  double big_h(double x) const;
  double small_h(double x) const;
  double big_h_inv(double x) const;
  uint64_t n_;
  double s_, lo_, hi_, cut_;
};

// ---- workload (tables.hpp:43-60) -----------------------------------------
struct HostStream {
  int32_t table_id = 0;
  std::vector<int64_t> offsets;  // batch + 1
  std::vector<int64_t> indices;
};

struct HostWorkload {
  int64_t batch_size = 0;
  std::vector<HostStream> per_table;  // ascending table_id
  bool pinned = false;
  int find(int32_t table_id) const;  // position or -1
  ~HostWorkload();
};

struct GenConfig {
  double hash_size_min = 1e3, hash_size_max = 1e7;
  double pooling_mean_target = 15.0, pooling_shape = 2.0, pooling_cap = 193.0;
  std::vector<int32_t> dim_choices = {16, 32};
  double access_ratio_min = 1e-3, access_ratio_max = 1.0;
  int32_t bytes_per_param = 2;
  void validate() const;
};

std::vector<as_table_spec> generate_pool(uint64_t seed, int n, const GenConfig& cfg);
HostStream generate_stream(uint64_t seed, const as_table_spec& t, int64_t batch, double zipf);
void generate_workload(uint64_t seed, const std::vector<as_table_spec>& tables, int64_t batch,
                       double zipf, int n_threads, HostWorkload* out);

// ---- files (workload_io.hpp) ---------------------------------------------
void save_pool(const std::string& path, const std::vector<as_table_spec>& tables);
std::vector<as_table_spec> load_pool(const std::string& path);
void save_workload(const std::string& path, const HostWorkload& wl,
                   const std::vector<as_table_spec>& tables);
void load_workload(const std::string& path, HostWorkload* wl, std::vector<as_table_spec>* tables);

// ---- fingerprints (tables.hpp:417-441) -----------------------------------
uint64_t fingerprint_pool(const as_table_spec* t, int n);
uint64_t fingerprint_task(const as_table_spec* t, int n, int k, const int64_t* budgets);

// ---- plans (tables.hpp:63-143, planners.hpp) -----------------------------
inline int64_t size_bytes(const as_table_spec& t) {
  return static_cast<int64_t>(t.dim) * t.hash_size * t.bytes_per_param;
}
void validate_task(int k, const int64_t* budgets);
void validate_plan(int n, int k, const int32_t* assignment);
double heuristic_cost(const as_table_spec& t, int kind);
void greedy_shard(const as_table_spec* t, int n, int k, const int64_t* budgets, int kind,
                  int32_t* out);
void random_shard(const as_table_spec* t, int n, int k, const int64_t* budgets, uint64_t seed,
                  int32_t* out);
double degree_of_balance(const double* c, int n);
void save_plan(const std::string& path, const as_table_spec* t, int n, int k,
               const int64_t* budgets, const int32_t* assignment, const double* costs);
bool load_plan(const std::string& path, const as_table_spec* t, int n, int k,
               const int64_t* budgets, int32_t* assignment, double* costs);

}  // namespace asb
