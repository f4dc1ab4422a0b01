/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the AutoShard
 * embedding-bag hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load liboracle.so. The product
 * (paper_2208_06399_b200/) never links or calls it.
 *
 * Plain-C restatement of the reference algorithm:
 *   - generator:  autoshard/common.hpp:52-80, autoshard/rng.hpp:15-131,
 *                 autoshard/tables.hpp:149-288
 *   - planners:   autoshard/planners.hpp:32-144
 *   - fingerprints: autoshard/tables.hpp:417-441
 * pinned bit-for-bit against the reference compiled in place
 * (oracle/_ref/libref.so, see oracle/Makefile) and against the golden
 * hashes of SURVEY.md §8c (tests/test_oracle.py).
 *
 * The embedding-bag arithmetic (sum-pooled forward, backward with exact
 * row-wise Adagrad) does NOT exist in the reference: it is
 * restated from PAPER.md:639,646,659 and FBGEMM's exact_rowwise_adagrad
 * semantics. That part is "parity unpinned" against the reference — it is
 * pinned instead against torch.nn.functional.embedding_bag (tests).
 */
#ifndef AUTOSHARD_ORACLE_H
#define AUTOSHARD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as as_table_spec (include/autoshard_b200.h) and TableDesc
 * (autoshard/tables.hpp:24-38). */
typedef struct {
  int32_t id;
  int32_t dim;
  int64_t hash_size;
  double pooling_mean;
  double access_ratio;
  int32_t bytes_per_param;
  int32_t _pad;
} orc_table;

typedef struct {
  double hash_size_min, hash_size_max;
  double pooling_mean_target, pooling_shape, pooling_cap;
  const int32_t* dim_choices;
  int32_t n_dim_choices;
  double access_ratio_min, access_ratio_max;
  int32_t bytes_per_param;
} orc_gen_cfg;

/* error codes mirror as_status */
enum { ORC_OK = 0, ORC_CONFIG = 1, ORC_INFEASIBLE = 5 };

uint64_t orc_fnv1a64(const void* p, size_t n, uint64_t h);
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t master, const char* stream, uint64_t index);

int orc_generate_pool(uint64_t seed, int n, const orc_gen_cfg* cfg, orc_table* out);
/* One table's stream (tables.hpp:258-286). *offsets has B+1 entries; both
 * arrays are malloc'd, free with orc_free. */
int orc_generate_stream(uint64_t seed, const orc_table* t, int64_t batch,
                        double zipf, int64_t** offsets, int64_t** indices,
                        int64_t* n_indices);
void orc_free(void* p);

uint64_t orc_fingerprint_pool(const orc_table* t, int n);
uint64_t orc_fingerprint_task(const orc_table* t, int n, int k, const int64_t* budgets);

/* kind: 0 size, 1 dim, 2 lookup (planners.hpp:20) */
int orc_greedy_shard(const orc_table* t, int n, int k, const int64_t* budgets,
                     int kind, int* assignment);
int orc_random_shard(const orc_table* t, int n, int k, const int64_t* budgets,
                     uint64_t seed, int* assignment);
double orc_degree_of_balance(const double* c, int n);

/* ---- embedding-bag arithmetic (restated; see header comment) ---- */

/* Initial weight W_t[row, d]: splitmix64 counter hash mapped to a 10-bit grid
 * k * 2^-12, k in [-512, 511]. Same definition as the device init kernel
 * (DESIGN.md "weight init"). */
float orc_weight_init(uint64_t seed, int32_t table_id, int64_t row, int32_t d);
/* Dense init of a whole table (OpenMP), out [rows, dim]. */
void orc_fill_weights(uint64_t seed, int32_t table_id, int64_t rows, int32_t dim, float* out);
/* Synthetic gradient G[b, col]: same grid, independent stream. */
float orc_grad_init(uint64_t seed, int64_t b, int64_t col);

/* Sum-pooled forward in fp64. out is [B, sum_dim] row-major, table columns in
 * the given table order. W[t] is a dense [hash, dim] fp32 table, or NULL to
 * use orc_weight_init(wseed, ...) on the fly. */
void orc_emb_forward_f64_rows(int T, const orc_table* tabs, int64_t B, int64_t b0, int64_t b1,
                              const int64_t* const* offsets, const int64_t* const* indices,
                              const float* const* W, uint64_t wseed, double* out);
void orc_emb_forward_f64(int T, const orc_table* tabs, int64_t B,
                         const int64_t* const* offsets,
                         const int64_t* const* indices, const float* const* W,
                         uint64_t wseed, double* out);

/* Backward + exact row-wise Adagrad (fp64 math) for one table. grad is
 * [B, grad_stride] fp32 and the table's columns start at col0. Outputs
 * (malloc'd, caller frees with orc_free): ascending unique rows, their counts,
 * the updated rows [U, dim] and momentum [U] in fp64. W / M: dense fp32 table
 * and momentum or NULL (hash init / zero). When W and M are given they are
 * also updated in place (rounded to fp32). */
int orc_emb_backward_adagrad_f64(const orc_table* t, int64_t B,
                                 const int64_t* offsets, const int64_t* indices,
                                 const float* grad, int64_t grad_stride,
                                 int64_t col0, float* W, float* M,
                                 uint64_t wseed, double lr, double eps,
                                 int64_t* n_unique, int64_t** rows,
                                 int64_t** counts, double** new_w,
                                 double** new_m);

/* fp32, OpenMP CPU implementation of one fwd+bwd step (the CPU baseline that
 * bench.py times; kind "port"). Tables packed like the device: W_all is
 * the concatenation of dense tables, M_all of momenta. Uses loss 1/2|out|^2
 * (grad = out). Returns the thread count used. */
int orc_cpu_step_f32(int T, const int32_t* dims, const int64_t* hash,
                     int64_t B, const int64_t* const* offsets,
                     const int64_t* const* indices, float* W_all, float* M_all,
                     float* out, float lr, float eps, int n_threads);

#ifdef __cplusplus
}
#endif
#endif
