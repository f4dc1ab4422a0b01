/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the AutoShard embedding-bag hot
 * path (see oracle.h for scope and who may call it). Compiled with
 * -O2 -ffp-contract=off so double arithmetic matches the reference's
 * canonical build.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* hashing and seed streams — autoshard/common.hpp:52-80                     */
/* ------------------------------------------------------------------------ */

uint64_t orc_fnv1a64(const void* p, size_t n, uint64_t h) {
  const unsigned char* c = (const unsigned char*)p;
  for (size_t i = 0; i < n; ++i) {
    h ^= c[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

static const uint64_t FNV_BASIS = 0xcbf29ce484222325ull;

uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* common.hpp:76-80 */
uint64_t orc_derive_seed(uint64_t master, const char* stream, uint64_t index) {
  uint64_t h = orc_fnv1a64(stream, strlen(stream), FNV_BASIS);
  return orc_splitmix64(master ^ orc_splitmix64(h + 0x9e3779b97f4a7c15ull * (index + 1)));
}

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the engine behind autoshard::Rng, rng.hpp:15-72)              */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t s[MT_N];
  int i;
} mt64;

static void mt_seed(mt64* m, uint64_t seed) {
  m->s[0] = seed;
  for (int k = 1; k < MT_N; ++k)
    m->s[k] = 6364136223846793005ull * (m->s[k - 1] ^ (m->s[k - 1] >> 62)) + (uint64_t)k;
  m->i = MT_N;
}

static uint64_t mt_next(mt64* m) {
  if (m->i >= MT_N) {
    const uint64_t UP = 0xffffffff80000000ull, LO = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (m->s[k] & UP) | (m->s[(k + 1) % MT_N] & LO);
      m->s[k] = m->s[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1) ? A : 0);
    }
    m->i = 0;
  }
  uint64_t x = m->s[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71d67fffeda60000ull;
  x ^= (x << 37) & 0xfff7eee000000000ull;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:22-24: 53-bit uniform in [0,1), one draw */
static double rng_uniform(mt64* m) { return (double)(mt_next(m) >> 11) * 0x1.0p-53; }

/* rng.hpp:29-31 */
static double rng_log_uniform(mt64* m, double lo, double hi) {
  double a = log(lo), b = log(hi);
  double u = rng_uniform(m);
  return exp(a + (b - a) * u);
}

/* rng.hpp:34-44: unbiased rejection */
static uint64_t rng_below(mt64* m, uint64_t n) {
  uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = mt_next(m);
  } while (x >= limit);
  return x % n;
}

/* rng.hpp:76-80: Lomax inverse CDF, one draw unless lambda <= 0 */
static double rng_lomax(mt64* m, double alpha, double lambda) {
  if (lambda <= 0.0) return 0.0;
  double u = rng_uniform(m);
  return lambda * (pow(1.0 - u, -1.0 / alpha) - 1.0);
}

/* rng.hpp:85-131: Zipf by rejection-inversion (Hormann & Derflinger 1996). */
typedef struct {
  uint64_t n;
  double s, hx1, hn, cut;
} zipf_t;

static double zh1(double x) { return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x / 2.0 + x * x / 3.0; }
static double zh2(double x) { return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x / 2.0 + x * x / 6.0; }
static double zH(const zipf_t* z, double x) {
  double lx = log(x);
  return zh2((1.0 - z->s) * lx) * lx;
}
static double zh(const zipf_t* z, double x) { return exp(-z->s * log(x)); }
static double zHinv(const zipf_t* z, double x) {
  double t = x * (1.0 - z->s);
  if (t < -1.0) t = -1.0;
  return exp(zh1(t) * x);
}
static void zipf_init(zipf_t* z, uint64_t n, double s) {
  z->n = n;
  z->s = s;
  z->hx1 = zH(z, 1.5) - 1.0;
  z->hn = zH(z, (double)n + 0.5);
  z->cut = 2.0 - zHinv(z, zH(z, 2.5) - zh(z, 2.0));
}
static uint64_t zipf_draw(const zipf_t* z, mt64* m) {
  if (z->n == 1) return 1;
  for (;;) {
    double u = z->hn + rng_uniform(m) * (z->hx1 - z->hn);
    double x = zHinv(z, u);
    double k = floor(x + 0.5);
    if (k < 1.0) k = 1.0;
    if (k > (double)z->n) k = (double)z->n;
    if (k - x <= z->cut || u >= zH(z, k + 0.5) - zh(z, k)) return (uint64_t)k;
  }
}

/* ------------------------------------------------------------------------ */
/* generator — tables.hpp:149-288                                           */
/* ------------------------------------------------------------------------ */

static int cfg_valid(const orc_gen_cfg* c) {
  if (c->hash_size_min < 1.0 || c->hash_size_max < c->hash_size_min) return 0;
  if (c->n_dim_choices < 1) return 0;
  if (c->access_ratio_min <= 0.0 || c->access_ratio_max < c->access_ratio_min ||
      c->access_ratio_max > 1.0)
    return 0;
  if (c->pooling_mean_target < 0.0 || c->pooling_shape <= 1.0 || c->pooling_cap <= 0.0) return 0;
  if (c->bytes_per_param < 1) return 0;
  return 1;
}

int orc_generate_pool(uint64_t seed, int n, const orc_gen_cfg* cfg, orc_table* out) {
  if (!cfg_valid(cfg) || n < 1) return ORC_CONFIG;
  double lambda = cfg->pooling_mean_target * (cfg->pooling_shape - 1.0);
  for (int i = 0; i < n; ++i) {
    mt64 m;
    mt_seed(&m, orc_derive_seed(seed, "pool-table", (uint64_t)i));
    orc_table t;
    memset(&t, 0, sizeof t);
    t.id = i;
    long long h = llround(rng_log_uniform(&m, cfg->hash_size_min, cfg->hash_size_max));
    t.hash_size = h < 1 ? 1 : h;
    double pm = rng_lomax(&m, cfg->pooling_shape, lambda);
    t.pooling_mean = pm < cfg->pooling_cap ? pm : cfg->pooling_cap;
    t.dim = cfg->dim_choices[rng_below(&m, (uint64_t)cfg->n_dim_choices)];
    t.access_ratio = rng_log_uniform(&m, cfg->access_ratio_min, cfg->access_ratio_max);
    t.bytes_per_param = cfg->bytes_per_param;
    out[i] = t;
  }
  return ORC_OK;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    int64_t r = a % b;
    a = b;
    b = r;
  }
  return a < 0 ? -a : a;
}

int orc_generate_stream(uint64_t seed, const orc_table* t, int64_t batch, double zipf,
                        int64_t** offsets_out, int64_t** indices_out, int64_t* n_out) {
  if (batch < 1 || t->hash_size < 1) return ORC_CONFIG;
  mt64 m;
  mt_seed(&m, orc_derive_seed(seed, "workload-table", (uint64_t)t->id));
  const int64_t hash = t->hash_size;
  int64_t acc = (int64_t)ceil(t->access_ratio * (double)hash);
  if (acc < 1) acc = 1;
  if (acc > hash) acc = hash;
  /* warm-row map, tables.hpp:210-230 */
  int64_t a = 1, b = 0;
  if (hash != 1) {
    do {
      a = 1 + (int64_t)rng_below(&m, (uint64_t)(hash - 1));
    } while (gcd64(a, hash) != 1);
    b = (int64_t)rng_below(&m, (uint64_t)hash);
  }
  zipf_t z;
  zipf_init(&z, (uint64_t)acc, zipf);
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(batch + 1));
  size_t cap = 1024, n = 0;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * cap);
  off[0] = 0;
  for (int64_t q = 0; q < batch; ++q) {
    double x = rng_lomax(&m, 3.0, 2.0 * t->pooling_mean);
    int64_t cnt = (int64_t)floor(x);
    if (rng_uniform(&m) < x - floor(x)) ++cnt;
    for (int64_t j = 0; j < cnt; ++j) {
      int64_t rank = (int64_t)zipf_draw(&z, &m) - 1;
      if (n == cap) {
        cap *= 2;
        idx = (int64_t*)realloc(idx, sizeof(int64_t) * cap);
      }
      idx[n++] = (a * rank + b) % hash;
    }
    off[q + 1] = (int64_t)n;
  }
  *offsets_out = off;
  *indices_out = idx;
  *n_out = (int64_t)n;
  return ORC_OK;
}

void orc_free(void* p) { free(p); }

/* ------------------------------------------------------------------------ */
/* fingerprints — tables.hpp:417-441                                        */
/* ------------------------------------------------------------------------ */

static uint64_t fp_table(const orc_table* t, uint64_t h) {
  h = orc_fnv1a64(&t->id, 4, h);
  h = orc_fnv1a64(&t->dim, 4, h);
  h = orc_fnv1a64(&t->hash_size, 8, h);
  h = orc_fnv1a64(&t->pooling_mean, 8, h);
  h = orc_fnv1a64(&t->access_ratio, 8, h);
  h = orc_fnv1a64(&t->bytes_per_param, 4, h);
  return h;
}

uint64_t orc_fingerprint_pool(const orc_table* t, int n) {
  uint64_t h = orc_fnv1a64("pool", 4, FNV_BASIS);
  for (int i = 0; i < n; ++i) h = fp_table(&t[i], h);
  return h;
}

uint64_t orc_fingerprint_task(const orc_table* t, int n, int k, const int64_t* budgets) {
  uint64_t h = orc_fnv1a64("task", 4, FNV_BASIS);
  h = orc_fingerprint_pool(t, n) ^ h;
  h = orc_fnv1a64(&k, 4, h);
  for (int i = 0; i < k; ++i) h = orc_fnv1a64(&budgets[i], 8, h);
  return h;
}

/* ------------------------------------------------------------------------ */
/* planners — planners.hpp:32-144                                           */
/* ------------------------------------------------------------------------ */

static int64_t tsize(const orc_table* t) { return (int64_t)t->dim * t->hash_size * t->bytes_per_param; }

static int task_check(const orc_table* t, int n, int k, const int64_t* budgets) {
  if (k < 1) return ORC_CONFIG;
  int64_t tot = 0, bud = 0;
  for (int i = 0; i < k; ++i) {
    if (budgets[i] <= 0) return ORC_CONFIG;
    bud += budgets[i];
  }
  for (int i = 0; i < n; ++i) tot += tsize(&t[i]);
  return tot > bud ? ORC_INFEASIBLE : ORC_OK;
}

static int most_free(const int64_t* f, int k) {
  int best = 0;
  for (int i = 1; i < k; ++i)
    if (f[i] > f[best]) best = i;
  return best;
}

typedef struct {
  double cost;
  int id, pos;
} gitem;

static int gcmp(const void* a, const void* b) {
  const gitem* x = (const gitem*)a;
  const gitem* y = (const gitem*)b;
  if (x->cost != y->cost) return x->cost > y->cost ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos - y->pos;
}

int orc_greedy_shard(const orc_table* t, int n, int k, const int64_t* budgets, int kind,
                     int* assignment) {
  if (kind < 0 || kind > 2) return ORC_CONFIG;
  int rc = task_check(t, n, k, budgets);
  if (rc) return rc;
  gitem* it = (gitem*)malloc(sizeof(gitem) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    double c = kind == 0 ? (double)t[i].dim * (double)t[i].hash_size
               : kind == 1 ? (double)t[i].dim
                           : (double)t[i].dim * t[i].pooling_mean;
    it[i].cost = c;
    it[i].id = t[i].id;
    it[i].pos = i;
  }
  qsort(it, (size_t)n, sizeof(gitem), gcmp);
  double* run = (double*)calloc((size_t)k, sizeof(double));
  int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  memcpy(fr, budgets, sizeof(int64_t) * (size_t)k);
  for (int q = 0; q < n; ++q) {
    int i = it[q].pos;
    int64_t sz = tsize(&t[i]);
    int ch = -1;
    for (int s = 0; s < k; ++s) {
      if (fr[s] < sz) continue;
      if (ch < 0 || run[s] < run[ch]) ch = s;
    }
    if (ch < 0) ch = most_free(fr, k);
    assignment[i] = ch;
    run[ch] += it[q].cost;
    fr[ch] -= sz;
  }
  free(it);
  free(run);
  free(fr);
  return ORC_OK;
}

int orc_random_shard(const orc_table* t, int n, int k, const int64_t* budgets, uint64_t seed,
                     int* assignment) {
  int rc = task_check(t, n, k, budgets);
  if (rc) return rc;
  mt64 m;
  mt_seed(&m, orc_derive_seed(seed, "random-shard", 0));
  int64_t* fr = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  memcpy(fr, budgets, sizeof(int64_t) * (size_t)k);
  for (int i = 0; i < n; ++i) {
    int64_t sz = tsize(&t[i]);
    int ch = -1;
    for (int a = 0; a < 16; ++a) {
      int s = (int)rng_below(&m, (uint64_t)k);
      if (fr[s] >= sz) {
        ch = s;
        break;
      }
    }
    if (ch < 0) ch = most_free(fr, k);
    assignment[i] = ch;
    fr[ch] -= sz;
  }
  free(fr);
  return ORC_OK;
}

double orc_degree_of_balance(const double* c, int n) {
  double mn = c[0], mx = c[0];
  for (int i = 1; i < n; ++i) {
    if (c[i] < mn) mn = c[i];
    if (c[i] > mx) mx = c[i];
  }
  return mx <= 0.0 ? 1.0 : mn / mx;
}

/* ------------------------------------------------------------------------ */
/* embedding-bag arithmetic (restated: PAPER.md:639,646,659; FBGEMM         */
/* exact_rowwise_adagrad). Parity unpinned against the reference.           */
/* ------------------------------------------------------------------------ */

float orc_weight_init(uint64_t seed, int32_t table_id, int64_t row, int32_t d) {
  uint64_t key = ((uint64_t)(uint32_t)table_id << 40) | ((uint64_t)row << 10) | (uint64_t)d;
  uint64_t h = orc_splitmix64(orc_splitmix64(seed) ^ key);
  int k = (int)(h >> 54) - 512;
  return (float)k * 0x1.0p-12f;
}

/* orc_weight_init with s0 = splitmix64(seed) hoisted out of the loops */
static inline float winit_s0(uint64_t s0, int32_t table_id, int64_t row, int32_t d) {
  uint64_t key = ((uint64_t)(uint32_t)table_id << 40) | ((uint64_t)row << 10) | (uint64_t)d;
  int k = (int)(orc_splitmix64(s0 ^ key) >> 54) - 512;
  return (float)k * 0x1.0p-12f;
}

float orc_grad_init(uint64_t seed, int64_t b, int64_t col) {
  uint64_t key = ((uint64_t)b << 20) | (uint64_t)col;
  uint64_t h = orc_splitmix64(orc_splitmix64(seed ^ 0x5eedf00d5eedf00dull) ^ key);
  int k = (int)(h >> 54) - 512;
  return (float)k * 0x1.0p-12f;
}

void orc_fill_weights(uint64_t seed, int32_t table_id, int64_t rows, int32_t dim, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int32_t d = 0; d < dim; ++d) out[r * dim + d] = orc_weight_init(seed, table_id, r, d);
}

/* Sum pooling in fp64 (out[b, col_t + d] = sum over the bag of
 * W_t[idx, d]; empty bag -> 0), rows [b0, b1) of the batch into out[b - b0, :].
 * OpenMP over (table, 64-bag chunk); each output element is summed in bag
 * order. W[t] = NULL uses the counter-hash init of table t (wseed). */
void orc_emb_forward_f64_rows(int T, const orc_table* tabs, int64_t B, int64_t b0, int64_t b1,
                              const int64_t* const* offsets, const int64_t* const* indices,
                              const float* const* W, uint64_t wseed, double* out) {
  int64_t sum_dim = 0;
  int64_t* col = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
  for (int t = 0; t < T; ++t) {
    col[t] = sum_dim;
    sum_dim += tabs[t].dim;
  }
  (void)B;
  const uint64_t s0 = orc_splitmix64(wseed);
  const int64_t CH = 64, nb = b1 - b0, nch = (nb + CH - 1) / CH;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t w = 0; w < (int64_t)T * nch; ++w) {
    const int t = (int)(w / nch);
    const int64_t c0 = b0 + (w % nch) * CH, c1 = c0 + CH < b1 ? c0 + CH : b1;
    const int D = tabs[t].dim;
    const float* wt = W ? W[t] : NULL;
    for (int64_t b = c0; b < c1; ++b) {
      double* o = out + (b - b0) * sum_dim + col[t];
      for (int d = 0; d < D; ++d) o[d] = 0.0;
      for (int64_t j = offsets[t][b]; j < offsets[t][b + 1]; ++j) {
        const int64_t r = indices[t][j];
        for (int d = 0; d < D; ++d)
          o[d] += wt ? (double)wt[r * D + d] : (double)winit_s0(s0, tabs[t].id, r, d);
      }
    }
  }
  free(col);
}

void orc_emb_forward_f64(int T, const orc_table* tabs, int64_t B, const int64_t* const* offsets,
                         const int64_t* const* indices, const float* const* W, uint64_t wseed,
                         double* out) {
  orc_emb_forward_f64_rows(T, tabs, B, 0, B, offsets, indices, W, wseed, out);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

int orc_emb_backward_adagrad_f64(const orc_table* t, int64_t B, const int64_t* offsets,
                                 const int64_t* indices, const float* grad, int64_t grad_stride,
                                 int64_t col0, float* W, float* M, uint64_t wseed, double lr,
                                 double eps, int64_t* n_unique, int64_t** rows_out,
                                 int64_t** counts_out, double** w_out, double** m_out) {
  const int D = t->dim;
  const int64_t L = offsets[B];
  uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(L > 0 ? L : 1));
  for (int64_t b = 0; b < B; ++b)
    for (int64_t j = offsets[b]; j < offsets[b + 1]; ++j)
      key[j] = ((uint64_t)indices[j] << 24) | (uint64_t)b; /* B < 2^24 */
  qsort(key, (size_t)L, sizeof(uint64_t), cmp_u64);
  int64_t U = 0;
  for (int64_t j = 0; j < L; ++j)
    if (j == 0 || (key[j] >> 24) != (key[j - 1] >> 24)) ++U;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U > 0 ? U : 1));
  int64_t* cnts = (int64_t*)malloc(sizeof(int64_t) * (size_t)(U > 0 ? U : 1));
  double* nw = (double*)malloc(sizeof(double) * (size_t)(U > 0 ? U * D : 1));
  double* nm = (double*)malloc(sizeof(double) * (size_t)(U > 0 ? U : 1));
  double* g = (double*)malloc(sizeof(double) * (size_t)D);
  int64_t u = -1;
  for (int64_t j = 0; j <= L; ++j) {
    int start = j < L && (j == 0 || (key[j] >> 24) != (key[j - 1] >> 24));
    if ((start || j == L) && u >= 0) {
      /* finish row u */
      int64_t r = rows[u];
      double sq = 0.0;
      for (int d = 0; d < D; ++d) sq += g[d] * g[d];
      double m0 = M ? (double)M[r] : 0.0;
      double m1 = m0 + sq / (double)D;
      double mult = lr / (sqrt(m1) + eps);
      for (int d = 0; d < D; ++d) {
        double w0 = W ? (double)W[r * D + d] : (double)orc_weight_init(wseed, t->id, r, d);
        nw[u * D + d] = w0 - mult * g[d];
        if (W) W[r * D + d] = (float)nw[u * D + d];
      }
      nm[u] = m1;
      if (M) M[r] = (float)m1;
    }
    if (j == L) break;
    if (start) {
      ++u;
      rows[u] = (int64_t)(key[j] >> 24);
      cnts[u] = 0;
      for (int d = 0; d < D; ++d) g[d] = 0.0;
    }
    int64_t b = (int64_t)(key[j] & 0xffffffull);
    cnts[u] += 1;
    const float* gr = grad + b * grad_stride + col0;
    for (int d = 0; d < D; ++d) g[d] += (double)gr[d];
  }
  free(key);
  free(g);
  *n_unique = U;
  *rows_out = rows;
  *counts_out = cnts;
  *w_out = nw;
  *m_out = nm;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* fp32 OpenMP CPU step (the timed CPU baseline; kind "port")               */
/* ------------------------------------------------------------------------ */

/* Stable LSD radix sort of 64-bit keys on bits [lo, hi), 11-bit digits. */
static void radix_sort_u64_bits(uint64_t* a, uint64_t* tmp, int64_t n, int lo, int hi) {
  const int R = 11, NB = 1 << R;
  int64_t cnt[1 << 11];
  uint64_t *src = a, *dst = tmp;
  for (int sh = lo; sh < hi; sh += R) {
    const int w = hi - sh < R ? hi - sh : R;
    const uint64_t m = ((uint64_t)1 << w) - 1;
    memset(cnt, 0, sizeof(int64_t) * (size_t)NB);
    for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> sh) & m]++;
    int64_t s = 0;
    for (int i = 0; i < NB; ++i) {
      int64_t c = cnt[i];
      cnt[i] = s;
      s += c;
    }
    for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> sh) & m]++] = src[i];
    uint64_t* x = src;
    src = dst;
    dst = x;
  }
  if (src != a) memcpy(a, src, sizeof(uint64_t) * (size_t)n);
}

/* The CPU port's step, every phase parallel over all threads:
 *  forward  — (table x 256-bag chunk) tasks, fp32 sums in bag order;
 *  backward — each table's lookups are bucketed by row range (64 buckets of
 *             the row's high bits; counting pass + stable scatter per (table,
 *             bag chunk) task), then every (table, bucket) task sorts its keys
 *             (row << 20 | bag; already in bag order, so a stable sort on the
 *             row bits alone) and runs the segment sum + exact row-wise Adagrad
 *             on its own rows (no two tasks touch the same row). */
#define ORC_NBK 64
int orc_cpu_step_f32(int T, const int32_t* dims, const int64_t* hash, int64_t B,
                     const int64_t* const* offsets, const int64_t* const* indices, float* W_all,
                     float* M_all, float* out, float lr, float eps, int n_threads) {
  int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
  int64_t* roff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
  int64_t* coff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
  int64_t* loff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T + 1));
  int* rbits = (int*)malloc(sizeof(int) * (size_t)(T > 0 ? T : 1));
  woff[0] = roff[0] = coff[0] = loff[0] = 0;
  for (int t = 0; t < T; ++t) {
    woff[t + 1] = woff[t] + hash[t] * dims[t];
    roff[t + 1] = roff[t] + hash[t];
    coff[t + 1] = coff[t] + dims[t];
    loff[t + 1] = loff[t] + offsets[t][B];
    int rb = 0;
    while ((1ll << rb) < hash[t]) ++rb;
    rbits[t] = rb;
  }
  const int64_t SD = coff[T], Ltot = loff[T];
  int used = 1;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
  }
#endif
  /* forward: out[b, coff_t:+D] = sum W_t[idx]; chunks of 256 bags */
  const int64_t CH = 256, nch = (B + CH - 1) / CH;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t w = 0; w < (int64_t)T * nch; ++w) {
    int t = (int)(w / nch);
    int64_t b0 = (w % nch) * CH, b1 = b0 + CH < B ? b0 + CH : B;
    const int D = dims[t];
    const float* Wt = W_all + woff[t];
    for (int64_t b = b0; b < b1; ++b) {
      float* o = out + b * SD + coff[t];
      for (int d = 0; d < D; ++d) o[d] = 0.f;
      for (int64_t j = offsets[t][b]; j < offsets[t][b + 1]; ++j) {
        const float* r = Wt + indices[t][j] * D;
        for (int d = 0; d < D; ++d) o[d] += r[d];
      }
    }
  }
  /* backward (grad = out): bucket by row range, sort, segment sum, Adagrad */
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(Ltot > 0 ? Ltot : 1));
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(Ltot > 0 ? Ltot : 1));
  int64_t* cnt = (int64_t*)calloc((size_t)T * (size_t)nch * ORC_NBK, sizeof(int64_t));
  int64_t* bstart = (int64_t*)malloc(sizeof(int64_t) * ((size_t)T * ORC_NBK + 1));
#define BSHIFT(t) (rbits[t] > 6 ? rbits[t] - 6 : 0)
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t w = 0; w < (int64_t)T * nch; ++w) { /* count */
    int t = (int)(w / nch);
    int64_t b0 = (w % nch) * CH, b1 = b0 + CH < B ? b0 + CH : B;
    int64_t* c = cnt + w * ORC_NBK;
    const int sh = BSHIFT(t);
    for (int64_t j = offsets[t][b0]; j < offsets[t][b1]; ++j) c[indices[t][j] >> sh]++;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < T; ++t) { /* exclusive offsets: bucket-major, then bag chunk */
    int64_t s = loff[t];
    for (int k = 0; k < ORC_NBK; ++k) {
      bstart[(int64_t)t * ORC_NBK + k] = s;
      for (int64_t c = 0; c < nch; ++c) {
        int64_t* x = cnt + ((int64_t)t * nch + c) * ORC_NBK + k;
        int64_t v = *x;
        *x = s;
        s += v;
      }
    }
  }
  bstart[(int64_t)T * ORC_NBK] = Ltot;
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t w = 0; w < (int64_t)T * nch; ++w) { /* stable scatter */
    int t = (int)(w / nch);
    int64_t b0 = (w % nch) * CH, b1 = b0 + CH < B ? b0 + CH : B;
    int64_t* c = cnt + w * ORC_NBK;
    const int sh = BSHIFT(t);
    for (int64_t b = b0; b < b1; ++b)
      for (int64_t j = offsets[t][b]; j < offsets[t][b + 1]; ++j) {
        const uint64_t r = (uint64_t)indices[t][j];
        keys[c[r >> sh]++] = (r << 20) | (uint64_t)b;
      }
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t w = 0; w < (int64_t)T * ORC_NBK; ++w) { /* sort + reduce + Adagrad */
    int t = (int)(w / ORC_NBK);
    const int64_t a0 = bstart[w], a1 = bstart[w + 1];
    if (a1 <= a0) continue;
    const int D = dims[t];
    uint64_t* k = keys + a0;
    const int64_t n = a1 - a0;
    radix_sort_u64_bits(k, tmp + a0, n, 20, 20 + BSHIFT(t));
    float g[1024];
    float* Wt = W_all + woff[t];
    float* Mt = M_all + roff[t];
    int64_t j = 0;
    while (j < n) {
      uint64_t r = k[j] >> 20;
      for (int d = 0; d < D; ++d) g[d] = 0.f;
      while (j < n && (k[j] >> 20) == r) {
        const float* gr = out + (int64_t)(k[j] & 0xfffff) * SD + coff[t];
        for (int d = 0; d < D; ++d) g[d] += gr[d];
        ++j;
      }
      float sq = 0.f;
      for (int d = 0; d < D; ++d) sq += g[d] * g[d];
      float m1 = Mt[r] + sq / (float)D;
      Mt[r] = m1;
      float mult = lr / (sqrtf(m1) + eps);
      float* wr = Wt + r * D;
      for (int d = 0; d < D; ++d) wr[d] -= mult * g[d];
    }
  }
#undef BSHIFT
  free(keys);
  free(tmp);
  free(cnt);
  free(bstart);
  free(loff);
  free(rbits);
  free(woff);
  free(roff);
  free(coff);
  return used;
}
