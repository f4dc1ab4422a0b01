// Device context of one shard on one B200: allocation, counter-hash init,
// stream loading with on-device validation, forward, backward (sort + segment
// reduce + row-wise Adagrad) and the micro-benchmark protocol.
//
// HBM layout (per context):
//   W      fp32, tables concatenated in context order, each [hash_t, dim_t] row-major
//   M      fp32 [sum hash_t]  row-wise Adagrad momentum, indexed by GLOBAL row
//   idx32  int32 [L]  lookups as table-local rows, table-major
//   off32  int32 [T*B + 1] rebased bag offsets (TBE layout)
//   bag    int32 [L]  bag id of each lookup (K4)
//   skey/sbag int32 [L] each table's lookups sorted by row (stable), with bag ids
//   pooled fp32 [B, sum dim_t], table columns in context order
#include "context.hpp"
#include "kernels.cuh"

#include "sort.cuh"

#include <algorithm>
#include <array>
#include <cmath>
#include <mutex>

#include <immintrin.h>

#include "../host/threadpool.hpp"
#include <cstdlib>
#include <cstring>

namespace asb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    fail(AS_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != d) cuda_check(cudaSetDevice(d), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

// Lane layout of a table: NV = vec float4 per lane when the row is wide enough
// for >= 8 lanes (one warp instruction then gathers 32/GL rows), else 1.
int kind_for_dim(int dim, int vec, bool half) {
  const int nvec = dim / 4;
  auto pow2ceil = [](int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
  };
  // fp16 tables: PAIRED layouts, one 16-B load (8 halves) per lane and slot pair
  if (half && dim % 8 == 0 && dim >= 64) {
    const int n8 = dim / 8;
    if (n8 <= 32) {
      const int gl = pow2ceil(n8);
      for (int k = 0; k < kNumKinds; ++k)
        if (kind_gl(k) == gl && kind_nv(k) == 2) return k;
    }
    if (n8 <= 64) return 7;
    return 8;
  }
  if (vec >= 2 && nvec >= 16 && nvec <= 32 * vec) {
    const int nv = (vec >= 4 && nvec >= 32) ? 4 : 2;
    const int gl = std::min(32, pow2ceil((nvec + nv - 1) / nv));
    for (int k = 0; k < kNumKinds; ++k)
      if (kind_gl(k) == gl && kind_nv(k) == nv) return k;
  }
  if (nvec <= 32) {
    const int gl = pow2ceil(std::max(1, nvec));
    for (int k = 0; k <= 5; ++k)
      if (kind_gl(k) == gl) return k;
  }
  if (nvec <= 64) return 6;
  if (nvec <= 128) return 7;
  return 8;
}

// Elements per chunk: ~target bytes of gathered rows per group, multiple of 32.
int chunk_len_for(int dim, double target_bytes) {
  int c = static_cast<int>(target_bytes / (dim * 4.0));
  c = (c / 32) * 32;
  return std::max(32, std::min(8192, c));
}

int bit_width_u64(uint64_t x) {
  int b = 0;
  while (x) {
    ++b;
    x >>= 1;
  }
  return b;
}

__global__ void gather_rows_kernel(const void* __restrict__ src, int half, long long w_off, int dim,
                                   const long long* __restrict__ rows, long long n,
                                   float* __restrict__ dst) {
  const long long total = n * dim;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long i = q / dim;
    const int d = (int)(q - i * dim);
    const long long e = w_off + rows[i] * dim + d;
    dst[q] = half ? __half2float(reinterpret_cast<const __half*>(src)[e]) : reinterpret_cast<const float*>(src)[e];
  }
}

// Device side of the staging split: int64 lookups copied raw
// are narrowed to int32 rows on the GPU and validated against [0, hash) with
// load_workload's check (workload_io.hpp:216-241); the first bad entry wins
// through the same (table, check, entry) key the host validation uses.
__global__ void narrow_validate_kernel(const long long* __restrict__ src, int* __restrict__ dst, long long n,
                                       long long hash, unsigned long long key_base,
                                       unsigned long long* __restrict__ err) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long v = src[j];
    dst[j] = (int)v;
    if ((unsigned long long)v >= (unsigned long long)hash) atomicMin(err, key_base | (unsigned long long)j);
  }
}

constexpr int kBlock = 256;
constexpr int kWarpsPerBlock = kBlock / 32;

unsigned grid_for(long long work, long long per_block) {
  long long g = (work + per_block - 1) / per_block;
  return (unsigned)std::max(1LL, g);
}

}  // namespace

cudaEvent_t EmbContext::ev_get() {
  if (ev_pool_.empty()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "event");
    return e;
  }
  cudaEvent_t e = ev_pool_.back();
  ev_pool_.pop_back();
  return e;
}

// Records a CUDA event pair around one phase when profiling is on.
struct EmbContext::Phase {
  EmbContext* c;
  int id;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  Phase(EmbContext* ctx, int phase, cudaStream_t st) : c(ctx), id(phase), s(st) {
    if (c->prof_) {
      a = c->ev_get();
      cuda_check(cudaEventRecord(a, s), "event");
    }
  }
  ~Phase() {
    if (a) {
      cudaEvent_t b = c->ev_get();
      cudaEventRecord(b, s);
      c->ev_used_.push_back({id, {a, b}});
    }
  }
};

void EmbContext::profile_enable(int mode) {
  prof_ = mode != 0;
  prof_serial_ = mode == 2;
}

void EmbContext::profile_read(double* ms, int64_t* launches, bool reset) {
  DeviceGuard g(device_);
  for (int i = 0; i < kPhases; ++i) ms[i] = 0.0;
  for (auto& u : ev_used_) {
    cuda_check(cudaEventSynchronize(u.second.second), "event sync");
    float x = 0.f;
    cuda_check(cudaEventElapsedTime(&x, u.second.first, u.second.second), "elapsed");
    ms[u.first] += x;
  }
  if (launches) *launches = launches_;
  if (reset) {
    for (auto& u : ev_used_) {
      ev_pool_.push_back(u.second.first);
      ev_pool_.push_back(u.second.second);
    }
    ev_used_.clear();
    launches_ = 0;
  }
}

void* EmbContext::dalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  bytes_ += static_cast<int64_t>(bytes);
  allocs_.push_back(p);
  return p;
}

// Per-table layout shared by both constructors: validation, lane layout,
// pooled columns, staging sizes (the storage offsets w_base / row_off are set
// by the caller).
void EmbContext::layout_tables() {
  const int n = T_;
  if ((int64_t)n * B_ >= (1LL << 31))
    fail(AS_SHAPE, "as_create: n_tables x batch_size = " + std::to_string((int64_t)n * B_) +
                       " bags; a shard takes at most 2^31-1 (int32 bag offsets)");
  htabs_.assign(static_cast<size_t>(n), DevTable{});
  for (int t = 0; t < n; ++t) {
    const as_table_spec& s = specs_[t];
    if (s.dim < 4 || s.dim > 1024 || s.dim % 4 != 0)
      fail(AS_CONFIG, "table " + std::to_string(s.id) + ": device path needs dim % 4 == 0 and 4 <= dim <= 1024, got " +
                          std::to_string(s.dim));
    if (s.hash_size < 1) fail(AS_CONFIG, "table " + std::to_string(s.id) + " has invalid hash_size");
    if (s.hash_size >= (1LL << 31))
      fail(AS_SHAPE, "table " + std::to_string(s.id) + ": at most 2^31-1 rows (int32 row ids), got " +
                         std::to_string(s.hash_size));
    DevTable& d = htabs_[t];
    std::memset(&d, 0, sizeof d);
    d.sort_bits = std::max(1, bit_width_u64(static_cast<uint64_t>(s.hash_size - 1)));
#ifdef ASB_NO_PACKED_SORT
    d.sort_packed = 0;
#else
    d.sort_packed = sort_passes_of(d.sort_bits) >= 2 && d.sort_bits + bag_bits() <= 32 ? 1 : 0;
#endif
    d.hash = s.hash_size;
    d.dim = s.dim;
    d.col = static_cast<int>(sum_dim_);
    d.table_id = s.id;
    d.kind = kind_for_dim(s.dim, std::find(vec2_dims_.begin(), vec2_dims_.end(), s.dim) != vec2_dims_.end() ? 2 : vec_,
                          w_half_);
    d.chunk_len = chunk_len_for(s.dim, 131072.0);
    sum_dim_ += s.dim;
    max_dim_ = std::max(max_dim_, s.dim);
    stage_x_ = std::max(stage_x_, stage_x_ints(d.kind));
    stage_s_ = std::max(stage_s_, stage_s_ints(d.kind));
  }
  stage_s_ = (stage_s_ + 3) & ~3;  // 16-B aligned id buffers (vector LDS of row ids)
  seg_smem_bytes_ = static_cast<size_t>(kSegWarps) * 2 * (stage_x_ + stage_s_) * sizeof(int);
}

static void check_device(int device) {
  int ndev = 0;
  cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    fail(AS_CONFIG, "as_create: device " + std::to_string(device) + " out of range (" + std::to_string(ndev) +
                        " visible)");
}

EmbContext::EmbContext(int device, const as_table_spec* tables, int n, int64_t batch, uint64_t seed, int flags)
    : device_(device), T_(n), B_(batch), seed_(seed), w_half_((flags & AS_WEIGHTS_FP16) != 0) {
  if (flags & ~AS_WEIGHTS_FP16) fail(AS_CONFIG, "as_create_ex: unknown flags " + std::to_string(flags));
  if (n < 0) fail(AS_CONFIG, "as_create: n_tables must be >= 0");
  if (batch < 1 || batch > (1LL << 30)) fail(AS_CONFIG, "as_create: batch_size must be in [1, 2^30]");
  check_device(device);
  if (const char* e = std::getenv("ASB_VEC")) vec_ = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("ASB_VEC2_DIMS")) {  // A/B: dims laid out with 2 float4 per lane
    vec2_dims_.clear();
    for (const char* c = e; *c;) {
      vec2_dims_.push_back(std::atoi(c));
      while (*c && *c != ',') ++c;
      if (*c) ++c;
    }
  }
  if (const char* e = std::getenv("ASB_CHUNK_KB")) chunk_cap_ = std::max(2.0, std::atof(e)) * 1024.0;
  if (const char* e = std::getenv("ASB_UNIT_KB")) unit_cap_ = std::max(2.0, std::atof(e)) * 1024.0;
  specs_.assign(tables, tables + n);
  layout_tables();
  for (int t = 0; t < n; ++t) {
    htabs_[t].row_off = total_rows_;
    htabs_[t].w_base = total_w_;
    total_rows_ += specs_[t].hash_size;
    // every table starts 128-B aligned (fp32; 64 B for fp16): 16-B vector rows,
    // and the paired fp16 layouts' 16-B loads, never straddle a table start
    total_w_ += (specs_[t].hash_size * specs_[t].dim + 31) / 32 * 32;
  }
  DeviceGuard g(device_);
  W_ = static_cast<float*>(dalloc((w_half_ ? 2 : 4) * static_cast<size_t>(total_w_)));
  M_ = static_cast<float*>(dalloc(sizeof(float) * static_cast<size_t>(total_rows_)));
  setup_runtime();

  // K6: weights from the counter hash, momentum zero.
  const unsigned long long s0 = splitmix64(seed_);
  for (int t = 0; t < n; ++t) {
    const int64_t off = htabs_[t].w_base;
    const long long nv = specs_[t].hash_size * (specs_[t].dim / 4);
    const unsigned grid = static_cast<unsigned>(std::min<long long>((nv + 255) / 256, 148LL * 64));
    if (w_half_)
      init_table_kernel<true><<<grid, 256>>>(reinterpret_cast<__half*>(W_) + off, specs_[t].hash_size, specs_[t].dim,
                                             specs_[t].id, s0);
    else
      init_table_kernel<false><<<grid, 256>>>(W_ + off, specs_[t].hash_size, specs_[t].dim, specs_[t].id, s0);
  }
  cuda_check(cudaGetLastError(), "init_table_kernel");
  cuda_check(cudaMemset(M_, 0, sizeof(float) * static_cast<size_t>(total_rows_)), "momentum init");
  cuda_check(cudaMemcpy(dtabs_, htabs_.data(), sizeof(DevTable) * n, cudaMemcpyHostToDevice), "tables H2D");
  cuda_check(cudaDeviceSynchronize(), "init");
}


// A shard over a subset of `parent`'s tables that uses the parent's weight and
// momentum storage (no copy, no init): steps through it update the parent's
// rows. The parent must outlive it.
EmbContext::EmbContext(const EmbContext& parent, const int* positions, int n)
    : device_(parent.device_), T_(n), B_(parent.B_), seed_(parent.seed_), w_half_(parent.w_half_) {
  if (n < 0) fail(AS_CONFIG, "as_create_subset: n_tables must be >= 0");
  vec_ = parent.vec_;
  vec2_dims_ = parent.vec2_dims_;
  chunk_cap_ = parent.chunk_cap_;
  unit_cap_ = parent.unit_cap_;
  specs_.resize(static_cast<size_t>(n));
  std::vector<char> seen(static_cast<size_t>(parent.T_), 0);
  for (int i = 0; i < n; ++i) {
    const int q = positions[i];
    if (q < 0 || q >= parent.T_)
      fail(AS_CONFIG, "as_create_subset: position " + std::to_string(q) + " out of range [0, " +
                          std::to_string(parent.T_) + ")");
    if (seen[q]++) fail(AS_CONFIG, "as_create_subset: table position " + std::to_string(q) + " given twice");
    specs_[i] = parent.specs_[q];
  }
  layout_tables();
  for (int i = 0; i < n; ++i) {
    htabs_[i].row_off = parent.htabs_[positions[i]].row_off;
    htabs_[i].w_base = parent.htabs_[positions[i]].w_base;
  }
  total_rows_ = parent.total_rows_;
  total_w_ = parent.total_w_;
  DeviceGuard g(device_);
  W_ = parent.W_;
  M_ = parent.M_;
  parent_ = &parent;
  setup_runtime();
  cuda_check(cudaMemcpy(dtabs_, htabs_.data(), sizeof(DevTable) * std::max(1, n), cudaMemcpyHostToDevice),
             "tables H2D");
}

// Point a subset context at another subset of its parent's tables, keeping
// its streams, events and (grow-only) buffers: the measured-cost hook times
// thousands of candidate shards with one context.
void EmbContext::retarget(const int* positions, int n) {
  if (!parent_) fail(AS_STATE, "as_retarget_subset: not a subset context (as_create_subset)");
  if (n < 0) fail(AS_CONFIG, "as_retarget_subset: n_tables must be >= 0");
  for (const Slot& sl : slots_)
    if (sl.staged) fail(AS_STATE, "as_retarget_subset: a staged batch is pending (commit it first)");
  if (peers_.n) fail(AS_STATE, "as_retarget_subset: the forward writes to peer buffers");
  const EmbContext& parent = *parent_;
  DeviceGuard g(device_);
  cuda_check(cudaDeviceSynchronize(), "retarget sync");
  std::vector<as_table_spec> specs(static_cast<size_t>(n));
  std::vector<char> seen(static_cast<size_t>(parent.T_), 0);
  for (int i = 0; i < n; ++i) {
    const int q = positions[i];
    if (q < 0 || q >= parent.T_)
      fail(AS_CONFIG, "as_retarget_subset: position " + std::to_string(q) + " out of range [0, " +
                          std::to_string(parent.T_) + ")");
    if (seen[q]++) fail(AS_CONFIG, "as_retarget_subset: table position " + std::to_string(q) + " given twice");
    specs[i] = parent.specs_[q];
  }
  const int old_T = T_;
  const int64_t old_out = B_ * sum_dim_;
  const int old_max_dim = max_dim_;
  specs_ = std::move(specs);
  T_ = n;
  sum_dim_ = 0;
  max_dim_ = 4;
  stage_x_ = 32;
  stage_s_ = 33;
  layout_tables();
  for (int i = 0; i < n; ++i) {
    htabs_[i].row_off = parent.htabs_[positions[i]].row_off;
    htabs_[i].w_base = parent.htabs_[positions[i]].w_base;
  }
  auto drop = [this](void* p) {
    auto it = std::find(allocs_.begin(), allocs_.end(), p);
    if (it != allocs_.end()) allocs_.erase(it);
    cudaFree(p);
  };
  if (n > cap_tables_) {
    drop(dtabs_);
    dtabs_ = static_cast<DevTable*>(dalloc(sizeof(DevTable) * std::max(1, n)));
    for (Slot& sl : slots_) {
      drop(sl.d_off32);
      cudaFreeHost(sl.h_off32);
      sl.d_off32 = static_cast<int*>(dalloc(sizeof(int) * static_cast<size_t>(T_ * B_ + 1)));
      cuda_check(cudaHostAlloc(&sl.h_off32, sizeof(int) * static_cast<size_t>(T_ * B_ + 1), cudaHostAllocDefault),
                 "pinned staging");
    }
    cap_tables_ = n;
  }
  if (B_ * sum_dim_ > std::max(old_out, cap_out_)) {
    drop(out_);
    out_ = static_cast<float*>(dalloc(sizeof(float) * static_cast<size_t>(B_ * sum_dim_)));
    cap_out_ = B_ * sum_dim_;
  }
  if (max_dim_ > old_max_dim) cap_chunks_ = 0;  // carries are [chunks][2][max dim]: regrow at the next commit
  (void)old_T;
  if (n > 0)
    cuda_check(cudaMemcpy(dtabs_, htabs_.data(), sizeof(DevTable) * n, cudaMemcpyHostToDevice), "tables H2D");
  loaded_ = false;
  sort_pending_ = false;
  bag_valid_ = false;
}

// Buffers, streams and events of a context (both constructors).
void EmbContext::setup_runtime() {
  const int n = T_;
  cap_tables_ = n;
  cap_out_ = B_ * sum_dim_;
  dtabs_ = static_cast<DevTable*>(dalloc(sizeof(DevTable) * std::max(1, n)));
  out_ = static_cast<float*>(dalloc(sizeof(float) * static_cast<size_t>(B_ * sum_dim_)));
  for (Slot& sl : slots_) {
    sl.d_off32 = static_cast<int*>(dalloc(sizeof(int) * static_cast<size_t>(T_ * B_ + 1)));
    cuda_check(cudaHostAlloc(&sl.h_off32, sizeof(int) * static_cast<size_t>(T_ * B_ + 1), cudaHostAllocDefault),
               "pinned staging");
    cuda_check(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&sl.retired, cudaEventDisableTiming), "event");
    sl.d_err = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long)));
    cuda_check(cudaHostAlloc(&sl.h_err, sizeof(unsigned long long), cudaHostAllocDefault), "pinned error key");
  }
  if (const char* e = std::getenv("ASB_RAW_EIGHTHS")) raw_eighths_ = std::max(0, std::min(8, std::atoi(e)));
  cuda_check(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking), "copy stream");
  {
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
    // GPU narrowing of staged pieces: highest priority, so its small CTAs take
    // the first free SM slots inside a running step instead of queueing behind it
    cuda_check(cudaStreamCreateWithPriority(&narrow_, cudaStreamNonBlocking, hi), "narrow stream");
  }
  err_ = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long)));
  loss_ = static_cast<double*>(dalloc(sizeof(double)));
  cuda_check(cudaHostAlloc(&h_loss_, sizeof(double), cudaHostAllocDefault), "pinned loss");
  counters_ = static_cast<int*>(dalloc(sizeof(int) * 6));
  int sms = 148;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "SM count");
  fixup_grid_ = static_cast<unsigned>(sms * 2);
  fixup_short_grid_ = static_cast<unsigned>(sms * 16);
  fixup_lane_grid_ = static_cast<unsigned>(sms * 4);
  int l2 = 0;
  cuda_check(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device_), "L2 size");
  flush_bytes_ = static_cast<size_t>(std::max(l2, 1 << 20)) * 2;
  flush_ = dalloc(flush_bytes_);

  // Index staging is small: carve out just enough shared memory for the
  // resident CTAs and leave the rest of the unified 228 KB to L1 (hot rows).
  // The carveout is a per-function, process-wide attribute: every launch
  // re-applies its context's (set_carveout), so contexts with other lane
  // layouts in the same process — subset contexts retargeted to other
  // shards — never run on a too-small carveout (fewer resident CTAs).
  {
    // index staging of 1-lane groups can pass the 48 KB default (any subset's kinds)
    int max_stage = 0;
    for (int k = 0; k < kNumKinds; ++k) max_stage = std::max(max_stage, stage_x_ints(k) + ((stage_s_ints(k) + 3) & ~3));
    const int max_dyn = static_cast<int>(kSegWarps * 2 * max_stage * sizeof(int));
    cuda_check(cudaFuncSetAttribute(seg_reduce_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn),
               "seg smem");
    cuda_check(cudaFuncSetAttribute(seg_reduce_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn),
               "seg smem");
  }
  {
    // the side stream runs K2 beside the forward gather; ASB_SIDE_PRIO (A/B):
    // -1 = greatest priority (the sort's CTAs are scheduled first), 1 = least
    int lo = 0, hi = 0, prio = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
    if (const char* e = std::getenv("ASB_SIDE_PRIO")) {
      const int v = std::atoi(e);
      prio = v < 0 ? hi : (v > 0 ? lo : 0);
    }
    cuda_check(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, prio), "side stream");
  }
  cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_k4_, cudaEventDisableTiming), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_done_, cudaEventDisableTiming | cudaEventBlockingSync), "event");

}

EmbContext::~EmbContext() {
  // a staged job may still be narrowing into / copying from the slot buffers
  for (Slot& sl : slots_)
    if (sl.job.joinable()) sl.job.join();
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  cudaDeviceSynchronize();
  for (void* p : allocs_) cudaFree(p);
  for (auto& u : ev_used_) {
    cudaEventDestroy(u.second.first);
    cudaEventDestroy(u.second.second);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  if (copy_) cudaStreamDestroy(copy_);
  if (narrow_) cudaStreamDestroy(narrow_);
  for (Slot& sl : slots_) {
    if (sl.job.joinable()) sl.job.join();
    if (sl.copied) cudaEventDestroy(sl.copied);
    if (sl.retired) cudaEventDestroy(sl.retired);
    if (sl.h_idx32) cudaFreeHost(sl.h_idx32);
    if (sl.h_off32) cudaFreeHost(sl.h_off32);
    if (sl.h_err) cudaFreeHost(sl.h_err);
    for (auto e : sl.raw_ev) cudaEventDestroy(e);
    if (sl.narrowed) cudaEventDestroy(sl.narrowed);
  }
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (ev_k4_) cudaEventDestroy(ev_k4_);
  if (ev_done_) cudaEventDestroy(ev_done_);
  if (h_loss_) cudaFreeHost(h_loss_);
  if (prev >= 0) cudaSetDevice(prev);
}

void EmbContext::ensure_capacity(int64_t L, int64_t n_chunks, int64_t n_units) {
  auto drop = [this](void* p) {
    if (!p) return;
    auto it = std::find(allocs_.begin(), allocs_.end(), p);
    if (it != allocs_.end()) allocs_.erase(it);
    cudaFree(p);
  };
  if (L > cap_L_) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    for (void* p : {(void*)bag_, (void*)skey_, (void*)sbag_, (void*)tkey_, (void*)tbag_}) drop(p);
    const int64_t cap = std::max<int64_t>(L + L / 8, 1024);
    bag_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    skey_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    sbag_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    tkey_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    tbag_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    cap_L_ = cap;
  }
  // K2 scratch: [superblocks][256] digit counts / output positions of the running pass
  const int64_t sbs = (L + kSortTile - 1) / kSortTile + T_;  // the smallest superblocks (1 tile)
  if (sbs > cap_sort_tiles_) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    drop(sort_scratch_);
    const int64_t cap = sbs + sbs / 8 + 16;
    sort_scratch_ = static_cast<int*>(dalloc(sizeof(int) * cap * kSortDigits));
    cap_sort_tiles_ = cap;
  }
  if (n_chunks > cap_chunks_) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    drop(carry_);
    drop(completers_);
    drop(completers_long_);
    drop(completers_mid_);
    const int64_t cap = std::max<int64_t>(n_chunks + n_chunks / 8, 64);
    carry_ = static_cast<float*>(dalloc(sizeof(float) * cap * 2 * max_dim_));
    completers_ = static_cast<int2*>(dalloc(sizeof(int2) * cap));
    completers_long_ = static_cast<int4*>(dalloc(sizeof(int4) * cap));
    completers_mid_ = static_cast<int2*>(dalloc(sizeof(int2) * cap));
    cap_chunks_ = cap;
  }
  if (n_units > cap_units_) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    drop(unit_table_);
    const int64_t cap = std::max<int64_t>(n_units + n_units / 8, 64);
    unit_table_ = static_cast<int*>(dalloc(sizeof(int) * cap));
    cap_units_ = cap;
  }
}

// ---- batch loading -----------------------------------------------------------
// stage(): lay the batch out on the host, then a background job narrows the
//   caller's int64 CSR to the device format (int32 GLOBAL rows, rebased int32
//   offsets) into a pinned slot buffer on the staging thread pool, validating
//   with load_workload's checks (workload_io.hpp:216-241), and enqueues each
//   finished piece's H2D on the copy stream right away (narrowing and PCIe
//   overlap; the copy is half the bytes of the int64 source).
// commit(): joins the job (raising the batch's first OffsetError /
//   IndexError, in the reference's table/check/entry order) and swaps the
//   slot's device arrays in as the current batch; the compute stream waits on
//   the slot's copy event. Two slots: batch i+1 stages while batch i computes.
namespace {
constexpr int64_t kNarrowChunk = 1 << 19;

// dst[j] = row0 + src[j]; returns true if any src[j] is outside [0, hash).
// The AVX-512 path uses streaming (non-temporal) stores into the pinned
// staging buffer: host memory bandwidth bounds this loop, and streaming
// stores skip the read-for-ownership of the destination lines.
__attribute__((target("avx512f"))) bool narrow_rows_avx512(const int64_t* __restrict__ src, int* __restrict__ dst,
                                                           int64_t n, int64_t hash, int row0) {
  int64_t j = 0;
  int64_t bad = 0;
  while (j < n && (reinterpret_cast<uintptr_t>(dst + j) & 31)) {
    bad |= (int64_t)((uint64_t)src[j] >= (uint64_t)hash);
    dst[j] = row0 + (int)src[j];
    ++j;
  }
  const __m512i vh = _mm512_set1_epi64(hash);
  const __m256i vr = _mm256_set1_epi32(row0);
  __mmask8 m = 0;
  for (; j + 8 <= n; j += 8) {
    const __m512i v = _mm512_loadu_si512(src + j);
    m |= _mm512_cmpge_epu64_mask(v, vh);
    const __m256i w = _mm256_add_epi32(_mm512_cvtepi64_epi32(v), vr);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + j), w);
  }
  for (; j < n; ++j) {
    bad |= (int64_t)((uint64_t)src[j] >= (uint64_t)hash);
    dst[j] = row0 + (int)src[j];
  }
  _mm_sfence();
  return bad != 0 || m != 0;
}

bool narrow_rows_scalar(const int64_t* __restrict__ src, int* __restrict__ dst, int64_t n, int64_t hash, int row0) {
  int64_t bad = 0;
  for (int64_t j = 0; j < n; ++j) {
    const int64_t v = src[j];
    bad |= (int64_t)((uint64_t)v >= (uint64_t)hash);
    dst[j] = row0 + (int)v;
  }
  return bad != 0;
}

bool narrow_rows(const int64_t* src, int* dst, int64_t n, int64_t hash, int row0) {
  static const bool avx512 = __builtin_cpu_supports("avx512f");
  return avx512 ? narrow_rows_avx512(src, dst, n, hash, row0) : narrow_rows_scalar(src, dst, n, hash, row0);
}
}

void EmbContext::stage(const int64_t* const* offsets, const int64_t* const* indices, const int64_t* n_idx) {
  DeviceGuard g(device_);
  Slot& sl = stage_layout(n_idx);
  stage_fill_host(sl, offsets, indices, n_idx);
}

// Lay a batch with n_idx[t] lookups per table out in a free slot (chunks,
// warp units, sort superblocks, grown buffers) and mark it staged; the data
// itself comes from stage_fill_host (the caller's int64 CSR) or
// stage_device (device-resident int32 arrays, e.g. after the KJT exchange).
EmbContext::Slot& EmbContext::stage_layout(const int64_t* n_idx) {
  int pick = -1;
  for (int k = 0; k < 2 && pick < 0; ++k)
    if (!slots_[k].staged && k != cur_slot_) pick = k;
  if (pick < 0)
    fail(AS_STATE, "as_stage_streams: no free staging slot (one batch may be staged ahead of the current one; "
                   "commit it first)");
  Slot& sl = slots_[pick];
  // Chunk length: ~256 KB of gathered rows per group, shrunk for small
  // batches so that there is at least about one wave of warps.
  double gbytes = 0.0;
  for (int t = 0; t < T_; ++t) gbytes += 4.0 * specs_[t].dim * (double)std::max<int64_t>(n_idx[t], 0);
  const double target = std::max(2048.0, std::min(chunk_cap_, gbytes / (148.0 * 24.0)));
  sl.tabs = htabs_;
  int64_t L = 0, nch = 0, nun = 0;
  std::vector<int64_t> units_of(static_cast<size_t>(T_));
  for (int t = 0; t < T_; ++t) {
    if (n_idx[t] < 0) fail(AS_OFFSET, "table " + std::to_string(specs_[t].id) + ": negative index count");
    DevTable& d = sl.tabs[t];
    const int R = 32 / kind_gl(d.kind);
    // a warp unit walks R chunks: cap the unit's bytes, not only the chunk's, so
    // narrow-row tables do not widen the in-flight window (L2 reuse of the
    // gathered gradient slabs in the backward)
    d.chunk_len = chunk_len_for(specs_[t].dim, std::min(target, unit_cap_ / R));
    const int64_t chunks = (n_idx[t] + d.chunk_len - 1) / d.chunk_len;
    const int64_t units = (chunks + R - 1) / R;
    units_of[t] = units;
    d.idx_off = L;
    d.n_lookups = n_idx[t];
    d.chunk_off = static_cast<int>(nch);
    d.n_units = static_cast<int>(units);
    L += n_idx[t];
    nch += units * R;
  }
  // warp units in table order
  for (int t = 0; t < T_; ++t) {
    sl.tabs[t].unit_off = static_cast<int>(nun);
    nun += units_of[t];
  }
  if (L >= (1LL << 31)) fail(AS_SHAPE, "as_load_streams: a shard takes at most 2^31-1 lookups per batch");
  if (nch >= (1LL << 31)) fail(AS_SHAPE, "as_load_streams: too many chunks");
  sl.L = L;
  sl.nch = nch;
  sl.nun = nun;
  // K2 layout: superblocks per table; meta = [superblock -> table] then, per
  // digit pass, the superblocks of the tables that still have digits left
  {
    // superblock = 1..16 tiles: about 6 waves of 3 CTAs per SM (5 are resident;
    // sized as measured in profiles/r2_ab/r2q, r2r)
    const int64_t want = 148LL * 3 * 6;
    int sbt = 1;
    while (sbt < kSortMaxSBTiles && L / ((int64_t)kSortTile * sbt * 2) >= want) sbt *= 2;
    sl.sort_sb_elems = kSortTile * sbt;
    const int64_t sbe = sl.sort_sb_elems;
    int64_t sbs = 0;
    int pmax = 0;
    std::vector<int64_t> sb_of(static_cast<size_t>(T_));
    for (int t = 0; t < T_; ++t) {
      if (n_idx[t] >= (1LL << 30))
        fail(AS_SHAPE, "table " + std::to_string(specs_[t].id) + ": at most 2^30-1 lookups per batch");
      sb_of[t] = (n_idx[t] + sbe - 1) / sbe;
      sl.tabs[t].sort_tile_off = static_cast<int>(sbs);
      sbs += sb_of[t];
      if (n_idx[t] > 0) pmax = std::max(pmax, sort_passes_of(sl.tabs[t].sort_bits));
    }
    std::vector<int>& m = sl.sort_meta;
    m.clear();
    m.reserve(static_cast<size_t>((1 + pmax) * sbs));
    for (int t = 0; t < T_; ++t) m.insert(m.end(), static_cast<size_t>(sb_of[t]), t);
    for (int p = 0; p < kMaxSortPasses; ++p) {
      sl.tile_tab_off[p] = static_cast<int64_t>(m.size());
      int64_t acc = 0;
      if (p < pmax)
        for (int t = 0; t < T_; ++t)
          if (n_idx[t] > 0 && sort_passes_of(sl.tabs[t].sort_bits) > p) {
            for (int64_t k = 0; k < sb_of[t]; ++k) m.push_back(static_cast<int>(sl.tabs[t].sort_tile_off + k));
            acc += sb_of[t];
          }
      sl.pass_tiles[p] = acc;
    }
    sl.n_sort_tiles = sbs;
    sl.sort_passes = pmax;
  }
  sl.utab.assign(static_cast<size_t>(nun), 0);
  for (int t = 0; t < T_; ++t)
    std::fill(sl.utab.begin() + sl.tabs[t].unit_off, sl.utab.begin() + sl.tabs[t].unit_off + sl.tabs[t].n_units, t);
  if (L > sl.cap) {
    // the slot's previous batch may still be in use on the device
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    auto drop = [this](void* p) {
      auto it = std::find(allocs_.begin(), allocs_.end(), p);
      if (it != allocs_.end()) allocs_.erase(it);
      cudaFree(p);
    };
    if (sl.d_idx32) drop(sl.d_idx32);
    if (sl.h_idx32) cudaFreeHost(sl.h_idx32);
    sl.cap = std::max<int64_t>(L + L / 8, 1024);
    sl.d_idx32 = static_cast<int*>(dalloc(sizeof(int) * sl.cap));
    cuda_check(cudaHostAlloc(&sl.h_idx32, sizeof(int) * sl.cap, cudaHostAllocDefault), "pinned staging");
  }
  // nobody may still read the slot: its last commit's kernels (device) and
  // its last H2D (host buffer reuse)
  cuda_check(cudaEventSynchronize(sl.retired), "slot reuse");
  cuda_check(cudaEventSynchronize(sl.copied), "slot reuse");
  sl.err_key = ~0ull;
  sl.err_val = 0;
  sl.raw_used = false;
  sl.staged = true;
  sl.seq = ++stage_seq_;
  return sl;
}

void EmbContext::stage_fill_host(Slot& sl, const int64_t* const* offsets, const int64_t* const* indices,
                                 const int64_t* n_idx) {
  // background job: narrow + validate + H2D, per table piece, on the pool.
  // raw_eighths_/8 of the index pieces of PINNED tables go host->device as
  // int64 and are narrowed + validated on the GPU (narrow_validate_kernel):
  // host memory bandwidth (narrowing) and PCIe (copies) then both work.
  std::vector<std::array<int64_t, 4>> tasks;  // {table, begin, end, raw offset or -1}; begin = -1: offsets
  int64_t raw_n = 0, piece = 0;
  for (int t = 0; t < T_; ++t) {
    tasks.push_back({t, -1, 0, -1});
    bool pinned = false;
    if (raw_eighths_ > 0 && n_idx[t] > 0) {
      cudaPointerAttributes a{};
      pinned = cudaPointerGetAttributes(&a, indices[t]) == cudaSuccess && a.type == cudaMemoryTypeHost;
      (void)cudaGetLastError();
    }
    for (int64_t b = 0; b < n_idx[t]; b += kNarrowChunk, ++piece) {
      const int64_t e = std::min(n_idx[t], b + kNarrowChunk);
      const bool raw = pinned && (piece % 8) < raw_eighths_;
      tasks.push_back({t, b, e, raw ? raw_n : -1});
      if (raw) raw_n += e - b;
    }
  }
  if (raw_n > sl.raw_cap) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    if (sl.d_raw) {
      auto it = std::find(allocs_.begin(), allocs_.end(), (void*)sl.d_raw);
      if (it != allocs_.end()) allocs_.erase(it);
      cudaFree(sl.d_raw);
    }
    sl.raw_cap = raw_n + raw_n / 8;
    sl.d_raw = static_cast<long long*>(dalloc(sizeof(long long) * sl.raw_cap));
  }
  sl.raw_used = raw_n > 0;
  {
    int64_t n_raw_tasks = 0;
    for (auto& tk : tasks) n_raw_tasks += tk[3] >= 0;
    while ((int64_t)sl.raw_ev.size() < n_raw_tasks) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      sl.raw_ev.push_back(e);
    }
    if (!sl.narrowed) cuda_check(cudaEventCreateWithFlags(&sl.narrowed, cudaEventDisableTiming), "event");
    int64_t r = 0;
    for (auto& tk : tasks)
      if (tk[3] >= 0) tk[3] |= (r++) << 40;  // event index in the high bits
  }
  sl.src_idx.assign(indices, indices + T_);
  std::vector<const int64_t*> off(offsets, offsets + T_), idx(indices, indices + T_);
  Slot* sp = &sl;
  const int dev = device_;
  sl.job = std::thread([this, sp, dev, tasks = std::move(tasks), off = std::move(off), idx = std::move(idx)] {
    try {
      cudaSetDevice(dev);
      if (sp->raw_used) {  // the reset precedes every narrowing kernel (narrow_ waits on copy_ events)
        cuda_check(cudaMemsetAsync(sp->d_err, 0xff, sizeof(unsigned long long), copy_), "error key");
      }
      std::mutex emu;
      auto report = [&](int t, int kind, int64_t entry, int64_t value) {
        const unsigned long long key =
            ((unsigned long long)t << 42) | ((unsigned long long)kind << 40) | (unsigned long long)entry;
        std::lock_guard<std::mutex> lk(emu);
        if (key < sp->err_key) {
          sp->err_key = key;
          sp->err_val = value;
        }
      };
      staging_pool().parallel_for((int64_t)tasks.size(), [&](int64_t k) {
        const int t = (int)tasks[k][0];
        const DevTable& d = sp->tabs[t];
        if (tasks[k][1] < 0) {
          const int64_t* o = off[t];
          int* dst = sp->h_off32 + (int64_t)t * B_;
          if (o[0] != 0) report(t, 0, 0, o[0]);
          for (int64_t q = 0; q < B_; ++q) {
            if (q > 0 && o[q] < o[q - 1]) report(t, 1, q, o[q]);
            dst[q] = (int)(d.idx_off + o[q]);
          }
          if (B_ > 0 && o[B_] < o[B_ - 1]) report(t, 1, B_, o[B_]);
          if (o[B_] != d.n_lookups) report(t, 2, B_, o[B_]);
          if (t == T_ - 1) sp->h_off32[(int64_t)T_ * B_] = (int)(d.idx_off + d.n_lookups);
          cuda_check(cudaMemcpyAsync(sp->d_off32 + (int64_t)t * B_, dst, sizeof(int) * (t == T_ - 1 ? B_ + 1 : B_),
                                     cudaMemcpyHostToDevice, copy_),
                     "offsets H2D");
        } else if (tasks[k][3] >= 0) {  // raw: int64 H2D, narrowed + validated on the GPU
          const int64_t b = tasks[k][1], e = tasks[k][2];
          long long* raw = sp->d_raw + (tasks[k][3] & ((1LL << 40) - 1));
          cudaEvent_t ev = sp->raw_ev[tasks[k][3] >> 40];
          cuda_check(cudaMemcpyAsync(raw, idx[t] + b, sizeof(long long) * (e - b), cudaMemcpyHostToDevice, copy_),
                     "indices H2D (raw)");
          cuda_check(cudaEventRecord(ev, copy_), "raw copied");
          cuda_check(cudaStreamWaitEvent(narrow_, ev, 0), "narrow wait");
          narrow_validate_kernel<<<(unsigned)std::min<int64_t>((e - b + 255) / 256, 1184), 256, 0, narrow_>>>(
              raw, sp->d_idx32 + d.idx_off + b, e - b, d.hash,
              ((unsigned long long)t << 42) | (3ull << 40) | (unsigned long long)b, sp->d_err);
          cuda_check(cudaGetLastError(), "narrow_validate_kernel");
        } else {
          const int64_t b = tasks[k][1], e = tasks[k][2];
          const int64_t* src = idx[t];
          int* dst = sp->h_idx32 + d.idx_off;
          const int64_t hash = d.hash;
          const bool bad = narrow_rows(src + b, dst + b, e - b, hash, 0);
          if (bad)
            for (int64_t j = b; j < e; ++j)
              if (src[j] < 0 || src[j] >= hash) {
                report(t, 3, j, src[j]);
                break;
              }
          cuda_check(cudaMemcpyAsync(sp->d_idx32 + d.idx_off + b, dst + b, sizeof(int) * (e - b),
                                     cudaMemcpyHostToDevice, copy_),
                     "indices H2D");
        }
      });
      if (sp->raw_used) {
        cuda_check(cudaEventRecord(sp->narrowed, narrow_), "narrowed");
        cuda_check(cudaStreamWaitEvent(copy_, sp->narrowed, 0), "join narrow");
        cuda_check(cudaMemcpyAsync(sp->h_err, sp->d_err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, copy_),
                   "error key D2H");
      }
      cuda_check(cudaEventRecord(sp->copied, copy_), "copied");
    } catch (...) {
      sp->job_error = std::current_exception();
    }
  });
}

void EmbContext::commit(cudaStream_t s) {
  DeviceGuard g(device_);
  int pick = -1;
  for (int k = 0; k < 2; ++k)
    if (slots_[k].staged && (pick < 0 || slots_[k].seq < slots_[pick].seq)) pick = k;  // oldest first
  if (pick < 0) fail(AS_STATE, "as_commit_staged: no staged batch");
  Slot& sl = slots_[pick];
  loaded_ = false;
  sl.staged = false;
  if (sl.job.joinable()) sl.job.join();
  if (sl.job_error) {
    auto e = sl.job_error;
    sl.job_error = nullptr;
    std::rethrow_exception(e);
  }
  if (sl.raw_used) {  // the GPU-validated pieces: wait for their first-error key
    cuda_check(cudaEventSynchronize(sl.copied), "staged batch");
    const unsigned long long dk = *sl.h_err;
    if (dk < sl.err_key) {
      sl.err_key = dk;
      sl.err_val = sl.src_idx[dk >> 42][dk & ((1ull << 40) - 1)];
    }
  }
  if (sl.err_key != ~0ull) {
    const int t = static_cast<int>(sl.err_key >> 42);
    const int kind = static_cast<int>((sl.err_key >> 40) & 3);
    const int64_t q = static_cast<int64_t>(sl.err_key & ((1ull << 40) - 1));
    const std::string where = "table " + std::to_string(specs_[t].id);
    switch (kind) {
      case 0: fail(AS_OFFSET, where + ": offsets must start at 0, got " + std::to_string(sl.err_val));
      case 1: fail(AS_OFFSET, where + ": offsets must be nondecreasing at entry " + std::to_string(q));
      case 2:
        fail(AS_OFFSET, where + ": final offset " + std::to_string(sl.err_val) + " != index count " +
                            std::to_string(sl.tabs[t].n_lookups));
      default:
        fail(AS_INDEX, where + ": index " + std::to_string(sl.err_val) + " out of range [0, " +
                           std::to_string(specs_[t].hash_size) + ")");
    }
  }
  if (sort_pending_) {  // a forward's side-stream sort still reads the previous batch
    cuda_check(cudaStreamWaitEvent(s, ev_join_, 0), "join sort");
    sort_pending_ = false;
  }
  if (sl.L > cap_L_ || sl.nch > cap_chunks_ || sl.nun > cap_units_) cuda_check(cudaStreamSynchronize(s), "grow sync");
  ensure_capacity(sl.L, sl.nch, sl.nun);
  // retire the batch being replaced, then swap the slot in
  cuda_check(cudaEventRecord(cur_slot_ >= 0 ? slots_[cur_slot_].retired : sl.retired, s), "retire");
  cuda_check(cudaStreamWaitEvent(s, sl.copied, 0), "wait copy");
  htabs_ = sl.tabs;
  if (T_ > 0)
    cuda_check(cudaMemcpyAsync(dtabs_, htabs_.data(), sizeof(DevTable) * T_, cudaMemcpyHostToDevice, s),
               "tables H2D");
  if (sl.nun > 0)
    cuda_check(cudaMemcpyAsync(unit_table_, sl.utab.data(), sizeof(int) * sl.nun, cudaMemcpyHostToDevice, s),
               "unit table H2D");
  if ((int64_t)sl.sort_meta.size() > cap_sort_meta_) {
    cuda_check(cudaStreamSynchronize(s), "grow sync");
    if (sort_meta_) {
      auto it = std::find(allocs_.begin(), allocs_.end(), (void*)sort_meta_);
      if (it != allocs_.end()) allocs_.erase(it);
      cudaFree(sort_meta_);
    }
    cap_sort_meta_ = (int64_t)sl.sort_meta.size() + (int64_t)sl.sort_meta.size() / 8 + 64;
    sort_meta_ = static_cast<int*>(dalloc(sizeof(int) * cap_sort_meta_));
  }
  if (!sl.sort_meta.empty())
    cuda_check(cudaMemcpyAsync(sort_meta_, sl.sort_meta.data(), sizeof(int) * sl.sort_meta.size(),
                               cudaMemcpyHostToDevice, s),
               "sort layout H2D");
  for (int p = 0; p < kMaxSortPasses; ++p) {
    tile_tab_off_[p] = sl.tile_tab_off[p];
    pass_tiles_[p] = sl.pass_tiles[p];
  }
  n_sort_tiles_ = sl.n_sort_tiles;
  sort_sb_elems_ = sl.sort_sb_elems;
  sort_passes_ = sl.sort_passes;
  idx32_ = sl.d_idx32;
  off32_ = sl.d_off32;
  cur_slot_ = (int)(&sl - slots_);
  L_ = sl.L;
  n_chunks_ = sl.nch;
  n_units_ = sl.nun;
  bag_valid_ = false;  // K4 of this batch has not run yet
  loaded_ = true;
}

// A batch whose int32 rows and rebased offsets are produced ON THE DEVICE:
// `fill(d_idx32, d_off32, tabs, stream)` enqueues the kernels that write the
// slot's arrays (table t's rows at tabs[t].idx_off, offsets[t*B + b] global);
// commit then orders the step after them (the slot's copied event).
void EmbContext::stage_device(const int64_t* n_idx,
                              const std::function<void(int*, int*, const DevTable*, cudaStream_t)>& fill) {
  DeviceGuard g(device_);
  Slot& sl = stage_layout(n_idx);
  sl.src_idx.assign(static_cast<size_t>(T_), nullptr);
  try {
    fill(sl.d_idx32, sl.d_off32, sl.tabs.data(), copy_);
    cuda_check(cudaEventRecord(sl.copied, copy_), "copied");
  } catch (...) {
    sl.staged = false;
    throw;
  }
}

// Validation now completes at commit; kept for the C-ABI contract.
void EmbContext::check() {}

void EmbContext::load(const int64_t* const* offsets, const int64_t* const* indices, const int64_t* n_idx,
                      cudaStream_t s) {
  stage(offsets, indices, n_idx);
  commit(s);
  check();
}

void EmbContext::require_loaded(const char* what) const {
  if (!loaded_) fail(AS_STATE, std::string(what) + ": no streams loaded (call as_load_streams first)");
}

SegParams EmbContext::seg_params(bool fwd) const {
  SegParams p;
  std::memset(&p, 0, sizeof p);
  p.tabs = dtabs_;
  p.unit_table = unit_table_;
  p.n_units = static_cast<int>(n_units_);
  p.completers = completers_;
  p.n_completers = counters_ + (fwd ? 0 : 3);
  p.completers_mid = completers_mid_;
  p.n_completers_mid = counters_ + (fwd ? 2 : 5);
  p.completers_long = completers_long_;
  p.n_completers_long = counters_ + (fwd ? 1 : 4);
  p.seg = fwd ? bag_ : skey_;
  p.src = fwd ? idx32_ : sbag_;
  p.carry = carry_;
  p.carry_stride = max_dim_;
  p.stage_x = stage_x_;
  p.stage_s = stage_s_;
  p.w_half = w_half_ ? 1 : 0;
  return p;
}

// Shared-memory carveout of the segment kernels for THIS context's staging
// size (process-wide attribute, re-applied only when it changes).
void EmbContext::set_carveout(bool fwd) {
  static std::mutex mu;
  static int last[3] = {-1, -1, -1};  // fwd fp32, fwd fp16, bwd
  const int blocks = fwd ? ASB_SEG_MINBLOCKS_FWD : ASB_SEG_MINBLOCKS_BWD;
  const double need = (double)blocks * (double)(seg_smem_bytes_ + 1024);
  const int pct = std::min(100, (int)std::ceil(100.0 * need / (228.0 * 1024.0)) + 1);
  const int which = fwd ? (w_half_ ? 1 : 0) : 2;
  std::lock_guard<std::mutex> lk(mu);
  if (last[which] == pct) return;
  const void* f = fwd ? (w_half_ ? (const void*)seg_reduce_kernel<true, true> : (const void*)seg_reduce_kernel<true>)
                      : (const void*)seg_reduce_kernel<false>;
  cuda_check(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct), "carveout");
  last[which] = pct;
}

// K1 / K3 launch: one warp per unit, every lane layout in one launch.
template <bool FWD>
void EmbContext::launch_seg(SegParams p, cudaStream_t s) {
  if (n_units_ == 0) return;
  set_carveout(FWD);
  p.unit_begin = 0;
  if (FWD && w_half_)
    seg_reduce_kernel<true, true><<<grid_for(n_units_, kWarpsPerBlock), kBlock, seg_smem_bytes_, s>>>(p);
  else
    seg_reduce_kernel<FWD><<<grid_for(n_units_, kWarpsPerBlock), kBlock, seg_smem_bytes_, s>>>(p);
  cuda_check(cudaGetLastError(), "seg_reduce_kernel");
  ++launches_;
}

void EmbContext::forward(float* out, double* loss_dev, cudaStream_t s) {
  require_loaded("as_forward");
  DeviceGuard g(device_);
  if (T_ == 0) return;
  float* target = out ? out : out_;
  const long long nb = (long long)T_ * B_;
  const bool fork = n_chunks_ > 0 && !prof_serial_;
  if (fork) cuda_check(cudaEventRecord(ev_fork_, s), "fork");
  {
    Phase ph(this, 0, s);
    bag_expand_kernel<<<grid_for(nb, 32LL * kWarpsPerBlock), kBlock, 0, s>>>(off32_, T_, (int)B_, dtabs_, bag_,
                                                                            target, sum_dim_, peers_);
    cuda_check(cudaGetLastError(), "bag_expand_kernel");
    ++launches_;
    bag_valid_ = true;
  }
  if (fork) {
    cuda_check(cudaEventRecord(ev_k4_, s), "K4 done");
    cuda_check(cudaStreamWaitEvent(side_, ev_fork_, 0), "fork wait");
    launch_sort(side_, ev_k4_);
    cuda_check(cudaEventRecord(ev_join_, side_), "join");
    sort_pending_ = true;
  }
  if (n_chunks_ == 0) return;
  SegParams p = seg_params(true);
  p.W_ro = W_;
  p.out = target;
  p.out_stride = sum_dim_;
  p.peers = peers_;
  p.loss = loss_dev;
  cuda_check(cudaMemsetAsync(counters_, 0, sizeof(int) * 3, s), "counter reset");
  {
    Phase ph(this, 1, s);
    launch_seg<true>(p, s);
  }
  {
    Phase ph(this, 2, s);
    seg_fixup_lane_kernel<true><<<fixup_lane_grid_, kBlock, 0, s>>>(p);
    seg_fixup_kernel<true><<<fixup_short_grid_, kBlock, 0, s>>>(p);
    seg_fixup_long_kernel<true><<<fixup_grid_, kBlock, 0, s>>>(p);
    cuda_check(cudaGetLastError(), "seg_fixup_kernel<fwd>");
  }
  launches_ += 3;
}

// K2: stable radix sort of each table's (row, bag) pairs (sort.cuh). Depends
// on the loaded batch and K4's bag ids: as_forward launches it on a side
// stream at the start of the step, where the pass-0 digit counts overlap K4
// and the rest overlaps the forward gather (the pass-0 downsweep waits on
// `k4_done`); the backward joins on it, or sorts inline when no forward ran
// since the load (K4 then runs in ids-only mode first).
void EmbContext::launch_sort(cudaStream_t s, cudaEvent_t k4_done) {
  if (!k4_done && !bag_valid_ && T_ > 0) {
    const long long nb = (long long)T_ * B_;
    bag_expand_kernel<<<grid_for(nb, 32LL * kWarpsPerBlock), kBlock, 0, s>>>(off32_, T_, (int)B_, dtabs_, bag_,
                                                                            nullptr, sum_dim_, PeerOut{});
    cuda_check(cudaGetLastError(), "bag_expand_kernel");
    ++launches_;
    bag_valid_ = true;
  }
  Phase ph(this, 3, s);
  if (sort_passes_ == 0) return;
  SortParams sp;
  std::memset(&sp, 0, sizeof sp);
  sp.tabs = dtabs_;
  sp.keys_in = reinterpret_cast<const unsigned*>(idx32_);
  sp.vals_in = bag_;
  sp.keys_out = reinterpret_cast<unsigned*>(skey_);
  sp.vals_out = sbag_;
  sp.keys_tmp = reinterpret_cast<unsigned*>(tkey_);
  sp.vals_tmp = tbag_;
  sp.hist = sort_scratch_;
  sp.sb_tab = sort_meta_;
  sp.sb_elems = sort_sb_elems_;
  sp.bag_bits = bag_bits();
  for (int p = 0; p < sort_passes_; ++p) {
    sp.pass = p;
    sp.pass_sb = sort_meta_ + tile_tab_off_[p];
    const unsigned g = static_cast<unsigned>(pass_tiles_[p]);
    sort_upsweep_kernel<<<g, kSortThreads, 0, s>>>(sp);
    sort_scan_kernel<<<(unsigned)T_, kSortDigits, 0, s>>>(sp);
    if (p == 0 && k4_done) cuda_check(cudaStreamWaitEvent(s, k4_done, 0), "wait K4");
    sort_downsweep_kernel<<<g, kSortThreads, 0, s>>>(sp);
    cuda_check(cudaGetLastError(), "sort_downsweep_kernel");
  }
  launches_ += 3 * sort_passes_;
}

void EmbContext::backward(const float* grad, float lr, float eps, cudaStream_t s) {
  require_loaded("as_backward_rowwise_adagrad");
  if (!grad && peers_.n)
    fail(AS_STATE, "as_backward_rowwise_adagrad: the forward writes to peer buffers (as_set_peer_outputs); pass the "
                   "gradient of this shard's pooled rows");
  DeviceGuard g(device_);
  if (T_ == 0 || n_chunks_ == 0) return;
  if (sort_pending_) {
    cuda_check(cudaStreamWaitEvent(s, ev_join_, 0), "join sort");
    sort_pending_ = false;
  } else {
    launch_sort(s);
  }
  SegParams p = seg_params(false);
  p.grad = grad ? grad : out_;
  p.grad_stride = sum_dim_;
  p.W = W_;
  p.M = M_;
  p.lr = lr;
  p.eps = eps;
  cuda_check(cudaMemsetAsync(counters_ + 3, 0, sizeof(int) * 3, s), "counter reset");
  {
    Phase ph(this, 4, s);
    launch_seg<false>(p, s);
  }
  {
    Phase ph(this, 5, s);
    seg_fixup_lane_kernel<false><<<fixup_lane_grid_, kBlock, 0, s>>>(p);
    seg_fixup_kernel<false><<<fixup_short_grid_, kBlock, 0, s>>>(p);
    seg_fixup_long_kernel<false><<<fixup_grid_, kBlock, 0, s>>>(p);
    cuda_check(cudaGetLastError(), "seg_fixup_kernel<bwd>");
  }
  launches_ += 3;
}

void EmbContext::set_peer_outputs(int n, float* const* bases, const int64_t* row_start) {
  if (n == 0) {
    std::memset(&peers_, 0, sizeof peers_);
    return;
  }
  if (n < 0 || n > kMaxPeers) fail(AS_CONFIG, "as_set_peer_outputs: 0..8 peers, got " + std::to_string(n));
  if (row_start[0] != 0 || row_start[n] != B_)
    fail(AS_SHAPE, "as_set_peer_outputs: the peers' row ranges must cover the batch [0, " + std::to_string(B_) + ")");
  for (int q = 0; q < n; ++q) {
    if (row_start[q + 1] < row_start[q])
      fail(AS_SHAPE, "as_set_peer_outputs: row_start must be nondecreasing at peer " + std::to_string(q + 1));
    if (!bases[q] && row_start[q + 1] > row_start[q])
      fail(AS_CONFIG, "as_set_peer_outputs: peer " + std::to_string(q) + " has a NULL base");
  }
  std::memset(&peers_, 0, sizeof peers_);
  for (int q = 0; q < n; ++q) peers_.base[q] = bases[q];
  for (int q = 0; q <= n; ++q) peers_.start[q] = static_cast<int>(row_start[q]);
  for (int q = n + 1; q <= kMaxPeers; ++q) peers_.start[q] = static_cast<int>(B_);
  peers_.n = n;
}

void EmbContext::step(float lr, float eps, double* loss_host, cudaStream_t s) {
  require_loaded("as_step");
  if (peers_.n)
    fail(AS_STATE, "as_step: the forward writes to peer buffers (as_set_peer_outputs); run as_forward, the "
                   "exchange and as_backward_rowwise_adagrad");
  DeviceGuard g(device_);
  if (loss_host) cuda_check(cudaMemsetAsync(loss_, 0, sizeof(double), s), "loss reset");
  forward(out_, loss_host ? loss_ : nullptr, s);
  backward(out_, lr, eps, s);
  if (loss_host) {
    // D2H into pinned memory, then sleep (not spin) until the step is done: a
    // pageable D2H would hold the driver inside the copy for the whole step and
    // stall the staging threads' H2D submissions; the pool also needs the cores
    cuda_check(cudaMemcpyAsync(h_loss_, loss_, sizeof(double), cudaMemcpyDeviceToHost, s), "loss D2H");
    cuda_check(cudaEventRecord(ev_done_, s), "done");
    cuda_check(cudaEventSynchronize(ev_done_), "step sync");
    *loss_host = *h_loss_;
    check();  // report a bad batch with the step's result
  }
}

double EmbContext::measure(int warmup, int measure, int trim, bool flush, float lr, float eps) {
  if (warmup < 0 || measure < 1 || trim < 0 || measure - 2 * trim < 1)
    fail(AS_CONFIG, "micro_benchmark: need measure - 2*trim >= 1, got B=" + std::to_string(measure) +
                        " R=" + std::to_string(trim));
  check();
  require_loaded("as_measure");
  DeviceGuard g(device_);
  // order the measurement after every earlier use of this context (staged
  // copies, async steps on other streams, shared scratch)
  cuda_check(cudaDeviceSynchronize(), "measure: drain prior work");
  cudaStream_t s;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  std::vector<cudaEvent_t> ev(static_cast<size_t>(2 * measure));
  for (auto& e : ev) cuda_check(cudaEventCreate(&e), "event");
  for (int i = 0; i < warmup; ++i) step(lr, eps, nullptr, s);
  for (int i = 0; i < measure; ++i) {
    if (flush) cuda_check(cudaMemsetAsync(flush_, i & 0xff, flush_bytes_, s), "l2 flush");
    cuda_check(cudaEventRecord(ev[2 * i], s), "event");
    step(lr, eps, nullptr, s);
    cuda_check(cudaEventRecord(ev[2 * i + 1], s), "event");
  }
  cuda_check(cudaStreamSynchronize(s), "measure sync");
  std::vector<double> ms(static_cast<size_t>(measure));
  for (int i = 0; i < measure; ++i) {
    float x = 0.f;
    cuda_check(cudaEventElapsedTime(&x, ev[2 * i], ev[2 * i + 1]), "elapsed");
    ms[i] = x;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  cudaStreamDestroy(s);
  std::sort(ms.begin(), ms.end());
  double sum = 0.0;
  for (int i = trim; i < measure - trim; ++i) sum += ms[i];
  return sum / static_cast<double>(measure - 2 * trim);
}

// Raw cost-model features of the loaded batch, laid out like FeatureVector::raw
// (tables.hpp:300-386): [dim, hash_size, observed pooling, size_gb, 17 bins].
void EmbContext::table_features(double* out, cudaStream_t s) {
  check();
  require_loaded("as_table_features");
  DeviceGuard g(device_);
  std::vector<unsigned long long> hist(static_cast<size_t>(std::max(1, T_)) * 18, 0ull);
  if (T_ > 0 && L_ > 0) {
    if (sort_pending_) {
      cuda_check(cudaStreamWaitEvent(s, ev_join_, 0), "join sort");
    } else {
      launch_sort(s);  // sorted keys of the current batch
    }
    std::vector<long long> starts(static_cast<size_t>(T_) + 1);
    for (int t = 0; t < T_; ++t) starts[t] = htabs_[t].idx_off;
    starts[T_] = L_;
    long long* d_starts = nullptr;
    unsigned long long* d_hist = nullptr;
    cuda_check(cudaMallocAsync(&d_starts, sizeof(long long) * (T_ + 1), s), "malloc");
    cuda_check(cudaMallocAsync(&d_hist, sizeof(unsigned long long) * T_ * 18, s), "malloc");
    cuda_check(cudaMemcpyAsync(d_starts, starts.data(), sizeof(long long) * (T_ + 1), cudaMemcpyHostToDevice, s),
               "starts H2D");
    cuda_check(cudaMemsetAsync(d_hist, 0, sizeof(unsigned long long) * T_ * 18, s), "hist reset");
    row_count_hist_kernel<<<grid_for(L_, 256), 256, 0, s>>>(skey_, d_starts, T_, L_, d_hist);
    cuda_check(cudaGetLastError(), "row_count_hist_kernel");
    cuda_check(cudaMemcpyAsync(hist.data(), d_hist, sizeof(unsigned long long) * T_ * 18, cudaMemcpyDeviceToHost, s),
               "hist D2H");
    cuda_check(cudaStreamSynchronize(s), "features sync");
    cudaFree(d_starts);
    cudaFree(d_hist);
    sort_pending_ = false;
  }
  for (int t = 0; t < T_; ++t) {
    double* f = out + (size_t)t * 21;
    const as_table_spec& sp = specs_[t];
    f[0] = (double)sp.dim;
    f[1] = (double)sp.hash_size;
    f[2] = (double)htabs_[t].n_lookups / (double)B_;  // observed_pooling (tables.hpp:337-342)
    f[3] = (double)((int64_t)sp.dim * sp.hash_size * sp.bytes_per_param) / (1024.0 * 1024.0 * 1024.0);
    const double distinct = (double)hist[(size_t)t * 18 + 17];
    for (int b = 0; b < 17; ++b) f[4 + b] = distinct > 0 ? (double)hist[(size_t)t * 18 + b] / distinct : 0.0;
  }
}

void EmbContext::read_rows(int t, const int64_t* rows, int64_t n, float* out) {
  check();
  if (t < 0 || t >= T_) fail(AS_LOOKUP, "as_read_rows: table position " + std::to_string(t) + " out of range");
  for (int64_t i = 0; i < n; ++i)
    if (rows[i] < 0 || rows[i] >= specs_[t].hash_size)
      fail(AS_INDEX, "table " + std::to_string(specs_[t].id) + ": row " + std::to_string(rows[i]) + " out of range");
  if (n == 0) return;
  DeviceGuard g(device_);
  long long* drows = nullptr;
  float* dst = nullptr;
  cuda_check(cudaMalloc(&drows, sizeof(long long) * n), "malloc");
  cuda_check(cudaMalloc(&dst, sizeof(float) * n * specs_[t].dim), "malloc");
  cuda_check(cudaMemcpy(drows, rows, sizeof(long long) * n, cudaMemcpyHostToDevice), "rows H2D");
  const long long w_off = htabs_[t].w_base;
  gather_rows_kernel<<<grid_for(n * specs_[t].dim, 256), 256>>>(W_, w_half_ ? 1 : 0, w_off, specs_[t].dim, drows, n,
                                                                 dst);
  cuda_check(cudaGetLastError(), "gather_rows_kernel");
  cuda_check(cudaMemcpy(out, dst, sizeof(float) * n * specs_[t].dim, cudaMemcpyDeviceToHost), "rows D2H");
  cudaFree(drows);
  cudaFree(dst);
}

void EmbContext::read_momentum(int t, const int64_t* rows, int64_t n, float* out) {
  check();
  if (t < 0 || t >= T_) fail(AS_LOOKUP, "as_read_momentum: table position out of range");
  if (n == 0) return;
  DeviceGuard g(device_);
  std::vector<float> all(static_cast<size_t>(specs_[t].hash_size));
  cuda_check(cudaMemcpy(all.data(), M_ + htabs_[t].row_off, sizeof(float) * all.size(), cudaMemcpyDeviceToHost),
             "momentum D2H");
  for (int64_t i = 0; i < n; ++i) {
    if (rows[i] < 0 || rows[i] >= specs_[t].hash_size) fail(AS_INDEX, "as_read_momentum: row out of range");
    out[i] = all[static_cast<size_t>(rows[i])];
  }
}

void EmbContext::read_buffer(int what, void* host, int64_t nbytes) {
  check();
  DeviceGuard g(device_);
  const void* src = nullptr;
  int64_t want = 0;
  switch (what) {
    case 0: src = out_; want = B_ * sum_dim_ * 4; break;
    case 1: src = bag_; want = L_ * 4; break;
    case 2: src = skey_; want = L_ * 4; break;
    case 3: src = sbag_; want = L_ * 4; break;
    case 4: src = idx32_; want = L_ * 4; break;
    default: fail(AS_CONFIG, "as_read_buffer: unknown buffer " + std::to_string(what));
  }
  if (what != 0) require_loaded("as_read_buffer");
  if (nbytes != want)
    fail(AS_SHAPE, "as_read_buffer: buffer " + std::to_string(what) + " has " + std::to_string(want) +
                       " bytes, caller passed " + std::to_string(nbytes));
  if (want) cuda_check(cudaMemcpy(host, src, static_cast<size_t>(want), cudaMemcpyDeviceToHost), "read D2H");
  if (what == 2 || what == 4) {  // device rows are table-local: report GLOBAL rows (row_off_t + r)
    int* h = static_cast<int*>(host);
    for (int t = 0; t < T_; ++t)
      for (int64_t j = htabs_[t].idx_off; j < htabs_[t].idx_off + htabs_[t].n_lookups; ++j)
        h[j] += static_cast<int>(htabs_[t].row_off);
  }
}

void EmbContext::write_table(int t, const float* w, const float* m) {
  if (t < 0 || t >= T_) fail(AS_LOOKUP, "as_write_table: table position out of range");
  DeviceGuard g(device_);
  const size_t rows = static_cast<size_t>(specs_[t].hash_size);
  if (w) {
    const long long w_off = htabs_[t].w_base;
    const size_t n = rows * specs_[t].dim;
    if (w_half_) {
      std::vector<__half> h(n);
      for (size_t i = 0; i < n; ++i) h[i] = __float2half_rn(w[i]);
      cuda_check(cudaMemcpy(reinterpret_cast<__half*>(W_) + w_off, h.data(), sizeof(__half) * n, cudaMemcpyHostToDevice),
                 "W H2D");
    } else {
      cuda_check(cudaMemcpy(W_ + w_off, w, sizeof(float) * n, cudaMemcpyHostToDevice), "W H2D");
    }
  }
  if (m) cuda_check(cudaMemcpy(M_ + htabs_[t].row_off, m, sizeof(float) * rows, cudaMemcpyHostToDevice), "M H2D");
}

void EmbContext::info(as_ctx_info* o) const {
  std::memset(o, 0, sizeof *o);
  o->device = device_;
  o->n_tables = T_;
  o->batch_size = B_;
  o->sum_dim = sum_dim_;
  o->total_rows = total_rows_;
  o->n_lookups = loaded_ ? L_ : 0;
  o->n_chunks = loaded_ ? n_chunks_ : 0;
  o->device_bytes = bytes_;
  o->pooled = out_;
  o->weights = W_;
  o->momentum = M_;
  // bag_expand + seg_reduce/fixup (fwd) + radix sort + seg_reduce/fixup (bwd)
  o->weight_bytes = w_half_ ? 2 : 4;
  o->kernels_per_step = T_ == 0 ? 0 : (n_chunks_ == 0 ? 1 : 9 + 3 * sort_passes_);
}

}  // namespace asb
