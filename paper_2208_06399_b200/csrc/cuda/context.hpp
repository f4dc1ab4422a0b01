// Device context: one shard of tables resident on one B200.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <exception>
#include <functional>
#include <thread>
#include <vector>

#include "../host/host.hpp"
#include "types.hpp"

namespace asb {

void cuda_check(cudaError_t e, const char* what);
// probe.cu: random-row gather GB/s over `footprint` bytes (roofline denominator)
double probe_gather_bw(int device, int64_t footprint, int row_bytes);

class EmbContext {
 public:
  EmbContext(int device, const as_table_spec* tables, int n, int64_t batch, uint64_t seed, int flags = 0);
  // subset of parent's tables on parent's weight / momentum storage (as_create_subset)
  EmbContext(const EmbContext& parent, const int* positions, int n);
  // subset context only: another subset of the same parent (as_retarget_subset)
  void retarget(const int* positions, int n);
  ~EmbContext();
  EmbContext(const EmbContext&) = delete;
  EmbContext& operator=(const EmbContext&) = delete;

  void load(const int64_t* const* offsets, const int64_t* const* indices, const int64_t* n_idx,
            cudaStream_t s);
  // asynchronous double-buffered loading: stage (H2D on the copy stream),
  // commit (pack + validate on s), check (sync + report errors)
  void stage(const int64_t* const* offsets, const int64_t* const* indices, const int64_t* n_idx);
  // a batch filled on the device (KJT exchange): layout from n_idx, then fill
  // enqueues kernels on `stream` writing (d_idx32, d_off32) for the host-built
  // table layout `tabs` (idx_off per table); commit as usual
  void stage_device(const int64_t* n_idx,
                    const std::function<void(int*, int*, const DevTable*, cudaStream_t)>& fill);
  void commit(cudaStream_t s);
  void check();
  void forward(float* out, double* loss_dev, cudaStream_t s);
  void backward(const float* grad, float lr, float eps, cudaStream_t s);
  void set_peer_outputs(int n, float* const* bases, const int64_t* row_start);
  bool has_peers() const { return peers_.n != 0; }
  bool profiling() const { return prof_; }
  int64_t batch() const { return B_; }
  int64_t sum_dim() const { return sum_dim_; }
  float* pooled() const { return out_; }
  void step(float lr, float eps, double* loss_host, cudaStream_t s);
  double measure(int warmup, int measure, int trim, bool flush, float lr, float eps);

  void table_features(double* out, cudaStream_t s);
  void read_rows(int t, const int64_t* rows, int64_t n, float* out);
  void read_momentum(int t, const int64_t* rows, int64_t n, float* out);
  void read_buffer(int what, void* host, int64_t nbytes);
  void write_table(int t, const float* w, const float* m);
  void info(as_ctx_info* out) const;

  // Per-phase CUDA-event timing (bag_expand, fwd_seg, fwd_fixup, sort,
  // bwd_seg, bwd_fixup) and launch counting, for bench.py's roofline.
  static constexpr int kPhases = 6;
  void profile_enable(int mode);  // 0 off, 1 on, 2 on + serialized (no side-stream sort)
  void profile_read(double* ms, int64_t* launches, bool reset);

  int device() const { return device_; }
  int n_tables() const { return T_; }
  int table_id(int t) const { return specs_[t].id; }
  // bits of the largest bag id (K2's packed keys)
  int bag_bits() const {
    int b = 0;
    while (b < 40 && (B_ - 1) >> b) ++b;
    return b;
  }
  const as_table_spec& spec(int t) const { return specs_[t]; }

 private:
  void require_loaded(const char* what) const;
  void ensure_capacity(int64_t L, int64_t n_chunks, int64_t n_units);
  void* dalloc(size_t bytes);
  SegParams seg_params(bool fwd) const;
  void launch_sort(cudaStream_t s, cudaEvent_t k4_done = nullptr);
  void layout_tables();
  void setup_runtime();
  void set_carveout(bool fwd);
  struct Slot;
  Slot& stage_layout(const int64_t* n_idx);
  void stage_fill_host(Slot& sl, const int64_t* const* offsets, const int64_t* const* indices, const int64_t* n_idx);
  template <bool FWD>
  void launch_seg(SegParams p, cudaStream_t s);

  int device_;
  int T_;
  int64_t B_;
  uint64_t seed_;
  bool w_half_ = false;  // AS_WEIGHTS_FP16: W stored as __half
  std::vector<as_table_spec> specs_;
  std::vector<DevTable> htabs_;
  int64_t sum_dim_ = 0, total_rows_ = 0, total_w_ = 0;
  const EmbContext* parent_ = nullptr;  // subset contexts: the storage owner
  int cap_tables_ = 0;                   // dtabs_ / off32 slots sized for this many tables
  int64_t cap_out_ = 0;                  // out_ floats
  int max_dim_ = 4;
  int stage_x_ = 32, stage_s_ = 33;
  size_t seg_smem_bytes_ = 0;
  // K2 (sort.cuh): per-batch layout, uploaded at commit
  int* sort_meta_ = nullptr;     // device copy of Slot::sort_meta
  int64_t cap_sort_meta_ = 0;
  int* sort_scratch_ = nullptr;  // [superblocks][256] digit counts of the running pass
  int64_t cap_sort_tiles_ = 0;
  int64_t tile_tab_off_[kMaxSortPasses] = {0, 0, 0, 0};
  int64_t pass_tiles_[kMaxSortPasses] = {0, 0, 0, 0};
  int64_t n_sort_tiles_ = 0;
  int sort_sb_elems_ = kSortTile;
  int sort_passes_ = 0;

  DevTable* dtabs_ = nullptr;
  float* W_ = nullptr;
  float* M_ = nullptr;
  float* out_ = nullptr;
  int* off32_ = nullptr;  // current batch (points into a slot)
  struct Slot {
    int* d_idx32 = nullptr;  // [cap] device: GLOBAL rows
    int* d_off32 = nullptr;  // [T*B + 1] device: rebased offsets
    int* h_idx32 = nullptr;  // pinned host staging of the same
    int* h_off32 = nullptr;
    int64_t cap = 0;
    std::vector<DevTable> tabs;  // per-batch table layout (lookups, chunks, units)
    std::vector<int> utab;
    int64_t L = 0, nch = 0, nun = 0;
    long long* d_raw = nullptr;  // int64 pieces narrowed on the GPU
    int64_t raw_cap = 0;
    bool raw_used = false;
    unsigned long long* d_err = nullptr;  // first GPU validation error key
    unsigned long long* h_err = nullptr;  // pinned copy
    std::vector<const int64_t*> src_idx;  // caller's index arrays (error value lookup)
    std::vector<cudaEvent_t> raw_ev;       // per raw piece: its H2D landed
    cudaEvent_t narrowed = nullptr;        // every GPU-narrowed piece done
    std::vector<int> sort_meta;  // superblock -> table | per pass: its superblocks
    int64_t tile_tab_off[kMaxSortPasses] = {0, 0, 0, 0};
    int64_t pass_tiles[kMaxSortPasses] = {0, 0, 0, 0};
    int64_t n_sort_tiles = 0;
    int sort_sb_elems = kSortTile;
    int sort_passes = 0;
    cudaEvent_t copied = nullptr;   // all H2D of the batch landed
    cudaEvent_t retired = nullptr;  // the device no longer reads the batch
    std::thread job;                // narrow + validate + H2D
    std::exception_ptr job_error;
    unsigned long long err_key = ~0ull;  // first validation error (table, kind, entry)
    int64_t err_val = 0;
    bool staged = false;
    uint64_t seq = 0;  // staging order (commit takes the oldest)
  };
  Slot slots_[2];
  int cur_slot_ = -1;
  uint64_t stage_seq_ = 0;
  cudaStream_t copy_ = nullptr;
  cudaStream_t narrow_ = nullptr;  // high-priority stream of the GPU narrowing kernels
  unsigned long long* err_ = nullptr;
  double* loss_ = nullptr;
  double* h_loss_ = nullptr;  // pinned: a pageable D2H would block every other thread's CUDA calls
  void* flush_ = nullptr;
  size_t flush_bytes_ = 0;

  // batch-dependent (grown on demand)
  int64_t cap_L_ = 0, cap_chunks_ = 0;
  int* idx32_ = nullptr;
  int* bag_ = nullptr;
  int* skey_ = nullptr;
  int* sbag_ = nullptr;
  int* tkey_ = nullptr;  // K2 ping-pong
  int* tbag_ = nullptr;
  int* unit_table_ = nullptr;
  int2* completers_ = nullptr;
  int4* completers_long_ = nullptr;
  int2* completers_mid_ = nullptr;
  int* counters_ = nullptr;  // [0,1,2] fwd completers (all, long, mid), [3,4,5] bwd
  unsigned fixup_grid_ = 296;
  unsigned fixup_short_grid_ = 2368;
  unsigned fixup_lane_grid_ = 592;
  int64_t cap_units_ = 0;
  int64_t n_units_ = 0;
  PeerOut peers_{};  // fused forward exchange (as_set_peer_outputs); n = 0: local output
  int raw_eighths_ = 0;  // ASB_RAW_EIGHTHS: eighths of the index pieces narrowed on the GPU
  int vec_ = 1;  // preferred float4 per lane (ASB_VEC, A/B)
  // dims laid out with 2 float4 per lane (ASB_VEC2_DIMS): 64 -> GL 8 x NV 2
  // (cfg3 step -1.9 %; 128 helps mixed-dim shards but costs 1.7 % on cfg2)
  std::vector<int> vec2_dims_{64};
  double chunk_cap_ = 262144.0;  // max gathered bytes per chunk (ASB_CHUNK_KB, A/B; 256 KB: -0.7 % cfg2, -1.2 % cfg3 step vs 128 KB)
  double unit_cap_ = 262144.0;  // max gathered bytes per warp unit (ASB_UNIT_KB, A/B)
  float* carry_ = nullptr;

  cudaStream_t side_ = nullptr;  // K2 sort overlapped with the forward
  cudaEvent_t ev_k4_ = nullptr;  // K4 of this step done (the sort's pass-0 downsweep waits on it)
  bool bag_valid_ = false;       // bag_ holds the current batch's bag ids (K4 ran since the commit)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_done_ = nullptr;
  bool sort_pending_ = false;
  int64_t L_ = 0;
  int64_t n_chunks_ = 0;
  bool loaded_ = false;
  int64_t bytes_ = 0;
  int64_t launches_ = 0;
  bool prof_ = false;
  bool prof_serial_ = false;
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used_;
  cudaEvent_t ev_get();
  struct Phase;
  std::vector<void*> allocs_;
};

}  // namespace asb
