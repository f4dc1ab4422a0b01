// One rank of the table-wise sharded step (sharded.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "autoshard_b200.h"
#include "types.hpp"

struct ncclComm;

namespace asb {

class EmbContext;

void nccl_unique_id(void* out);

class ShardComm {
 public:
  ShardComm(EmbContext* ctx, const void* unique_id, int rank, int world);
  ~ShardComm();
  ShardComm(const ShardComm&) = delete;
  ShardComm& operator=(const ShardComm&) = delete;

  void setup(const int64_t* shard_dims, const int64_t* row_start, int mode);
  void handle(void* blob, int64_t* nbytes);
  void open(const void* all_blobs);
  void forward(cudaStream_t s);
  void backward(const float* grad_recv, float lr, float eps, cudaStream_t s);
  void step(float lr, float eps, double* loss_host, cudaStream_t s);
  void info(as_comm_info* out) const;
  // KJT all-to-all: this rank's mini-batch of every table -> the owners (as_load_streams_exchanged)
  void load_exchanged(int n_all, const as_table_spec* all, const int32_t* owner, const int64_t* const* local_offsets,
                      const int64_t* const* local_indices, cudaStream_t s);
  void profile_read(double* ms2, bool reset);
  // ranks sharing ONE device: a host-side barrier instead of the device one
  void set_host_barrier(as_host_barrier_fn fn, void* user) {
    host_fn_ = fn;
    host_user_ = user;
  }

 private:
  void require_open(const char* what) const;
  void check_async();
  void barrier(cudaStream_t s);
  void timed(int which, cudaStream_t s, bool begin);
  void collect();
  void grow(void** p, int64_t* cap, int64_t bytes);
  void grow_host(void** p, int64_t* cap, int64_t bytes);

  EmbContext* ctx_;
  int rank_, world_;
  int mode_ = 0;
  ncclComm* comm_ = nullptr;
  bool setup_ = false, open_ = false;
  std::vector<int64_t> dims_, start_, col_;  // shard widths, sample ranges, receive-block columns
  int64_t rows_ = 0;                          // this rank's samples
  float* recv_ = nullptr;                     // [world blocks [rows_, dims_[k]]]
  float* grad_ = nullptr;                     // [B, dims_[rank_]]
  unsigned long long* flags_ = nullptr;       // barrier flags [kMaxPeers]
  float* peer_recv_[kMaxPeers] = {};
  float* peer_grad_[kMaxPeers] = {};
  unsigned long long* peer_flags_[kMaxPeers] = {};
  bool opened_[kMaxPeers] = {};
  unsigned long long epoch_ = 0;
  as_host_barrier_fn host_fn_ = nullptr;
  void* host_user_ = nullptr;
  int* err_ = nullptr;   // device: barrier timeout
  int* h_err_ = nullptr; // pinned mirror (copied after every barrier)
  double* loss_ = nullptr;
  double* h_loss_ = nullptr;
  void* blob_dev_ = nullptr;
  cudaEvent_t ev_[4] = {};
  bool pending_[2] = {false, false};
  double ms_[2] = {0.0, 0.0};
  int64_t launches_ = 0;
  // KJT exchange buffers (grow-only)
  void *kjt_meta_ = nullptr, *kjt_send_ = nullptr, *kjt_recv_ = nullptr, *kjt_geo_ = nullptr, *kjt_tabs_ = nullptr;
  void* kjt_h_ = nullptr;  // pinned send staging
  int64_t kjt_meta_cap_ = 0, kjt_send_cap_ = 0, kjt_recv_cap_ = 0, kjt_geo_cap_ = 0, kjt_tabs_cap_ = 0, kjt_h_cap_ = 0;
  cudaEvent_t ev_kjt_ = nullptr;
};

}  // namespace asb
