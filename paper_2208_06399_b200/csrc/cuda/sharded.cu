// Table-wise sharded step over G processes, one per GPU (
// SURVEY.md §8e): rank k holds the tables of plan.assignment == k and pools
// them for the whole global batch; sample owner p receives its rows
// [row_start[p], row_start[p+1]) of every shard and sends the gradient of
// those rows back.
//
// Receive buffer of rank p: world blocks in rank order, block k = [rows_p,
// SD_k] fp32 (rows contiguous, so every block is one contiguous region on
// both sides of the exchange). Gradient buffer of rank k: [B, SD_k].
//
// Exchange, per direction (as_alltoall_setup mode bits):
//   peer memory — forward: the ctx's K4/K1/fixup epilogues store each pooled
//     row straight into its owner's receive block (PeerOut, kernels.cuh), then
//     a system-scope release/acquire barrier kernel; backward: one copy-engine
//     push per owner into the table owners' gradient buffers, then the barrier.
//     Buffers of other processes are mapped with cudaIpc handles.
//   NCCL — grouped ncclSend/ncclRecv of the same contiguous blocks.
// NCCL is loaded at run time (dlopen libnccl.so.2): a process that already
// has torch's NCCL loaded gets that same library.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../host/host.hpp"
#include "context.hpp"
#include "sharded.hpp"

namespace asb {

// ---- NCCL, resolved at run time ---------------------------------------------
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
#define ASB_SYM(name)                                                                          \
  a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, "nccl" #name));                         \
  if (!a.name) {                                                                               \
    a.error = "libnccl.so.2 lacks nccl" #name;                                                 \
    return a;                                                                                  \
  }
    ASB_SYM(GetUniqueId)
    ASB_SYM(CommInitRank)
    ASB_SYM(CommDestroy)
    ASB_SYM(CommGetAsyncError)
    ASB_SYM(GetErrorString)
    ASB_SYM(GroupStart)
    ASB_SYM(GroupEnd)
    ASB_SYM(Send)
    ASB_SYM(Recv)
    ASB_SYM(AllGather)
#undef ASB_SYM
    return a;
  }();
  if (!api.error.empty()) fail(AS_NCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess && r != ncclInProgress)
    fail(AS_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---- device pieces -----------------------------------------------------------
struct BarrierFlags {
  unsigned long long* peer[kMaxPeers];  // rank q's flag array (slot `rank` is ours to write)
  unsigned long long* mine;             // our flag array (slot q written by rank q)
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// System-scope barrier of `world` ranks: lane q publishes our arrival in rank
// q's flags (release: every write this process made to peer memory before it —
// the forward's NVLink stores, the backward's pushes, both stream-ordered
// before this kernel — is visible to q once q acquires), then waits for q's
// arrival in ours (acquire). A peer that never arrives sets *err after 60 s
// instead of hanging the device.
__global__ void peer_barrier_kernel(BarrierFlags f, int rank, int world, unsigned long long epoch, int* err) {
  const int q = threadIdx.x;
  if (q >= world) return;
  __threadfence_system();
  unsigned long long* slot = f.peer[q] + rank;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(epoch) : "memory");
  const unsigned long long* mine = f.mine + q;
  const unsigned long long t0 = global_ns();
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
    if (v >= epoch) break;
    if (global_ns() - t0 > 60ull * 1000000000ull) {
      atomicExch(err, 1);
      break;
    }
    __nanosleep(200);
  }
}

// 1/2 sum x^2 over n floats into *out (fp64 accumulation per block).
__global__ void __launch_bounds__(256) half_sumsq_kernel(const float4* __restrict__ x, long long n4,
                                                         double* __restrict__ out) {
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    acc += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += part[w];
    if (s != 0.0) atomicAdd(out, 0.5 * s);
  }
}

struct HandleBlob {
  unsigned magic;
  int rank;
  int device;
  int pid;
  cudaIpcMemHandle_t recv, grad, flags;
};
constexpr unsigned kBlobMagic = 0xa5b20001u;
static_assert(sizeof(HandleBlob) <= AS_HANDLE_BYTES, "handle blob too large");

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
}  // namespace

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

ShardComm::ShardComm(EmbContext* ctx, const void* uid, int rank, int world) : ctx_(ctx), rank_(rank), world_(world) {
  if (world < 1 || world > kMaxPeers) fail(AS_CONFIG, "as_comm_init: world must be in [1, 8], got " + std::to_string(world));
  if (rank < 0 || rank >= world)
    fail(AS_CONFIG, "as_comm_init: rank " + std::to_string(rank) + " out of range for world " + std::to_string(world));
  DeviceGuard g(ctx_->device());
  if (uid) {
    static_assert(sizeof(ncclUniqueId) == AS_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    nccl_check(nccl().CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  cuda_check(cudaMalloc(&err_, sizeof(int)), "cudaMalloc");
  cuda_check(cudaMemset(err_, 0, sizeof(int)), "memset");
  cuda_check(cudaHostAlloc(&h_err_, sizeof(int), cudaHostAllocDefault), "pinned");
  *h_err_ = 0;
  cuda_check(cudaMalloc(&loss_, sizeof(double)), "cudaMalloc");
  cuda_check(cudaHostAlloc(&h_loss_, sizeof(double), cudaHostAllocDefault), "pinned");
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "event");
  cuda_check(cudaEventCreateWithFlags(&ev_kjt_, cudaEventDisableTiming), "event");
}

ShardComm::~ShardComm() {
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx_->device());
  cudaDeviceSynchronize();
  ctx_->set_peer_outputs(0, nullptr, nullptr);
  for (int q = 0; q < world_; ++q)
    if (q != rank_ && opened_[q]) {
      if (peer_recv_[q]) cudaIpcCloseMemHandle(peer_recv_[q]);
      if (peer_grad_[q]) cudaIpcCloseMemHandle(peer_grad_[q]);
      if (peer_flags_[q]) cudaIpcCloseMemHandle(peer_flags_[q]);
    }
  if (comm_) nccl().CommDestroy(comm_);
  for (void* p : {(void*)recv_, (void*)grad_, (void*)flags_, (void*)err_, (void*)loss_, (void*)blob_dev_, kjt_meta_,
                  kjt_send_, kjt_recv_, kjt_geo_, kjt_tabs_})
    if (p) cudaFree(p);
  if (kjt_h_) cudaFreeHost(kjt_h_);
  if (ev_kjt_) cudaEventDestroy(ev_kjt_);
  if (h_err_) cudaFreeHost(h_err_);
  if (h_loss_) cudaFreeHost(h_loss_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (prev >= 0) cudaSetDevice(prev);
}

void ShardComm::setup(const int64_t* shard_dims, const int64_t* row_start, int mode) {
  if (setup_) fail(AS_STATE, "as_alltoall_setup: already set up");
  if (mode & ~3) fail(AS_CONFIG, "as_alltoall_setup: unknown mode " + std::to_string(mode));
  if ((mode & 3) && !comm_) fail(AS_CONFIG, "as_alltoall_setup: an NCCL exchange needs an NCCL communicator");
  const int64_t B = ctx_->batch();
  if (row_start[0] != 0 || row_start[world_] != B)
    fail(AS_SHAPE, "as_alltoall_setup: row_start must run from 0 to the batch " + std::to_string(B));
  dims_.assign(shard_dims, shard_dims + world_);
  start_.assign(row_start, row_start + world_ + 1);
  col_.assign(world_ + 1, 0);
  for (int k = 0; k < world_; ++k) {
    if (dims_[k] < 0) fail(AS_SHAPE, "as_alltoall_setup: shard " + std::to_string(k) + " has negative width");
    if (start_[k + 1] < start_[k])
      fail(AS_SHAPE, "as_alltoall_setup: row_start must be nondecreasing at rank " + std::to_string(k + 1));
    col_[k + 1] = col_[k] + dims_[k];
  }
  if (dims_[rank_] != ctx_->sum_dim())
    fail(AS_SHAPE, "as_alltoall_setup: shard_dims[" + std::to_string(rank_) + "] = " + std::to_string(dims_[rank_]) +
                       " but this rank's tables have " + std::to_string(ctx_->sum_dim()) + " pooled columns");
  mode_ = mode;
  rows_ = start_[rank_ + 1] - start_[rank_];
  DeviceGuard g(ctx_->device());
  cuda_check(cudaMalloc(&recv_, sizeof(float) * std::max<int64_t>(4, rows_ * col_[world_])), "cudaMalloc recv");
  cuda_check(cudaMalloc(&grad_, sizeof(float) * std::max<int64_t>(4, B * dims_[rank_])), "cudaMalloc grad");
  cuda_check(cudaMalloc(&flags_, sizeof(unsigned long long) * kMaxPeers), "cudaMalloc flags");
  cuda_check(cudaMemset(flags_, 0, sizeof(unsigned long long) * kMaxPeers), "memset");
  cuda_check(cudaMemset(recv_, 0, sizeof(float) * std::max<int64_t>(4, rows_ * col_[world_])), "memset");
  cuda_check(cudaDeviceSynchronize(), "setup");
  setup_ = true;
  if (comm_) {  // all-gather the handle blobs over NCCL, then open them
    std::vector<unsigned char> all((size_t)AS_HANDLE_BYTES * world_);
    int64_t n = 0;
    handle(all.data() + (size_t)AS_HANDLE_BYTES * rank_, &n);
    cuda_check(cudaMalloc(&blob_dev_, all.size()), "cudaMalloc");
    cuda_check(cudaMemcpy((char*)blob_dev_ + (size_t)AS_HANDLE_BYTES * rank_, all.data() + (size_t)AS_HANDLE_BYTES * rank_,
                          AS_HANDLE_BYTES, cudaMemcpyHostToDevice),
               "blob H2D");
    nccl_check(nccl().AllGather((char*)blob_dev_ + (size_t)AS_HANDLE_BYTES * rank_, blob_dev_, AS_HANDLE_BYTES, ncclChar,
                                comm_, nullptr),
               "ncclAllGather (handles)");
    cuda_check(cudaMemcpy(all.data(), blob_dev_, all.size(), cudaMemcpyDeviceToHost), "blob D2H");
    check_async();
    open(all.data());
  }
}

void ShardComm::handle(void* blob, int64_t* nbytes) {
  if (!setup_) fail(AS_STATE, "as_alltoall_handle: call as_alltoall_setup first");
  DeviceGuard g(ctx_->device());
  HandleBlob h;
  std::memset(&h, 0, sizeof h);
  h.magic = kBlobMagic;
  h.rank = rank_;
  h.device = ctx_->device();
  h.pid = (int)getpid();
  cuda_check(cudaIpcGetMemHandle(&h.recv, recv_), "cudaIpcGetMemHandle");
  cuda_check(cudaIpcGetMemHandle(&h.grad, grad_), "cudaIpcGetMemHandle");
  cuda_check(cudaIpcGetMemHandle(&h.flags, flags_), "cudaIpcGetMemHandle");
  std::memset(blob, 0, AS_HANDLE_BYTES);
  std::memcpy(blob, &h, sizeof h);
  if (nbytes) *nbytes = (int64_t)sizeof h;
}

void ShardComm::open(const void* all) {
  if (!setup_) fail(AS_STATE, "as_alltoall_open: call as_alltoall_setup first");
  if (open_) fail(AS_STATE, "as_alltoall_open: already open");
  DeviceGuard g(ctx_->device());
  const unsigned char* p = static_cast<const unsigned char*>(all);
  for (int q = 0; q < world_; ++q) {
    HandleBlob h;
    std::memcpy(&h, p + (size_t)AS_HANDLE_BYTES * q, sizeof h);
    if (h.magic != kBlobMagic || h.rank != q)
      fail(AS_CONFIG, "as_alltoall_open: blob " + std::to_string(q) + " is not rank " + std::to_string(q) + "'s handle");
    if (q == rank_) {
      peer_recv_[q] = recv_;
      peer_grad_[q] = grad_;
      peer_flags_[q] = flags_;
      continue;
    }
    if (h.pid == (int)getpid())
      fail(AS_CONFIG, "as_alltoall_open: ranks " + std::to_string(rank_) + " and " + std::to_string(q) +
                          " share a process (one process per GPU)");
    void* r = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&r, h.recv, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle (recv)");
    peer_recv_[q] = static_cast<float*>(r);
    cuda_check(cudaIpcOpenMemHandle(&r, h.grad, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle (grad)");
    peer_grad_[q] = static_cast<float*>(r);
    cuda_check(cudaIpcOpenMemHandle(&r, h.flags, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle (flags)");
    peer_flags_[q] = static_cast<unsigned long long*>(r);
    opened_[q] = true;
  }
  open_ = true;
  if (!(mode_ & AS_XCHG_FWD_NCCL)) {
    // the forward's epilogues store into owner q's block of THIS shard
    float* bases[kMaxPeers];
    for (int q = 0; q < world_; ++q) {
      const int64_t rows_q = start_[q + 1] - start_[q];
      bases[q] = peer_recv_[q] + rows_q * col_[rank_];
    }
    ctx_->set_peer_outputs(world_, bases, start_.data());
  }
}

void ShardComm::require_open(const char* what) const {
  if (!open_) fail(AS_STATE, std::string(what) + ": the exchange is not set up (as_alltoall_setup / as_alltoall_open)");
}

void ShardComm::check_async() {
  if (*h_err_)
    fail(AS_NCCL, "peer barrier timed out (a rank did not arrive within 60 s); the exchange is broken");
  if (comm_) {
    ncclResult_t r = ncclSuccess;
    nccl_check(nccl().CommGetAsyncError(comm_, &r), "ncclCommGetAsyncError");
    if (r != ncclSuccess && r != ncclInProgress)
      fail(AS_NCCL, std::string("NCCL communicator error: ") + nccl().GetErrorString(r));
  }
}

void ShardComm::barrier(cudaStream_t s) {
  if (host_fn_) {
    // ranks on one device: nothing guarantees that two processes' kernels run
    // at the same time, so no kernel may wait on another rank. Our peer
    // stores / pushes complete with the stream; the host barrier then orders
    // every rank's completed writes before anyone's next launch.
    cuda_check(cudaStreamSynchronize(s), "host barrier: drain");
    if (host_fn_(host_user_) != 0) fail(AS_NCCL, "host barrier callback failed; the exchange is broken");
    return;
  }
  BarrierFlags f;
  std::memset(&f, 0, sizeof f);
  for (int q = 0; q < world_; ++q) f.peer[q] = peer_flags_[q];
  f.mine = flags_;
  ++epoch_;
  peer_barrier_kernel<<<1, 32, 0, s>>>(f, rank_, world_, epoch_, err_);
  cuda_check(cudaGetLastError(), "peer_barrier_kernel");
  cuda_check(cudaMemcpyAsync(h_err_, err_, sizeof(int), cudaMemcpyDeviceToHost, s), "barrier error D2H");
  ++launches_;
}

void ShardComm::timed(int which, cudaStream_t s, bool begin) {
  if (!ctx_->profiling()) return;
  if (begin) {
    cuda_check(cudaEventRecord(ev_[2 * which], s), "event");
  } else {
    cuda_check(cudaEventRecord(ev_[2 * which + 1], s), "event");
    pending_[which] = true;
  }
}

void ShardComm::collect() {
  for (int w = 0; w < 2; ++w)
    if (pending_[w]) {
      float x = 0.f;
      cuda_check(cudaEventSynchronize(ev_[2 * w + 1]), "event sync");
      cuda_check(cudaEventElapsedTime(&x, ev_[2 * w], ev_[2 * w + 1]), "elapsed");
      ms_[w] += x;
      pending_[w] = false;
    }
}

void ShardComm::forward(cudaStream_t s) {
  require_open("as_forward_sharded");
  check_async();
  DeviceGuard g(ctx_->device());
  collect();
  const int64_t SDr = dims_[rank_];
  if (mode_ & AS_XCHG_FWD_NCCL) {
    ctx_->forward(ctx_->pooled(), nullptr, s);
    timed(0, s, true);
    const NcclApi& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < world_; ++q) {
      const int64_t rq = start_[q + 1] - start_[q];
      if (rq * SDr > 0)
        nccl_check(N.Send(ctx_->pooled() + start_[q] * SDr, rq * SDr, ncclFloat32, q, comm_, s), "ncclSend");
      if (rows_ * dims_[q] > 0)
        nccl_check(N.Recv(recv_ + rows_ * col_[q], rows_ * dims_[q], ncclFloat32, q, comm_, s), "ncclRecv");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
    timed(0, s, false);
  } else {
    ctx_->forward(nullptr, nullptr, s);  // epilogues store into the owners' receive blocks
    timed(0, s, true);
    barrier(s);
    timed(0, s, false);
  }
}

void ShardComm::backward(const float* grad_recv, float lr, float eps, cudaStream_t s) {
  require_open("as_backward_sharded");
  check_async();
  DeviceGuard g(ctx_->device());
  const float* src = grad_recv ? grad_recv : recv_;
  const int64_t SDr = dims_[rank_];
  timed(1, s, true);
  if (mode_ & AS_XCHG_BWD_NCCL) {
    const NcclApi& N = nccl();
    nccl_check(N.GroupStart(), "ncclGroupStart");
    for (int k = 0; k < world_; ++k) {
      if (rows_ * dims_[k] > 0)
        nccl_check(N.Send(src + rows_ * col_[k], rows_ * dims_[k], ncclFloat32, k, comm_, s), "ncclSend");
      const int64_t rq = start_[k + 1] - start_[k];
      if (rq * SDr > 0)
        nccl_check(N.Recv(grad_ + start_[k] * SDr, rq * SDr, ncclFloat32, k, comm_, s), "ncclRecv");
    }
    nccl_check(N.GroupEnd(), "ncclGroupEnd");
  } else {
    // push our rows of every shard's gradient into that shard's owner
    for (int k = 0; k < world_; ++k)
      if (rows_ * dims_[k] > 0)
        cuda_check(cudaMemcpyAsync(peer_grad_[k] + start_[rank_] * dims_[k], src + rows_ * col_[k],
                                   sizeof(float) * rows_ * dims_[k], cudaMemcpyDefault, s),
                   "gradient push");
    barrier(s);
  }
  timed(1, s, false);
  ctx_->backward(grad_, lr, eps, s);
}

void ShardComm::step(float lr, float eps, double* loss_host, cudaStream_t s) {
  forward(s);
  DeviceGuard g(ctx_->device());
  if (loss_host) {
    cuda_check(cudaMemsetAsync(loss_, 0, sizeof(double), s), "loss reset");
    const long long n = rows_ * col_[world_];
    if (n % 4) fail(AS_SHAPE, "as_step_sharded: receive buffer must hold a multiple of 4 floats");
    int sms = 148;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx_->device()), "SM count");
    half_sumsq_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>((n / 4 + 255) / 256, 4LL * sms)), 256, 0, s>>>(
        reinterpret_cast<const float4*>(recv_), n / 4, loss_);
    cuda_check(cudaGetLastError(), "half_sumsq_kernel");
    ++launches_;
  }
  backward(nullptr, lr, eps, s);
  if (loss_host) {
    cuda_check(cudaMemcpyAsync(h_loss_, loss_, sizeof(double), cudaMemcpyDeviceToHost, s), "loss D2H");
    cuda_check(cudaStreamSynchronize(s), "step sync");
    check_async();
    *loss_host = *h_loss_;
  }
}

void ShardComm::info(as_comm_info* o) const {
  std::memset(o, 0, sizeof *o);
  o->rank = rank_;
  o->world = world_;
  o->mode = mode_;
  o->has_nccl = comm_ != nullptr;
  o->recv_rows = rows_;
  o->recv_cols = col_.empty() ? 0 : col_[world_];
  o->recv = recv_;
  o->grad = grad_;
  if (setup_) {
    const int64_t B = ctx_->batch();
    o->bytes_sent_fwd = 4 * (B - rows_) * dims_[rank_];
    o->bytes_sent_bwd = 4 * rows_ * (col_[world_] - dims_[rank_]);
  }
}

void ShardComm::profile_read(double* ms2, bool reset) {
  DeviceGuard g(ctx_->device());
  collect();
  ms2[0] = ms_[0];
  ms2[1] = ms_[1];
  if (reset) ms_[0] = ms_[1] = 0.0;
}

// ---- input-side exchange of the sparse features (KJT all-to-all) -------------
// before the forward, every device sends the indices of ITS
// mini-batch to the owners of the tables. Wire format from rank r to owner q:
// one int32 block [lengths of q's tables for r's rows, table-major][their
// indices, table-major]. The owner assembles its tables' streams over the
// whole batch (sources in rank = sample order) straight into the staging slot
// of its context: rebased int32 offsets and int32 rows.
namespace {
// counts[j * G + r] = sum of source r's lengths of table j
__global__ void kjt_count_kernel(const int* recv, const long long* src_base, const long long* src_rows, int T, int G,
                                 long long* counts) {
  const int j = blockIdx.x, r = blockIdx.y;
  const int* lens = recv + src_base[r] + (long long)j * src_rows[r];
  long long sum = 0;
  for (long long i = threadIdx.x; i < src_rows[r]; i += blockDim.x) sum += lens[i];
  for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __shared__ long long ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    counts[(long long)j * G + r] = t;
  }
}
struct KjtAssemble {
  const int* recv;
  const long long* src_base;  // [G] start of source r's block in recv
  const long long* src_rows;  // [G] rows of source r
  const long long* row_start; // [G] first sample of source r
  const long long* seg;       // [T*G] offset of (j, r)'s indices inside r's index part
  const long long* dst;       // [T*G] element offset of (j, r) inside table j (sum of earlier sources)
  const long long* cnt;       // [T*G]
  const DevTable* tabs;       // slot layout (idx_off)
  int* idx32;
  int* off32;
  int T, G;
  long long B, L;
};
// CTA per (table j, source r): copy the indices, write the rebased offsets of
// r's rows (exclusive scan of the lengths in 1024-row pieces)
__global__ void __launch_bounds__(1024) kjt_assemble_kernel(KjtAssemble a) {
  const int j = blockIdx.x, r = blockIdx.y;
  const long long k = (long long)j * a.G + r;
  const long long rows = a.src_rows[r];
  const int* lens = a.recv + a.src_base[r] + (long long)j * rows;
  const int* src = a.recv + a.src_base[r] + (long long)a.T * rows + a.seg[k];
  const long long base = a.tabs[j].idx_off + a.dst[k];
  int* dst = a.idx32 + base;
  for (long long i = threadIdx.x; i < a.cnt[k]; i += blockDim.x) dst[i] = src[i];
  __shared__ long long ws[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int* off = a.off32 + (long long)j * a.B + a.row_start[r];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long i0 = 0; i0 < rows; i0 += blockDim.x) {
    const long long i = i0 + threadIdx.x;
    const long long v = i < rows ? lens[i] : 0;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    long long pre = carry;
    for (int q = 0; q < w; ++q) pre += ws[q];
    if (i < rows) off[i] = (int)(base + pre + x - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = pre + x;
    __syncthreads();
  }
  if (j == a.T - 1 && r == a.G - 1 && threadIdx.x == 0) a.off32[(long long)a.T * a.B] = (int)a.L;
}
}  // namespace

void ShardComm::load_exchanged(int n_all, const as_table_spec* all, const int32_t* owner,
                               const int64_t* const* loff, const int64_t* const* lidx, cudaStream_t s) {
  if (!setup_) fail(AS_STATE, "as_load_streams_exchanged: call as_alltoall_setup first (the sample split)");
  if (!comm_) fail(AS_STATE, "as_load_streams_exchanged: needs an NCCL communicator (as_comm_init with an id)");
  const int G = world_;
  const int64_t rows = rows_;  // this rank's samples
  // this rank's tables in task order must be the ctx's tables
  std::vector<int> mine;
  for (int t = 0; t < n_all; ++t) {
    if (owner[t] < 0 || owner[t] >= G)
      fail(AS_CONFIG, "as_load_streams_exchanged: table " + std::to_string(all[t].id) + " has owner " +
                          std::to_string(owner[t]) + " outside [0, " + std::to_string(G) + ")");
    if (owner[t] == rank_) mine.push_back(t);
  }
  if ((int)mine.size() != ctx_->n_tables())
    fail(AS_SHAPE, "as_load_streams_exchanged: rank " + std::to_string(rank_) + " owns " + std::to_string(mine.size()) +
                       " tables, its context has " + std::to_string(ctx_->n_tables()));
  for (size_t i = 0; i < mine.size(); ++i)
    if (ctx_->table_id(static_cast<int>(i)) != all[mine[i]].id)
      fail(AS_SHAPE, "as_load_streams_exchanged: context table " + std::to_string(i) + " is id " +
                         std::to_string(ctx_->table_id(static_cast<int>(i))) + ", the plan's is " +
                         std::to_string(all[mine[i]].id));
  // ---- sender: validate this rank's mini-batch (load_workload's checks and
  // messages, workload_io.hpp:216-241) and pack one block per owner ----
  std::string err;
  as_status err_code = AS_OK;
  std::vector<int64_t> send_n(G, 0), send_off(G + 1, 0);
  for (int t = 0; t < n_all && err.empty(); ++t) {
    const int64_t* o = loff[t];
    const std::string where = "table " + std::to_string(all[t].id);
    if (o[0] != 0) err = where + ": offsets must start at 0, got " + std::to_string(o[0]), err_code = AS_OFFSET;
    for (int64_t q = 1; q <= rows && err.empty(); ++q)
      if (o[q] < o[q - 1]) err = where + ": offsets must be nondecreasing at entry " + std::to_string(q), err_code = AS_OFFSET;
    for (int64_t j = 0; j < (err.empty() ? o[rows] : 0); ++j)
      if (lidx[t][j] < 0 || lidx[t][j] >= all[t].hash_size) {
        err = where + ": index " + std::to_string(lidx[t][j]) + " out of range [0, " + std::to_string(all[t].hash_size) + ")";
        err_code = AS_INDEX;
        break;
      }
    if (err.empty()) send_n[owner[t]] += rows + o[rows];
  }
  for (int q = 0; q < G; ++q) send_off[q + 1] = send_off[q] + send_n[q];
  // ---- 1: block sizes and status, all-to-all of one int64 pair per rank pair ----
  std::vector<long long> meta(2 * G), rmeta(2 * G);
  for (int q = 0; q < G; ++q) {
    meta[2 * q] = err.empty() ? send_n[q] : -1;
    meta[2 * q + 1] = err.empty() ? 0 : err_code;
  }
  grow(&kjt_meta_, &kjt_meta_cap_, 4 * G * sizeof(long long));
  long long* dmeta = static_cast<long long*>(kjt_meta_);
  cuda_check(cudaMemcpyAsync(dmeta, meta.data(), 2 * G * sizeof(long long), cudaMemcpyHostToDevice, s), "kjt meta H2D");
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < G; ++q) {
    nccl_check(nccl().Send(dmeta + 2 * q, 2, ncclInt64, q, comm_, s), "ncclSend");
    nccl_check(nccl().Recv(dmeta + 2 * G + 2 * q, 2, ncclInt64, q, comm_, s), "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  cuda_check(cudaMemcpyAsync(rmeta.data(), dmeta + 2 * G, 2 * G * sizeof(long long), cudaMemcpyDeviceToHost, s),
             "kjt meta D2H");
  cuda_check(cudaStreamSynchronize(s), "kjt meta");
  check_async();
  if (!err.empty()) fail(err_code, "as_load_streams_exchanged: rank " + std::to_string(rank_) + ": " + err);
  for (int r = 0; r < G; ++r)
    if (rmeta[2 * r] < 0)
      fail(static_cast<as_status>(rmeta[2 * r + 1]),
           "as_load_streams_exchanged: rank " + std::to_string(r) + "'s mini-batch failed validation");
  // ---- 2: pack (pinned) and exchange the blocks ----
  std::vector<int64_t> recv_off(G + 1, 0), src_rows(G);
  for (int r = 0; r < G; ++r) {
    recv_off[r + 1] = recv_off[r] + rmeta[2 * r];
    src_rows[r] = start_[r + 1] - start_[r];
  }
  grow_host(&kjt_h_, &kjt_h_cap_, std::max<int64_t>(1, send_off[G]) * sizeof(int));
  int* h = static_cast<int*>(kjt_h_);
  {
    std::vector<int64_t> lpos(G), ipos(G);
    std::vector<int64_t> tq(G, 0);
    for (int t = 0; t < n_all; ++t) ++tq[owner[t]];
    for (int q = 0; q < G; ++q) {
      lpos[q] = send_off[q];
      ipos[q] = send_off[q] + tq[q] * rows;
    }
    for (int t = 0; t < n_all; ++t) {
      const int q = owner[t];
      const int64_t* o = loff[t];
      for (int64_t i = 0; i < rows; ++i) h[lpos[q] + i] = static_cast<int>(o[i + 1] - o[i]);
      lpos[q] += rows;
      for (int64_t j = 0; j < o[rows]; ++j) h[ipos[q] + j] = static_cast<int>(lidx[t][j]);
      ipos[q] += o[rows];
    }
  }
  grow(&kjt_send_, &kjt_send_cap_, std::max<int64_t>(1, send_off[G]) * sizeof(int));
  grow(&kjt_recv_, &kjt_recv_cap_, std::max<int64_t>(1, recv_off[G]) * sizeof(int));
  int* dsend = static_cast<int*>(kjt_send_);
  int* drecv = static_cast<int*>(kjt_recv_);
  cuda_check(cudaMemcpyAsync(dsend, h, send_off[G] * sizeof(int), cudaMemcpyHostToDevice, s), "kjt H2D");
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int q = 0; q < G; ++q) {
    if (send_n[q] > 0) nccl_check(nccl().Send(dsend + send_off[q], send_n[q], ncclInt32, q, comm_, s), "ncclSend");
    if (rmeta[2 * q] > 0) nccl_check(nccl().Recv(drecv + recv_off[q], rmeta[2 * q], ncclInt32, q, comm_, s), "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  // ---- 3: per (table, source) counts -> the batch layout on the host ----
  const int T = ctx_->n_tables();
  std::vector<long long> geo(4 * G + 3 * (size_t)T * G);  // src_base | src_rows | row_start | cnt... staged below
  long long* g_base = geo.data();
  long long* g_rows = g_base + G;
  long long* g_start = g_rows + G;
  for (int r = 0; r < G; ++r) {
    g_base[r] = recv_off[r];
    g_rows[r] = src_rows[r];
    g_start[r] = start_[r];
  }
  grow(&kjt_geo_, &kjt_geo_cap_, geo.size() * sizeof(long long));
  long long* dgeo = static_cast<long long*>(kjt_geo_);
  long long* dcnt = dgeo + 4 * G;
  cuda_check(cudaMemcpyAsync(dgeo, geo.data(), 3 * G * sizeof(long long), cudaMemcpyHostToDevice, s), "kjt geo H2D");
  std::vector<long long> cnt((size_t)T * G, 0);
  if (T > 0) {
    kjt_count_kernel<<<dim3(T, G), 256, 0, s>>>(drecv, dgeo, dgeo + G, T, G, dcnt);
    cuda_check(cudaGetLastError(), "kjt_count_kernel");
    cuda_check(cudaMemcpyAsync(cnt.data(), dcnt, cnt.size() * sizeof(long long), cudaMemcpyDeviceToHost, s), "kjt counts");
  }
  cuda_check(cudaStreamSynchronize(s), "kjt exchange");
  check_async();
  std::vector<int64_t> n_idx(T, 0);
  long long* seg = dcnt + (size_t)T * G;
  std::vector<long long> hseg((size_t)T * G), hdst((size_t)T * G);
  for (int r = 0; r < G; ++r) {
    long long acc = 0;
    for (int j = 0; j < T; ++j) {
      hseg[(size_t)j * G + r] = acc;
      acc += cnt[(size_t)j * G + r];
    }
  }
  long long L = 0;
  for (int j = 0; j < T; ++j) {
    long long acc = 0;
    for (int r = 0; r < G; ++r) {
      hdst[(size_t)j * G + r] = acc;
      acc += cnt[(size_t)j * G + r];
    }
    n_idx[j] = acc;
    L += acc;
  }
  cuda_check(cudaMemcpyAsync(seg, hseg.data(), hseg.size() * sizeof(long long), cudaMemcpyHostToDevice, s), "kjt seg");
  cuda_check(cudaMemcpyAsync(seg + (size_t)T * G, hdst.data(), hdst.size() * sizeof(long long), cudaMemcpyHostToDevice, s),
             "kjt dst");
  cuda_check(cudaEventRecord(ev_kjt_, s), "kjt ready");
  // ---- 4: assemble into the context's staging slot, commit ----
  const int64_t B = ctx_->batch();
  ctx_->stage_device(n_idx.data(), [&](int* idx32, int* off32, const DevTable* tabs, cudaStream_t cs) {
    cuda_check(cudaStreamWaitEvent(cs, ev_kjt_, 0), "kjt wait");
    if (T == 0) return;
    // the slot's host-built layout (idx_off per table) goes with the kernel
    grow(&kjt_tabs_, &kjt_tabs_cap_, sizeof(DevTable) * T);
    cuda_check(cudaMemcpyAsync(kjt_tabs_, tabs, sizeof(DevTable) * T, cudaMemcpyHostToDevice, cs), "kjt tabs");
    KjtAssemble a;
    a.recv = drecv;
    a.src_base = dgeo;
    a.src_rows = dgeo + G;
    a.row_start = dgeo + 2 * G;
    a.cnt = dcnt;
    a.seg = seg;
    a.dst = seg + (size_t)T * G;
    a.tabs = static_cast<const DevTable*>(kjt_tabs_);
    a.idx32 = idx32;
    a.off32 = off32;
    a.T = T;
    a.G = G;
    a.B = B;
    a.L = L;
    kjt_assemble_kernel<<<dim3(T, G), 1024, 0, cs>>>(a);
    cuda_check(cudaGetLastError(), "kjt_assemble_kernel");
  });
  ctx_->commit(s);
  launches_ += 2;
}

void ShardComm::grow(void** p, int64_t* cap, int64_t bytes) {
  if (bytes <= *cap) return;
  if (*p) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    cudaFree(*p);
  }
  *cap = bytes + bytes / 8 + 256;
  cuda_check(cudaMalloc(p, static_cast<size_t>(*cap)), "cudaMalloc");
}

void ShardComm::grow_host(void** p, int64_t* cap, int64_t bytes) {
  if (bytes <= *cap) return;
  if (*p) {
    cuda_check(cudaDeviceSynchronize(), "grow sync");
    cudaFreeHost(*p);
  }
  *cap = bytes + bytes / 8 + 256;
  cuda_check(cudaHostAlloc(p, static_cast<size_t>(*cap), cudaHostAllocDefault), "cudaHostAlloc");
}

}  // namespace asb
