/*
 * autoshard_b200.h — C-ABI of the B200-native AutoShard embedding-bag hot path.
 *
 * This is the drop-in boundary. Everything is plain C: POD
 * structs, raw pointers and sizes, status codes, no exceptions and no torch
 * types. The C++ header autoshard_b200.hpp wraps it back into the reference's
 * own C++ shapes (autoshard::gpu::measure_plan etc.).
 *
 * Each entry point names the reference interface it replaces
 * (paths under /root/reference/proj/include/autoshard/).
 *
 * Threading: an as_ctx is bound to one CUDA device and is not thread-safe;
 * use one host thread (or process) per device. Host-side generator / planner
 * calls are pure and reentrant. Errors: every call returns an as_status; the
 * message of the last failure on the calling thread is as_last_error().
 */
#ifndef AUTOSHARD_B200_H
#define AUTOSHARD_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define AS_API __attribute__((visibility("default")))
#else
#define AS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors the exception taxonomy of common.hpp:15-50 (+ device failures). */
typedef enum as_status {
  AS_OK = 0,
  AS_CONFIG = 1,     /* ConfigError */
  AS_PARSE = 2,      /* ParseError */
  AS_OFFSET = 3,     /* OffsetError (ParseError subclass) */
  AS_INDEX = 4,      /* IndexError (ParseError subclass) */
  AS_INFEASIBLE = 5, /* InfeasibleError */
  AS_SHAPE = 6,      /* ShapeError */
  AS_LOOKUP = 7,     /* LookupError */
  AS_GUARD = 8,      /* GuardError */
  AS_STATE = 9,      /* StateError */
  AS_CUDA = 10,      /* CUDA runtime / launch failure */
  AS_NCCL = 11       /* collective failure */
} as_status;

/* TableDesc, tables.hpp:24-38. Same field order/meaning. */
typedef struct as_table_spec {
  int32_t id;
  int32_t dim;              /* embedding length; device path needs dim % 4 == 0, 4..1024 */
  int64_t hash_size;        /* rows */
  double pooling_mean;      /* declared mean lookups per query */
  double access_ratio;      /* fraction of rows ever accessed */
  int32_t bytes_per_param;  /* planning size only (size_bytes); device stores fp32 */
  int32_t _pad;
} as_table_spec;

/* GeneratorConfig, tables.hpp:149-174. */
typedef struct as_generator_config {
  double hash_size_min, hash_size_max;
  double pooling_mean_target, pooling_shape, pooling_cap;
  const int32_t* dim_choices;
  int32_t n_dim_choices;
  double access_ratio_min, access_ratio_max;
  int32_t bytes_per_param;
} as_generator_config;

/* BenchConfig, simcost.hpp:163-171, plus the GPU-only knobs. */
typedef struct as_bench_config {
  int32_t warmup;   /* W (default 5) */
  int32_t measure;  /* B (default 10) */
  int32_t trim;     /* R (default 2); needs measure - 2*trim >= 1 */
  int32_t flush_l2; /* overwrite a buffer of 2x L2 before each measured run */
  uint64_t seed;    /* weight-init seed of the measured contexts */
  float lr, eps;    /* row-wise Adagrad hyper-parameters of the measured step */
} as_bench_config;

typedef struct as_workload as_workload; /* host-side Workload (tables.hpp:43-60) */
typedef struct as_ctx as_ctx;           /* one device, one shard of tables */

AS_API const char* as_version(void);
AS_API const char* as_last_error(void);

/* ---------------------------------------------------------------------- */
/* L1 — synthetic tables and streams (tables.hpp, workload_io.hpp)        */
/* ---------------------------------------------------------------------- */

/* GeneratorConfig{} defaults; dim_choices points at static {16, 32}. */
AS_API void as_generator_config_default(as_generator_config* cfg);

/* generate_pool, tables.hpp:178-200 (bit-exact). out has n entries. */
AS_API as_status as_generate_pool(uint64_t seed, int32_t n_tables, const as_generator_config* cfg,
                                  as_table_spec* out);

/* generate_workload, tables.hpp:237-288 (bit-exact; tables processed in
 * parallel on n_threads host threads, 0 = all cores). */
AS_API as_status as_generate_workload(uint64_t seed, const as_table_spec* tables, int32_t n_tables,
                                      int64_t batch_size, double zipf_exponent, int32_t n_threads,
                                      as_workload** out);

/* Workload::find (tables.hpp:53-59) and accessors; pointers owned by wl. */
AS_API int64_t as_workload_batch_size(const as_workload* wl);
AS_API int32_t as_workload_num_tables(const as_workload* wl);
AS_API as_status as_workload_stream(const as_workload* wl, int32_t i, int32_t* table_id,
                                    const int64_t** offsets, const int64_t** indices,
                                    int64_t* n_indices);
AS_API as_status as_workload_find(const as_workload* wl, int32_t table_id, int32_t* position);
/* Build a workload from caller arrays (copied). offsets[i] has batch+1 entries. */
AS_API as_status as_workload_from_arrays(int64_t batch_size, int32_t n_tables,
                                         const int32_t* table_ids, const int64_t* const* offsets,
                                         const int64_t* const* indices, const int64_t* n_indices,
                                         as_workload** out);
/* Page-lock the stream buffers (cudaHostRegister) so device loads run at full
 * PCIe rate; undone by as_workload_destroy. */
AS_API as_status as_workload_pin(as_workload* wl);
AS_API void as_workload_destroy(as_workload* wl);

/* save_workload / load_workload (workload_io.hpp:151-245): same file format,
 * same validation and error classes (OffsetError / IndexError naming the table). */
AS_API as_status as_workload_save(const as_workload* wl, const as_table_spec* tables,
                                  const char* path);
/* tables_out: capacity max_tables; n_tables receives the count. */
AS_API as_status as_workload_load(const char* path, as_workload** out, as_table_spec* tables_out,
                                  int32_t max_tables, int32_t* n_tables);
AS_API as_status as_pool_save(const as_table_spec* tables, int32_t n, const char* path);
AS_API as_status as_pool_load(const char* path, as_table_spec* tables_out, int32_t max_tables,
                              int32_t* n_tables);

/* fingerprint(pool) / fingerprint(ShardingTask), tables.hpp:417-441. */
AS_API uint64_t as_fingerprint_pool(const as_table_spec* tables, int32_t n);
AS_API uint64_t as_fingerprint_task(const as_table_spec* tables, int32_t n, int32_t num_shards,
                                    const int64_t* mem_budget);

/* ---------------------------------------------------------------------- */
/* L3 — plans (tables.hpp:63-143, planners.hpp, SPEC.md:291 plan file)    */
/* ---------------------------------------------------------------------- */

/* kind: 0 size-greedy, 1 dim-greedy, 2 lookup-greedy (HeuristicKind, planners.hpp:20). */
AS_API as_status as_heuristic_cost(const as_table_spec* t, int32_t kind, double* cost);
AS_API as_status as_greedy_shard(const as_table_spec* tables, int32_t n, int32_t num_shards,
                                 const int64_t* mem_budget, int32_t kind, int32_t* assignment);
AS_API as_status as_random_shard(const as_table_spec* tables, int32_t n, int32_t num_shards,
                                 const int64_t* mem_budget, uint64_t seed, int32_t* assignment);
/* ShardingPlan::validate / mem_used / feasible. */
AS_API as_status as_plan_validate(int32_t n, int32_t num_shards, const int32_t* assignment);
AS_API as_status as_plan_mem_used(const as_table_spec* tables, int32_t n, int32_t num_shards,
                                  const int32_t* assignment, int64_t* used);
AS_API as_status as_degree_of_balance(const double* costs, int32_t n, double* balance);
/* Plan file: "autoshard-plan 1", task fingerprint, assignment, optional costs. */
AS_API as_status as_plan_save(const char* path, const as_table_spec* tables, int32_t n,
                              int32_t num_shards, const int64_t* mem_budget,
                              const int32_t* assignment, const double* costs_or_null);
/* Validates the fingerprint against (tables, budgets); costs_out may be NULL. */
AS_API as_status as_plan_load(const char* path, const as_table_spec* tables, int32_t n,
                              int32_t num_shards, const int64_t* mem_budget, int32_t* assignment,
                              double* costs_out, int32_t* has_costs);

/* ---------------------------------------------------------------------- */
/* L2 — the device hot path (replaces SIM-1/SIM-2, simcost.hpp:60-115)    */
/* ---------------------------------------------------------------------- */

/* One shard on one device: allocates fp32 tables [hash, dim] (counter-hash
 * init from weight_seed), fp32 row-wise momentum (0), and
 * workspaces for batch_size. Tables keep the given order; their pooled
 * columns are laid out in that order. n_tables may be 0 (empty shard). */
AS_API as_status as_create(int32_t device, const as_table_spec* tables, int32_t n_tables,
                           int64_t batch_size, uint64_t weight_seed, as_ctx** out);

/* as_create with flags. AS_WEIGHTS_FP16: tables stored as IEEE fp16
 * (bytes_per_param = 2, tables.hpp:30) — the
 * forward gathers half rows and accumulates in fp32, the row-wise Adagrad
 * update is computed in fp32 and rounded to nearest fp16; momentum, pooled
 * rows and gradients stay fp32. Unknown flags: AS_CONFIG. */
#define AS_WEIGHTS_FP16 1
AS_API as_status as_create_ex(int32_t device, const as_table_spec* tables, int32_t n_tables,
                              int64_t batch_size, uint64_t weight_seed, int32_t flags, as_ctx** out);
AS_API as_status as_destroy(as_ctx* ctx);

/* A shard over n_tables of parent's tables (positions into parent's table
 * order, each at most once; their pooled columns in the given order) that
 * works on parent's weight and momentum storage — nothing is copied or
 * initialised, steps through it update parent's rows. Its own workspaces and
 * batch. The cost hook of an RL environment measures candidate shards this
 * way without re-creating the tables (rl.hpp:161-167).
 * parent must outlive the subset. AS_CONFIG for a bad or repeated position. */
AS_API as_status as_create_subset(const as_ctx* parent, const int32_t* positions, int32_t n_tables,
                                  as_ctx** out);
/* Point a subset context at another subset of the same parent, keeping its
 * streams, events and grow-only workspaces (cheap: the measured-cost hook
 * times thousands of candidate shards through one context). Load streams
 * again afterwards. AS_STATE if ctx is not a subset or a batch is staged. */
AS_API as_status as_retarget_subset(as_ctx* ctx, const int32_t* positions, int32_t n_tables);

/* Load one batch of streams (host int64 CSR per table, ctx table order,
 * TableStream layout tables.hpp:43-47). Host memory is borrowed for the call
 * only. Validation reproduces load_workload's checks (workload_io.hpp:216-241)
 * on the library's host staging threads while they narrow the streams to the
 * device format (opt-in: part of the index pieces narrowed and checked on the
 * device, ASB_RAW_EIGHTHS) and reports OffsetError / IndexError naming the
 * table, the same first error either way.
 * stream: a cudaStream_t (NULL = legacy default). Synchronises. */
AS_API as_status as_load_streams(as_ctx* ctx, const int64_t* const* offsets,
                                 const int64_t* const* indices, const int64_t* n_indices,
                                 void* stream);
/* Same, picking the ctx's tables from a workload by id (LookupError if absent). */
AS_API as_status as_load_workload(as_ctx* ctx, const as_workload* wl, void* stream);

/* Asynchronous, double-buffered loading for training loops: stage batch i+1
 * while batch i computes, then commit it. as_stage_* returns immediately; a
 * background job on the library's host thread pool narrows the int64 CSR to
 * the device format (int32 global rows, rebased int32 offsets) into a pinned
 * slot buffer, validating it like load_workload (workload_io.hpp:216-241),
 * and enqueues each finished piece's host->device copy on the context's copy
 * stream. The caller's host arrays must stay valid and unmodified until the
 * matching as_commit_staged returns. as_commit_staged joins the job, reports
 * the batch's first OffsetError / IndexError (table, check, entry order),
 * and makes the slot the current batch (the compute `stream` waits for its
 * copy). Two slots: staging a third batch before a commit returns AS_STATE.
 * as_check_batch is kept for callers that separate commit and error checks
 * (validation completes at commit). as_load_streams = stage + commit. */
AS_API as_status as_stage_streams(as_ctx* ctx, const int64_t* const* offsets,
                                  const int64_t* const* indices, const int64_t* n_indices);
AS_API as_status as_stage_workload(as_ctx* ctx, const as_workload* wl);
AS_API as_status as_commit_staged(as_ctx* ctx, void* stream);
AS_API as_status as_check_batch(as_ctx* ctx);

/* K4+K1: pooled[b, col_t + d] = sum_{j in bag (t,b)} W_t[idx_j, d]; empty bag -> 0.
 * out: device [batch, sum_dim] fp32, or NULL for the ctx's own buffer. */
AS_API as_status as_forward(as_ctx* ctx, float* out_or_null, void* stream);

/* Fused forward exchange for table-wise sharding over G GPUs (
 * replaces the pooled-row all-to-all that follows the forward). Once set,
 * as_forward writes pooled row b of every table of this shard to the receive
 * buffer of the sample owner q = b / rows_per_peer, at
 *   peer_bases[q] + (b - q * rows_per_peer) * sum_dim + col_t
 * (peer_bases[q]: a device address valid on this ctx's device — the owner's
 * receive block for this shard, e.g. from torch symmetric memory / CUDA IPC;
 * on another GPU the epilogue's stores go over NVLink), and ignores
 * out_or_null. The caller orders readers after the writers (a barrier after
 * the forward). n_peers = 0 restores the local [batch, sum_dim] output.
 * AS_SHAPE unless n_peers * rows_per_peer == batch; at most 8 peers. */
AS_API as_status as_set_peer_outputs(as_ctx* ctx, int n_peers, float* const* peer_bases, int64_t rows_per_peer);

/* as_set_peer_outputs with UNEVEN sample ranges: peer q owns batch rows
 * [row_start[q], row_start[q+1]) (row_start[0] = 0, row_start[n_peers] = batch,
 * nondecreasing), pooled row b of this shard is stored at
 *   peer_bases[q] + (b - row_start[q]) * sum_dim + col_t. */
AS_API as_status as_set_peer_outputs_v(as_ctx* ctx, int n_peers, float* const* peer_bases,
                                       const int64_t* row_start);

/* K2+K3: sort (row, bag), segment-sum the gradient rows per unique row and
 * apply exact row-wise Adagrad in place:
 *   m_r += |g_r|^2 / dim ;  W_r -= lr * g_r / (sqrt(m_r) + eps).
 * grad: device [batch, sum_dim] fp32, or NULL = the ctx's pooled output
 * (loss = 1/2 |pooled|^2). */
AS_API as_status as_backward_rowwise_adagrad(as_ctx* ctx, const float* grad_or_null, float lr,
                                             float eps, void* stream);

/* One training step on the loaded batch: forward into the ctx buffer, loss
 * 1/2 |pooled|^2 (if loss_out != NULL it is computed and copied to host,
 * which synchronises), backward with grad = pooled. */
AS_API as_status as_step(as_ctx* ctx, float lr, float eps, double* loss_out, void* stream);

/* Micro-benchmark of this shard (simcost.hpp:140-154 on
 * real kernels): W warm-up steps, B measured steps (each after an L2 flush
 * when flush_l2), CUDA-event timed, sorted, R dropped at each end, mean ms. */
AS_API as_status as_measure(as_ctx* ctx, int32_t warmup, int32_t measure, int32_t trim,
                            int32_t flush_l2, float lr, float eps, double* ms_out);

/* measure_plan (simcost.hpp:194-204) on the GPU: for shard k a ctx holding
 * plan's tables is created on devices[k % n_devices], its streams loaded from
 * wl, and as_measure run; costs[k] in ms. Same validation as the reference
 * (ConfigError on a bad plan, LookupError on a table absent from wl). */
AS_API as_status as_measure_plan(const as_table_spec* tables, int32_t n, int32_t num_shards,
                                 const int32_t* assignment, const as_workload* wl,
                                 const int32_t* devices, int32_t n_devices,
                                 const as_bench_config* bench, double* costs);

/* ---------------------------------------------------------------------- */
/* L4 — table-wise sharded step over G processes, one per GPU             */
/*      (SURVEY.md §8e). Replaces the pooled-row          */
/*      all-to-all around the embedding operator.                          */
/* ---------------------------------------------------------------------- */
typedef struct as_comm as_comm;

#define AS_UNIQUE_ID_BYTES 128 /* sizeof(ncclUniqueId) */
#define AS_HANDLE_BYTES 512    /* as_alltoall_handle blob (>= what it writes) */

/* Exchange modes of as_alltoall_setup (bit flags). Without a flag a direction
 * goes over peer memory:
 *   forward  — fused into K4/K1's epilogues: pooled rows are stored straight
 *              into the sample owners' receive buffers (NVLink stores), then a
 *              system-scope release/acquire device barrier;
 *   backward — each gradient block is pushed into its table owner's gradient
 *              buffer by the copy engines (peer memory), then the barrier.
 * With the flag that direction is a grouped ncclSend / ncclRecv all-to-all
 * (needs an NCCL communicator). */
#define AS_XCHG_PEER 0
#define AS_XCHG_FWD_NCCL 1
#define AS_XCHG_BWD_NCCL 2
#define AS_XCHG_NCCL 3

/* ncclGetUniqueId: rank 0 calls it and hands the 128 bytes to every rank.
 * NCCL is loaded at run time (libnccl.so.2; the one torch loaded if present):
 * AS_NCCL when it cannot be loaded. */
AS_API as_status as_comm_unique_id(void* unique_id_out);

/* One rank of a G-rank sharded execution, bound to ctx (this rank's shard of
 * tables on its device). unique_id != NULL: an NCCL communicator of the G ranks
 * (ncclCommInitRank; collective: every rank must call it) — peer-memory
 * handles are then exchanged over it. unique_id == NULL: no NCCL (AS_XCHG_PEER
 * only); the caller moves the handle blobs itself (as_alltoall_handle /
 * as_alltoall_open: all-gather them with MPI, torch.distributed, files ...).
 * 1 <= world <= 8. ctx must outlive the comm. */
AS_API as_status as_comm_init(as_ctx* ctx, const void* unique_id_or_null, int32_t rank, int32_t world,
                              as_comm** out);
AS_API as_status as_comm_destroy(as_comm* comm);

/* Layout of the pooled-row all-to-all: rank k's shard has shard_dims[k] pooled
 * columns (its tables in ctx order); sample owner p holds batch rows
 * [row_start[p], row_start[p+1]) (uneven splits allowed; row_start[0] = 0,
 * row_start[world] = batch). Allocates this rank's receive buffer (world
 * blocks, block k = [rows_p, shard_dims[k]] fp32, in rank order), its gradient
 * buffer [batch, shard_dims[rank]] and the barrier flags. With an NCCL comm it
 * also all-gathers the peer handles (collective), and the exchange is ready;
 * without, call as_alltoall_handle / as_alltoall_open next. AS_SHAPE when the
 * layout does not match the ctx (shard_dims[rank] != sum of its dims, batch). */
AS_API as_status as_alltoall_setup(as_comm* comm, const int64_t* shard_dims, const int64_t* row_start,
                                   int32_t mode);
/* This rank's handle blob (cudaIpc handles of its receive / gradient / flag
 * buffers); *nbytes <= AS_HANDLE_BYTES. */
AS_API as_status as_alltoall_handle(as_comm* comm, void* blob_out, int64_t* nbytes);
/* all_blobs: world blobs of AS_HANDLE_BYTES each, in rank order. Opens the
 * peers' buffers (cudaIpcOpenMemHandle, peer access enabled lazily) and
 * points this ctx's forward at the owners' receive blocks. */
AS_API as_status as_alltoall_open(as_comm* comm, const void* all_blobs);
/* Host-side exchange barrier, for ranks that SHARE one device (functional
 * tests on a 1-GPU box). The device barrier is a kernel that waits for the
 * other ranks' arrival; kernels of different processes on one GPU are not
 * guaranteed to run at the same time, so there it would rely on time-slicing.
 * With fn set, the barrier instead synchronises the stream (this rank's peer
 * stores and pushes are complete) and calls fn(user), which must return 0 once
 * every rank has called it for this barrier (MPI_Barrier, a gloo barrier, a
 * file rendezvous ...), non-zero on failure (-> AS_NCCL). fn == NULL restores
 * the device barrier. */
typedef int32_t (*as_host_barrier_fn)(void* user);
AS_API as_status as_alltoall_host_barrier(as_comm* comm, as_host_barrier_fn fn, void* user);

/* The sharded forward: K4/K1 of this rank's tables with every pooled row
 * delivered to its sample owner, then the exchange barrier (AS_XCHG_PEER) or
 * the NCCL all-to-all; on return (stream order) this rank's receive buffer
 * holds the pooled rows of its samples for ALL tables. */
AS_API as_status as_forward_sharded(as_comm* comm, void* stream);
/* The sharded backward: grad_recv (device, the receive buffer's layout; NULL =
 * the receive buffer itself, i.e. loss 1/2 |recv|^2) goes back to the table
 * owners (inverse all-to-all), then K2/K3 + row-wise Adagrad on this shard. */
AS_API as_status as_backward_sharded(as_comm* comm, const float* grad_recv_or_null, float lr, float eps,
                                     void* stream);
/* as_forward_sharded + loss 1/2 |recv|^2 of this rank's samples (if loss_out:
 * computed on the device and copied to host, which synchronises) +
 * as_backward_sharded(grad = recv). */
AS_API as_status as_step_sharded(as_comm* comm, float lr, float eps, double* loss_out, void* stream);

/* Input-side exchange of the sparse features (KJT all-to-all):
 * every rank passes ITS mini-batch — the streams of its samples
 * [row_start[rank], row_start[rank+1]) for ALL n_all tables of the task, host
 * int64 CSR per table in task order (TableStream layout, offsets over its own
 * rows) — with the task's tables and owner[t] = the rank holding table t
 * (plan.assignment). Each rank validates its own mini-batch with
 * load_workload's checks and messages, the ranks agree on the outcome, the
 * lengths and int32 indices go to the owners over NCCL (grouped send/recv),
 * and every owner assembles its tables' streams over the WHOLE batch (sources
 * in sample order) on the device and loads them into its ctx as
 * as_load_streams would. Collective; needs as_alltoall_setup (the sample
 * split) and an NCCL communicator. AS_SHAPE if the ctx's tables are not this
 * rank's owner[] tables in task order; AS_OFFSET / AS_INDEX name the table
 * (and, on the other ranks, the failing rank). */
AS_API as_status as_load_streams_exchanged(as_comm* comm, int32_t n_all, const as_table_spec* all_tables,
                                           const int32_t* owner, const int64_t* const* local_offsets,
                                           const int64_t* const* local_indices, void* stream);

typedef struct as_comm_info {
  int32_t rank, world, mode, has_nccl;
  int64_t recv_rows;     /* rows_p of this rank */
  int64_t recv_cols;     /* sum_k shard_dims[k] */
  float* recv;           /* device [world blocks of [rows_p, shard_dims[k]]] */
  float* grad;           /* device [batch, shard_dims[rank]] */
  int64_t bytes_sent_fwd;   /* pooled-row bytes this rank sends to OTHER ranks per forward */
  int64_t bytes_sent_bwd;   /* gradient bytes this rank sends to other ranks per backward */
} as_comm_info;
AS_API as_status as_comm_info_get(const as_comm* comm, as_comm_info* info);
/* Per-step exchange timing (CUDA events on the launching stream, when the
 * ctx's profiling is on): ms[0] forward exchange (barrier wait, or the NCCL
 * all-to-all), ms[1] backward exchange; accumulated until reset. */
AS_API as_status as_comm_profile_read(as_comm* comm, double* ms2, int32_t reset);

/* Introspection for hosts that drive collectives themselves. */
typedef struct as_ctx_info {
  int32_t device;
  int32_t n_tables;
  int64_t batch_size;
  int64_t sum_dim;       /* pooled row width */
  int64_t total_rows;    /* sum hash_size */
  int64_t n_lookups;     /* of the loaded batch (0 before a load) */
  int64_t n_chunks;      /* work chunks of the loaded batch */
  int64_t device_bytes;  /* bytes allocated on the device */
  float* pooled;         /* device [batch, sum_dim] */
  float* weights;        /* device, concatenated [hash_t, dim_t] (fp16 if weight_bytes == 2) */
  float* momentum;       /* device [total_rows] */
  int32_t kernels_per_step; /* kernel launches of one as_step */
  int32_t weight_bytes;     /* 4 (fp32) or 2 (AS_WEIGHTS_FP16) */
} as_ctx_info;
AS_API as_status as_ctx_info_get(const as_ctx* ctx, as_ctx_info* info);

/* Per-kernel CUDA-event timing for roofline accounting (bench.py). enable:
 * 0 off, 1 on, 2 on with the K2 sort serialized into the backward (no
 * side-stream overlap) so each phase is timed alone. When enabled, every phase of as_forward / as_backward_rowwise_adagrad records an
 * event pair on the launching stream. as_profile_read synchronises and returns
 * the accumulated ms per phase: [0] bag_expand (K4), [1] forward segment
 * reduce (K1), [2] forward fixup, [3] radix sort (K2), [4] backward segment
 * reduce + Adagrad (K3), [5] backward fixup; *launches = kernels launched. */
#define AS_NUM_PHASES 6
AS_API as_status as_profile_enable(as_ctx* ctx, int32_t enable);
AS_API as_status as_profile_read(as_ctx* ctx, double* ms_per_phase, int64_t* launches, int32_t reset);

/* Cost-model features of the loaded batch, computed on the
 * device from the backward's sorted keys instead of a host hash map:
 * out[t*21 + :] = FeatureVector::raw of extract_features (tables.hpp:344-386):
 * dim, hash_size, observed pooling, size_gb, 17 frequency-bin ratios over the
 * table's distinct rows. Synchronises. */
AS_API as_status as_table_features(as_ctx* ctx, double* out, void* stream);

/* Roofline denominator (bench.py): GB/s of random row gathers of row_bytes
 * (16..512, power of two) over a device buffer of footprint_bytes — an
 * L2-resident footprint measures the L2 gather ceiling of cache-resident
 * workloads, a multi-GB one the HBM gather ceiling. Synchronises. */
AS_API as_status as_probe_gather_bw(int32_t device, int64_t footprint_bytes, int32_t row_bytes, double* gbs);

/* Readbacks for parity (synchronise). */
/* rows: n row ids (table-local) of ctx table position t -> out [n, dim] fp32. */
AS_API as_status as_read_rows(as_ctx* ctx, int32_t t, const int64_t* rows, int64_t n, float* out);
AS_API as_status as_read_momentum(as_ctx* ctx, int32_t t, const int64_t* rows, int64_t n,
                                  float* out);
/* what: 0 pooled [batch, sum_dim] fp32; 1 bag id per lookup int32 [n_lookups];
 *       2 sorted global rows int32 [n_lookups]; 3 sorted bag ids int32;
 *       4 device index array (global rows) int32 [n_lookups]. */
AS_API as_status as_read_buffer(as_ctx* ctx, int32_t what, void* host_out, int64_t nbytes);
/* Overwrite dense table t / momentum from host (tests). */
AS_API as_status as_write_table(as_ctx* ctx, int32_t t, const float* w_or_null,
                                const float* m_or_null);

#ifdef __cplusplus
}
#endif
#endif /* AUTOSHARD_B200_H */
