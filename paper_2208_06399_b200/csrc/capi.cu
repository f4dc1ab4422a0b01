// extern "C" boundary (include/autoshard_b200.h): converts C++ exceptions of
// the host library / device context into as_status codes and a thread-local
// message, mirroring the reference's exception taxonomy (common.hpp:15-50).
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "autoshard_b200.h"
#include "cuda/context.hpp"
#include "cuda/sharded.hpp"
#include "host/host.hpp"

struct as_workload {
  asb::HostWorkload wl;
};
struct as_ctx {
  std::unique_ptr<asb::EmbContext> impl;
};
struct as_comm {
  std::unique_ptr<asb::ShardComm> impl;
};

namespace {
thread_local std::string g_err;

as_status set_err(as_status c, const std::string& m) {
  g_err = m;
  return c;
}

template <class F>
as_status guard(F&& f) {
  try {
    f();
    return AS_OK;
  } catch (const asb::Error& e) {
    return set_err(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return set_err(AS_CONFIG, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(AS_CONFIG, e.what());
  }
}

void need(const void* p, const char* what) {
  if (!p) asb::fail(AS_CONFIG, std::string(what) + " must not be NULL");
}

asb::GenConfig to_cfg(const as_generator_config* c) {
  asb::GenConfig g;
  if (!c) return g;
  g.hash_size_min = c->hash_size_min;
  g.hash_size_max = c->hash_size_max;
  g.pooling_mean_target = c->pooling_mean_target;
  g.pooling_shape = c->pooling_shape;
  g.pooling_cap = c->pooling_cap;
  g.dim_choices.assign(c->dim_choices, c->dim_choices + (c->n_dim_choices > 0 ? c->n_dim_choices : 0));
  g.access_ratio_min = c->access_ratio_min;
  g.access_ratio_max = c->access_ratio_max;
  g.bytes_per_param = c->bytes_per_param;
  return g;
}

const int32_t kDefaultDims[2] = {16, 32};

// Per-table stream pointers of ctx's tables, picked from a workload by id.
struct Picked {
  std::vector<const int64_t*> off, idx;
  std::vector<int64_t> n;
};
Picked pick_streams(asb::EmbContext& ctx, const asb::HostWorkload& wl) {
  const int T = ctx.n_tables();
  Picked p;
  p.off.resize(static_cast<size_t>(T));
  p.idx.resize(static_cast<size_t>(T));
  p.n.resize(static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) {
    const int pos = wl.find(ctx.spec(t).id);
    if (pos < 0)
      asb::fail(AS_LOOKUP, "measure: table " + std::to_string(ctx.spec(t).id) + " absent from workload");
    const auto& st = wl.per_table[static_cast<size_t>(pos)];
    if (static_cast<int64_t>(st.offsets.size()) != wl.batch_size + 1)
      asb::fail(AS_OFFSET, "table " + std::to_string(st.table_id) + ": offsets length " +
                               std::to_string(st.offsets.size()) + " != batch_size + 1");
    p.off[t] = st.offsets.data();
    p.idx[t] = st.indices.data();
    p.n[t] = static_cast<int64_t>(st.indices.size());
  }
  return p;
}

void load_from_workload(asb::EmbContext& ctx, const asb::HostWorkload& wl, cudaStream_t s) {
  const int T = ctx.n_tables();
  std::vector<const int64_t*> off(static_cast<size_t>(T)), idx(static_cast<size_t>(T));
  std::vector<int64_t> n(static_cast<size_t>(T));
  for (int t = 0; t < T; ++t) {
    const int pos = wl.find(ctx.spec(t).id);
    if (pos < 0)
      asb::fail(AS_LOOKUP, "measure: table " + std::to_string(ctx.spec(t).id) + " absent from workload");
    const auto& st = wl.per_table[static_cast<size_t>(pos)];
    if (static_cast<int64_t>(st.offsets.size()) != wl.batch_size + 1)
      asb::fail(AS_OFFSET, "table " + std::to_string(st.table_id) + ": offsets length " +
                               std::to_string(st.offsets.size()) + " != batch_size + 1");
    off[t] = st.offsets.data();
    idx[t] = st.indices.data();
    n[t] = static_cast<int64_t>(st.indices.size());
  }
  ctx.load(off.data(), idx.data(), n.data(), s);
}
}  // namespace

asb::HostWorkload::~HostWorkload() {
  if (pinned)
    for (auto& s : per_table) {
      if (!s.offsets.empty()) cudaHostUnregister(s.offsets.data());
      if (!s.indices.empty()) cudaHostUnregister(s.indices.data());
    }
}

extern "C" {

AS_API const char* as_version(void) { return "autoshard-b200 0.1.0 (sm_100a)"; }
AS_API const char* as_last_error(void) { return g_err.c_str(); }

AS_API void as_generator_config_default(as_generator_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->hash_size_min = 1e3;
  c->hash_size_max = 1e7;
  c->pooling_mean_target = 15.0;
  c->pooling_shape = 2.0;
  c->pooling_cap = 193.0;
  c->dim_choices = kDefaultDims;
  c->n_dim_choices = 2;
  c->access_ratio_min = 1e-3;
  c->access_ratio_max = 1.0;
  c->bytes_per_param = 2;
}

AS_API as_status as_generate_pool(uint64_t seed, int32_t n, const as_generator_config* cfg,
                                  as_table_spec* out) {
  return guard([&] {
    need(out, "out");
    auto pool = asb::generate_pool(seed, n, to_cfg(cfg));
    std::memcpy(out, pool.data(), sizeof(as_table_spec) * pool.size());
  });
}

AS_API as_status as_generate_workload(uint64_t seed, const as_table_spec* tables, int32_t n,
                                      int64_t batch, double zipf, int32_t n_threads, as_workload** out) {
  return guard([&] {
    need(out, "out");
    if (n > 0) need(tables, "tables");
    auto w = std::make_unique<as_workload>();
    asb::generate_workload(seed, std::vector<as_table_spec>(tables, tables + n), batch, zipf, n_threads, &w->wl);
    *out = w.release();
  });
}

AS_API int64_t as_workload_batch_size(const as_workload* wl) { return wl ? wl->wl.batch_size : 0; }
AS_API int32_t as_workload_num_tables(const as_workload* wl) {
  return wl ? static_cast<int32_t>(wl->wl.per_table.size()) : 0;
}

AS_API as_status as_workload_stream(const as_workload* wl, int32_t i, int32_t* table_id,
                                    const int64_t** offsets, const int64_t** indices, int64_t* n_indices) {
  return guard([&] {
    need(wl, "wl");
    if (i < 0 || i >= static_cast<int32_t>(wl->wl.per_table.size()))
      asb::fail(AS_LOOKUP, "as_workload_stream: position " + std::to_string(i) + " out of range");
    const auto& s = wl->wl.per_table[static_cast<size_t>(i)];
    if (table_id) *table_id = s.table_id;
    if (offsets) *offsets = s.offsets.data();
    if (indices) *indices = s.indices.data();
    if (n_indices) *n_indices = static_cast<int64_t>(s.indices.size());
  });
}

AS_API as_status as_workload_find(const as_workload* wl, int32_t table_id, int32_t* position) {
  return guard([&] {
    need(wl, "wl");
    const int p = wl->wl.find(table_id);
    if (p < 0) asb::fail(AS_LOOKUP, "table " + std::to_string(table_id) + " absent from workload");
    *position = p;
  });
}

AS_API as_status as_workload_from_arrays(int64_t batch, int32_t n, const int32_t* ids,
                                         const int64_t* const* offsets, const int64_t* const* indices,
                                         const int64_t* n_indices, as_workload** out) {
  return guard([&] {
    need(out, "out");
    if (batch < 1) asb::fail(AS_CONFIG, "batch_size must be >= 1");
    auto w = std::make_unique<as_workload>();
    w->wl.batch_size = batch;
    w->wl.per_table.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      auto& s = w->wl.per_table[static_cast<size_t>(i)];
      s.table_id = ids[i];
      if (i > 0 && ids[i] <= ids[i - 1])
        asb::fail(AS_CONFIG, "as_workload_from_arrays: table ids must be strictly ascending");
      s.offsets.assign(offsets[i], offsets[i] + batch + 1);
      s.indices.assign(indices[i], indices[i] + n_indices[i]);
    }
    *out = w.release();
  });
}

AS_API as_status as_workload_pin(as_workload* wl) {
  return guard([&] {
    need(wl, "wl");
    if (wl->wl.pinned) return;
    for (auto& s : wl->wl.per_table) {
      if (!s.offsets.empty())
        asb::cuda_check(cudaHostRegister(s.offsets.data(), s.offsets.size() * 8, cudaHostRegisterDefault),
                        "cudaHostRegister");
      if (!s.indices.empty())
        asb::cuda_check(cudaHostRegister(s.indices.data(), s.indices.size() * 8, cudaHostRegisterDefault),
                        "cudaHostRegister");
    }
    wl->wl.pinned = true;
  });
}

AS_API void as_workload_destroy(as_workload* wl) { delete wl; }

AS_API as_status as_workload_save(const as_workload* wl, const as_table_spec* tables, const char* path) {
  return guard([&] {
    need(wl, "wl");
    need(path, "path");
    asb::save_workload(path, wl->wl, std::vector<as_table_spec>(tables, tables + wl->wl.per_table.size()));
  });
}

AS_API as_status as_workload_load(const char* path, as_workload** out, as_table_spec* tables_out,
                                  int32_t max_tables, int32_t* n_tables) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto w = std::make_unique<as_workload>();
    std::vector<as_table_spec> tabs;
    asb::load_workload(path, &w->wl, &tabs);
    if (n_tables) *n_tables = static_cast<int32_t>(tabs.size());
    if (tables_out) {
      if (static_cast<int32_t>(tabs.size()) > max_tables)
        asb::fail(AS_SHAPE, "as_workload_load: file has " + std::to_string(tabs.size()) +
                                " tables, capacity " + std::to_string(max_tables));
      std::memcpy(tables_out, tabs.data(), sizeof(as_table_spec) * tabs.size());
    }
    *out = w.release();
  });
}

AS_API as_status as_pool_save(const as_table_spec* tables, int32_t n, const char* path) {
  return guard([&] { asb::save_pool(path, std::vector<as_table_spec>(tables, tables + n)); });
}

AS_API as_status as_pool_load(const char* path, as_table_spec* out, int32_t max_tables, int32_t* n_tables) {
  return guard([&] {
    auto tabs = asb::load_pool(path);
    if (n_tables) *n_tables = static_cast<int32_t>(tabs.size());
    if (out) {
      if (static_cast<int32_t>(tabs.size()) > max_tables)
        asb::fail(AS_SHAPE, "as_pool_load: capacity too small");
      std::memcpy(out, tabs.data(), sizeof(as_table_spec) * tabs.size());
    }
  });
}

AS_API uint64_t as_fingerprint_pool(const as_table_spec* t, int32_t n) { return asb::fingerprint_pool(t, n); }
AS_API uint64_t as_fingerprint_task(const as_table_spec* t, int32_t n, int32_t k, const int64_t* b) {
  return asb::fingerprint_task(t, n, k, b);
}

AS_API as_status as_heuristic_cost(const as_table_spec* t, int32_t kind, double* cost) {
  return guard([&] {
    need(t, "table");
    *cost = asb::heuristic_cost(*t, kind);
  });
}

AS_API as_status as_greedy_shard(const as_table_spec* t, int32_t n, int32_t k, const int64_t* b, int32_t kind,
                                 int32_t* a) {
  return guard([&] { asb::greedy_shard(t, n, k, b, kind, a); });
}

AS_API as_status as_random_shard(const as_table_spec* t, int32_t n, int32_t k, const int64_t* b, uint64_t seed,
                                 int32_t* a) {
  return guard([&] { asb::random_shard(t, n, k, b, seed, a); });
}

AS_API as_status as_plan_validate(int32_t n, int32_t k, const int32_t* a) {
  return guard([&] {
    if (k < 1) asb::fail(AS_CONFIG, "task: num_shards must be >= 1");
    asb::validate_plan(n, k, a);
  });
}

AS_API as_status as_plan_mem_used(const as_table_spec* t, int32_t n, int32_t k, const int32_t* a, int64_t* used) {
  return guard([&] {
    if (k < 1) asb::fail(AS_CONFIG, "task: num_shards must be >= 1");
    asb::validate_plan(n, k, a);
    for (int s = 0; s < k; ++s) used[s] = 0;
    for (int i = 0; i < n; ++i) used[a[i]] += asb::size_bytes(t[i]);
  });
}

AS_API as_status as_degree_of_balance(const double* c, int32_t n, double* out) {
  return guard([&] { *out = asb::degree_of_balance(c, n); });
}

AS_API as_status as_plan_save(const char* path, const as_table_spec* t, int32_t n, int32_t k, const int64_t* b,
                              const int32_t* a, const double* costs) {
  return guard([&] { asb::save_plan(path, t, n, k, b, a, costs); });
}

AS_API as_status as_plan_load(const char* path, const as_table_spec* t, int32_t n, int32_t k, const int64_t* b,
                              int32_t* a, double* costs, int32_t* has_costs) {
  return guard([&] {
    const bool hc = asb::load_plan(path, t, n, k, b, a, costs);
    if (has_costs) *has_costs = hc ? 1 : 0;
  });
}

// ---- device context -----------------------------------------------------
AS_API as_status as_create_ex(int32_t device, const as_table_spec* tables, int32_t n, int64_t batch, uint64_t seed,
                              int32_t flags, as_ctx** out) {
  return guard([&] {
    need(out, "out");
    if (n > 0) need(tables, "tables");
    auto c = std::make_unique<as_ctx>();
    c->impl = std::make_unique<asb::EmbContext>(device, tables, n, batch, seed, flags);
    *out = c.release();
  });
}

AS_API as_status as_create(int32_t device, const as_table_spec* tables, int32_t n, int64_t batch, uint64_t seed,
                           as_ctx** out) {
  return as_create_ex(device, tables, n, batch, seed, 0, out);
}

AS_API as_status as_create_subset(const as_ctx* parent, const int32_t* positions, int32_t n, as_ctx** out) {
  return guard([&] {
    need(parent, "parent");
    need(out, "out");
    if (n > 0) need(positions, "positions");
    auto c = std::make_unique<as_ctx>();
    c->impl = std::make_unique<asb::EmbContext>(*parent->impl, positions, n);
    *out = c.release();
  });
}

AS_API as_status as_retarget_subset(as_ctx* ctx, const int32_t* positions, int32_t n) {
  return guard([&] {
    need(ctx, "ctx");
    if (n > 0) need(positions, "positions");
    ctx->impl->retarget(positions, n);
  });
}

AS_API as_status as_destroy(as_ctx* ctx) {
  return guard([&] { delete ctx; });
}

AS_API as_status as_load_streams(as_ctx* ctx, const int64_t* const* offsets, const int64_t* const* indices,
                                 const int64_t* n_indices, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    if (ctx->impl->n_tables() > 0) {
      need(offsets, "offsets");
      need(indices, "indices");
      need(n_indices, "n_indices");
    }
    ctx->impl->load(offsets, indices, n_indices, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_load_workload(as_ctx* ctx, const as_workload* wl, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    need(wl, "wl");
    load_from_workload(*ctx->impl, wl->wl, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_stage_streams(as_ctx* ctx, const int64_t* const* offsets, const int64_t* const* indices,
                                  const int64_t* n_indices) {
  return guard([&] {
    need(ctx, "ctx");
    if (ctx->impl->n_tables() > 0) {
      need(offsets, "offsets");
      need(indices, "indices");
      need(n_indices, "n_indices");
    }
    ctx->impl->stage(offsets, indices, n_indices);
  });
}

AS_API as_status as_stage_workload(as_ctx* ctx, const as_workload* wl) {
  return guard([&] {
    need(ctx, "ctx");
    need(wl, "wl");
    Picked p = pick_streams(*ctx->impl, wl->wl);
    ctx->impl->stage(p.off.data(), p.idx.data(), p.n.data());
  });
}

AS_API as_status as_commit_staged(as_ctx* ctx, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->commit(static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_check_batch(as_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->check();
  });
}

AS_API as_status as_forward(as_ctx* ctx, float* out, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->forward(out, nullptr, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_set_peer_outputs(as_ctx* ctx, int n_peers, float* const* peer_bases, int64_t rows_per_peer) {
  return guard([&] {
    need(ctx, "ctx");
    if (n_peers > 0) need(peer_bases, "peer_bases");
    if (n_peers < 0 || n_peers > 8) asb::fail(AS_CONFIG, "as_set_peer_outputs: 0..8 peers, got " + std::to_string(n_peers));
    int64_t starts[9];
    for (int q = 0; q <= n_peers; ++q) starts[q] = rows_per_peer * q;
    if (n_peers > 0 && rows_per_peer * n_peers != ctx->impl->batch())
      asb::fail(AS_SHAPE, "as_set_peer_outputs: " + std::to_string(n_peers) + " peers x " + std::to_string(rows_per_peer) +
                              " rows must cover the batch of " + std::to_string(ctx->impl->batch()));
    ctx->impl->set_peer_outputs(n_peers, peer_bases, starts);
  });
}

AS_API as_status as_set_peer_outputs_v(as_ctx* ctx, int n_peers, float* const* peer_bases, const int64_t* row_start) {
  return guard([&] {
    need(ctx, "ctx");
    if (n_peers > 0) {
      need(peer_bases, "peer_bases");
      need(row_start, "row_start");
    }
    ctx->impl->set_peer_outputs(n_peers, peer_bases, row_start);
  });
}

AS_API as_status as_backward_rowwise_adagrad(as_ctx* ctx, const float* grad, float lr, float eps, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->backward(grad, lr, eps, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_step(as_ctx* ctx, float lr, float eps, double* loss, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->step(lr, eps, loss, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_measure(as_ctx* ctx, int32_t w, int32_t m, int32_t r, int32_t flush, float lr, float eps,
                            double* ms) {
  return guard([&] {
    need(ctx, "ctx");
    need(ms, "ms_out");
    *ms = ctx->impl->measure(w, m, r, flush != 0, lr, eps);
  });
}

AS_API as_status as_measure_plan(const as_table_spec* tables, int32_t n, int32_t k, const int32_t* assignment,
                                 const as_workload* wl, const int32_t* devices, int32_t n_devices,
                                 const as_bench_config* bench, double* costs) {
  return guard([&] {
    need(wl, "wl");
    need(bench, "bench");
    need(costs, "costs");
    if (k < 1) asb::fail(AS_CONFIG, "task: num_shards must be >= 1");
    if (static_cast<int32_t>(0) > n) asb::fail(AS_CONFIG, "n_tables must be >= 0");
    asb::validate_plan(n, k, assignment);  // ShardingPlan::validate, tables.hpp:96-108
    if (bench->warmup < 0 || bench->measure < 1 || bench->trim < 0 || bench->measure - 2 * bench->trim < 1)
      asb::fail(AS_CONFIG, "micro_benchmark: need measure - 2*trim >= 1, got B=" + std::to_string(bench->measure) +
                               " R=" + std::to_string(bench->trim));
    for (int i = 0; i < n; ++i)
      if (wl->wl.find(tables[i].id) < 0)
        asb::fail(AS_LOOKUP, "measure_plan: table " + std::to_string(tables[i].id) + " absent from workload");
    for (int s = 0; s < k; ++s) {
      std::vector<as_table_spec> members;
      for (int i = 0; i < n; ++i)
        if (assignment[i] == s) members.push_back(tables[i]);
      const int dev = (devices && n_devices > 0) ? devices[s % n_devices] : 0;
      asb::EmbContext ctx(dev, members.data(), static_cast<int>(members.size()), wl->wl.batch_size, bench->seed);
      load_from_workload(ctx, wl->wl, nullptr);
      costs[s] = ctx.measure(bench->warmup, bench->measure, bench->trim, bench->flush_l2 != 0, bench->lr,
                             bench->eps);
    }
  });
}

AS_API as_status as_ctx_info_get(const as_ctx* ctx, as_ctx_info* info) {
  return guard([&] {
    need(ctx, "ctx");
    need(info, "info");
    ctx->impl->info(info);
  });
}

AS_API as_status as_profile_enable(as_ctx* ctx, int32_t enable) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->profile_enable(enable);
  });
}

AS_API as_status as_profile_read(as_ctx* ctx, double* ms, int64_t* launches, int32_t reset) {
  return guard([&] {
    need(ctx, "ctx");
    need(ms, "ms");
    ctx->impl->profile_read(ms, launches, reset != 0);
  });
}

AS_API as_status as_table_features(as_ctx* ctx, double* out, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    ctx->impl->table_features(out, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_read_rows(as_ctx* ctx, int32_t t, const int64_t* rows, int64_t n, float* out) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->read_rows(t, rows, n, out);
  });
}

AS_API as_status as_read_momentum(as_ctx* ctx, int32_t t, const int64_t* rows, int64_t n, float* out) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->read_momentum(t, rows, n, out);
  });
}

AS_API as_status as_read_buffer(as_ctx* ctx, int32_t what, void* host, int64_t nbytes) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->read_buffer(what, host, nbytes);
  });
}

AS_API as_status as_write_table(as_ctx* ctx, int32_t t, const float* w, const float* m) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->impl->write_table(t, w, m);
  });
}

AS_API as_status as_load_streams_exchanged(as_comm* comm, int32_t n_all, const as_table_spec* all_tables,
                                           const int32_t* owner, const int64_t* const* local_offsets,
                                           const int64_t* const* local_indices, void* stream) {
  return guard([&] {
    need(comm, "comm");
    if (n_all < 0) asb::fail(AS_CONFIG, "as_load_streams_exchanged: n_all must be >= 0");
    if (n_all > 0) {
      need(all_tables, "all_tables");
      need(owner, "owner");
      need(local_offsets, "local_offsets");
      need(local_indices, "local_indices");
    }
    comm->impl->load_exchanged(n_all, all_tables, owner, local_offsets, local_indices,
                               static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_comm_unique_id(void* id) {
  return guard([&] {
    need(id, "unique_id_out");
    asb::nccl_unique_id(id);
  });
}

AS_API as_status as_comm_init(as_ctx* ctx, const void* uid, int32_t rank, int32_t world, as_comm** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    auto c = std::make_unique<as_comm>();
    c->impl = std::make_unique<asb::ShardComm>(ctx->impl.get(), uid, rank, world);
    *out = c.release();
  });
}

AS_API as_status as_comm_destroy(as_comm* comm) {
  return guard([&] { delete comm; });
}

AS_API as_status as_alltoall_setup(as_comm* comm, const int64_t* shard_dims, const int64_t* row_start, int32_t mode) {
  return guard([&] {
    need(comm, "comm");
    need(shard_dims, "shard_dims");
    need(row_start, "row_start");
    comm->impl->setup(shard_dims, row_start, mode);
  });
}

AS_API as_status as_alltoall_handle(as_comm* comm, void* blob, int64_t* nbytes) {
  return guard([&] {
    need(comm, "comm");
    need(blob, "blob_out");
    comm->impl->handle(blob, nbytes);
  });
}

AS_API as_status as_alltoall_open(as_comm* comm, const void* all) {
  return guard([&] {
    need(comm, "comm");
    need(all, "all_blobs");
    comm->impl->open(all);
  });
}

AS_API as_status as_alltoall_host_barrier(as_comm* comm, as_host_barrier_fn fn, void* user) {
  return guard([&] {
    need(comm, "comm");
    comm->impl->set_host_barrier(fn, user);
  });
}

AS_API as_status as_forward_sharded(as_comm* comm, void* stream) {
  return guard([&] {
    need(comm, "comm");
    comm->impl->forward(static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_backward_sharded(as_comm* comm, const float* grad_recv, float lr, float eps, void* stream) {
  return guard([&] {
    need(comm, "comm");
    comm->impl->backward(grad_recv, lr, eps, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_step_sharded(as_comm* comm, float lr, float eps, double* loss_out, void* stream) {
  return guard([&] {
    need(comm, "comm");
    comm->impl->step(lr, eps, loss_out, static_cast<cudaStream_t>(stream));
  });
}

AS_API as_status as_comm_info_get(const as_comm* comm, as_comm_info* info) {
  return guard([&] {
    need(comm, "comm");
    need(info, "info");
    comm->impl->info(info);
  });
}

AS_API as_status as_comm_profile_read(as_comm* comm, double* ms2, int32_t reset) {
  return guard([&] {
    need(comm, "comm");
    need(ms2, "ms2");
    comm->impl->profile_read(ms2, reset != 0);
  });
}

AS_API as_status as_probe_gather_bw(int32_t device, int64_t footprint_bytes, int32_t row_bytes, double* gbs) {
  return guard([&] {
    need(gbs, "gbs");
    *gbs = asb::probe_gather_bw(device, footprint_bytes, row_bytes);
  });
}

}  // extern "C"
