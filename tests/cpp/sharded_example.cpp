// The table-wise sharded step from C++ over the plain C-ABI only
// (include/autoshard_b200.h): one process per rank, no Python, no torch, no
// MPI. The peer-memory handle blobs are exchanged through files in a shared
// directory (any launcher's control plane would do); with one GPU both ranks
// run on device 0 (cudaIpc between processes on one device; the exchange
// barrier then runs on the host through files), with several rank r uses
// device r.
//
//   env: RANK, WORLD (1..8), XDIR (shared directory), ASB_DEVICE (default RANK)
//   prints: "rank R loss L0 L1 L2" — the loss 1/2|recv|^2 of this rank's
//   samples over ALL tables for three steps (weights evolve).
//
// tests/test_sharded_multiproc.py runs it with WORLD=2 and WORLD=1 and checks
// that the ranks' losses add up to the unsharded run's.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "autoshard_b200.h"

static void check(as_status s, const char* what) {
  if (s != AS_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, (int)s, as_last_error());
    std::exit(1);
  }
}

static void file_barrier(const std::string& dir, const char* tag, int rank, int world) {
  std::ofstream(dir + "/" + tag + "_" + std::to_string(rank)).put('1');
  for (int q = 0; q < world; ++q) {
    const std::string f = dir + "/" + tag + "_" + std::to_string(q);
    for (int tries = 0; !std::ifstream(f).good(); ++tries) {
      if (tries > 60000) {
        std::fprintf(stderr, "rank %d: timeout waiting for %s\n", rank, f.c_str());
        std::exit(2);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(5));
    }
  }
}

// Ranks sharing one device (ASB_DEVICE set): the exchange barrier runs on the
// host (as_alltoall_host_barrier) — no kernel waits on another process's kernel.
struct HostBarrier {
  std::string dir;
  int rank, world, epoch;
};
static int32_t host_barrier(void* user) {
  HostBarrier* h = static_cast<HostBarrier*>(user);
  const std::string tag = "x" + std::to_string(h->epoch++);
  file_barrier(h->dir, tag.c_str(), h->rank, h->world);
  return 0;
}

int main() {
  const int rank = std::atoi(std::getenv("RANK") ? std::getenv("RANK") : "0");
  const int world = std::atoi(std::getenv("WORLD") ? std::getenv("WORLD") : "1");
  const std::string dir = std::getenv("XDIR") ? std::getenv("XDIR") : "/tmp";
  const int device = std::getenv("ASB_DEVICE") ? std::atoi(std::getenv("ASB_DEVICE")) : rank;

  // tables (generate_pool, tables.hpp:178) and a plan (random_shard, planners.hpp:111)
  as_generator_config gc;
  as_generator_config_default(&gc);
  const int32_t dims[] = {16, 64};
  gc.dim_choices = dims;
  gc.n_dim_choices = 2;
  gc.hash_size_max = 4e4;
  gc.pooling_mean_target = 12.0;
  const int n = 9;
  std::vector<as_table_spec> pool(n);
  check(as_generate_pool(4, n, &gc, pool.data()), "as_generate_pool");
  const int64_t B = 64 * 2 + 3;  // uneven split for WORLD=2
  std::vector<int64_t> budget(world, int64_t(1) << 40);
  std::vector<int32_t> assign(n, 0);
  if (world > 1) check(as_random_shard(pool.data(), n, world, budget.data(), 5, assign.data()), "as_random_shard");
  std::vector<as_table_spec> mine;
  std::vector<int64_t> shard_dims(world, 0);
  for (int t = 0; t < n; ++t) {
    shard_dims[assign[t]] += pool[t].dim;
    if (assign[t] == rank) mine.push_back(pool[t]);
  }
  std::vector<int64_t> row_start(world + 1);
  for (int p = 0; p <= world; ++p) row_start[p] = B * p / world;

  // this rank's shard: its tables' streams over the whole batch
  as_ctx* ctx = nullptr;
  check(as_create(device, mine.data(), (int32_t)mine.size(), B, 3, &ctx), "as_create");
  as_workload* wl = nullptr;
  check(as_generate_workload(0, mine.data(), (int32_t)mine.size(), B, 1.05, 0, &wl), "as_generate_workload");
  check(as_load_workload(ctx, wl, nullptr), "as_load_workload");

  // the exchange: peer-memory handles through files, no NCCL
  as_comm* comm = nullptr;
  check(as_comm_init(ctx, nullptr, rank, world, &comm), "as_comm_init");
  check(as_alltoall_setup(comm, shard_dims.data(), row_start.data(), AS_XCHG_PEER), "as_alltoall_setup");
  std::vector<char> blob(AS_HANDLE_BYTES, 0), all(static_cast<size_t>(AS_HANDLE_BYTES) * world, 0);
  int64_t nb = 0;
  check(as_alltoall_handle(comm, blob.data(), &nb), "as_alltoall_handle");
  std::ofstream(dir + "/blob_" + std::to_string(rank), std::ios::binary).write(blob.data(), AS_HANDLE_BYTES);
  file_barrier(dir, "blobs", rank, world);
  for (int q = 0; q < world; ++q)
    std::ifstream(dir + "/blob_" + std::to_string(q), std::ios::binary).read(&all[(size_t)q * AS_HANDLE_BYTES],
                                                                             AS_HANDLE_BYTES);
  check(as_alltoall_open(comm, all.data()), "as_alltoall_open");
  HostBarrier hb{dir, rank, world, 0};
  if (std::getenv("ASB_DEVICE")) check(as_alltoall_host_barrier(comm, host_barrier, &hb), "as_alltoall_host_barrier");

  double loss[3];
  for (double& l : loss) check(as_step_sharded(comm, 0.01f, 1e-8f, &l, nullptr), "as_step_sharded");
  std::printf("rank %d loss %.17g %.17g %.17g\n", rank, loss[0], loss[1], loss[2]);
  std::fflush(stdout);
  file_barrier(dir, "done", rank, world);  // no rank unmaps while a peer still stores into it
  check(as_comm_destroy(comm), "as_comm_destroy");
  as_workload_destroy(wl);
  check(as_destroy(ctx), "as_destroy");
  return 0;
}
