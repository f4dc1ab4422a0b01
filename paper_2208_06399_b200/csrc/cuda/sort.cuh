// K2: stable LSD radix sort of (table-local row, bag) pairs, SEGMENTED BY
// TABLE. The lookups of a shard are table-major already, and row ids are
// table-local (< hash_t), so every table is sorted in its own element range
// with only ceil(bits(hash_t - 1) / 8) digit passes: a 10^4-row table needs
// 2 passes, a 10^7-row table 3, where one global sort over the shard's
// concatenated row space (log2(sum hash) = 26..30 bits) needs 4 for every
// table (pool856: 2.62 passes per lookup on average instead of 4).
//
// Per pass, every tile (kSortTile elements of ONE table) runs CUB's onesweep
// agent (block ranking with warp match-any, decoupled look-back, CCCL 2.8,
// namespaced asb_cub) against the table's own look-back region, tile counter
// and digit offsets; our kernels around it: the per-table digit histograms of
// all passes in one read of the keys, their exclusive scans, and the tile ->
// table mapping. Ping-pong buffers are picked per table so that its LAST pass
// writes the output arrays.
#pragma once

#include <cub/block/block_load.cuh>
#include <cub/block/block_store.cuh>
#include <cub/agent/agent_radix_sort_onesweep.cuh>
#include <cub/block/block_scan.cuh>

#include "types.hpp"


namespace asb {

namespace cubns = CUB_NS_QUALIFIER;

constexpr int kHistThreads = 256;

#ifndef ASB_SORT_PARTS
#define ASB_SORT_PARTS 1
#endif
#ifndef ASB_SORT_RANK
#define ASB_SORT_RANK RADIX_RANK_MATCH_EARLY_COUNTS_ANY
#endif
#ifndef ASB_SORT_SCAN
#define ASB_SORT_SCAN BLOCK_SCAN_RAKING_MEMOIZE
#endif
using OnesweepPolicy =
    cubns::AgentRadixSortOnesweepPolicy<ASB_SORT_THREADS, ASB_SORT_ITEMS, unsigned, ASB_SORT_PARTS,
                                        cubns::ASB_SORT_RANK, cubns::ASB_SORT_SCAN, cubns::RADIX_SORT_STORE_DIRECT,
                                        kSortBits>;
using OnesweepAgent = cubns::detail::radix_sort::AgentRadixSortOnesweep<OnesweepPolicy, false, unsigned, int, int, int>;


struct SortParams {
  const DevTable* tabs;
  int T;
  const unsigned* keys_in;  // batch order (table-local rows)
  const int* vals_in;       // bag ids
  unsigned* keys_out;       // sorted (final)
  int* vals_out;
  unsigned* keys_tmp;  // ping-pong
  int* vals_tmp;
  int* bins;      // [T][kMaxSortPasses][256]: digit counts, then (in place) exclusive offsets
  int* lookback;  // [kMaxSortPasses][n_tiles][256]
  int* ctrs;      // [kMaxSortPasses][T] per-table tile counters (+ kMaxSortPasses spare)
  int n_tiles;    // sum over tables of ceil(L_t / kSortTile)
  // work maps (built on the host per batch): histogram CTA -> (table, chunk of
  // kHistTilesPerCta tiles in the table); pass p: tile (blockIdx) -> table
  const int* hist_tab;
  const int* hist_chunk;
  const int* tile_tab[kMaxSortPasses];
};

// Digit counts of every pass of one table, over kHistTilesPerCta sort tiles.
// Per-warp private sub-histograms keep Zipf-hot digits from serialising the
// shared-memory atomics of the whole CTA.
__global__ void __launch_bounds__(kHistThreads) sort_hist_kernel(SortParams sp) {
  constexpr int kWarps = kHistThreads / 32;
  __shared__ int h[kWarps][kMaxSortPasses][kSortDigits];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kMaxSortPasses * kSortDigits; i += kHistThreads) (&h[0][0][0])[i] = 0;
  __syncthreads();
  const int t = __ldg(sp.hist_tab + blockIdx.x);
  const DevTable tb = sp.tabs[t];
  const int np = sort_passes_of(tb.sort_bits);
  const long long lo = (long long)__ldg(sp.hist_chunk + blockIdx.x) * kHistTilesPerCta * kSortTile;
  const long long hi = min((long long)tb.n_lookups, lo + (long long)kHistTilesPerCta * kSortTile);
  const unsigned* keys = sp.keys_in + tb.idx_off;
  int* hw = &h[warp][0][0];
  for (long long j = lo + threadIdx.x; j < hi; j += kHistThreads) {
    const unsigned k = __ldcs(keys + j);
#pragma unroll
    for (int p = 0; p < kMaxSortPasses; ++p)
      if (p < np) atomicAdd(hw + p * kSortDigits + ((k >> (p * kSortBits)) & (kSortDigits - 1)), 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < np * kSortDigits; i += kHistThreads) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += (&h[w][0][0])[i];
    if (s) atomicAdd(sp.bins + (long long)t * kMaxSortPasses * kSortDigits + i, s);
  }
  (void)lane;
}

// Exclusive scan of each (table, pass) digit histogram, in place.
__global__ void __launch_bounds__(kSortDigits) sort_scan_kernel(SortParams sp) {
  using Scan = cubns::BlockScan<int, kSortDigits>;
  __shared__ typename Scan::TempStorage tmp;
  const int t = blockIdx.x, p = blockIdx.y;
  if (p >= sort_passes_of(sp.tabs[t].sort_bits) || sp.tabs[t].n_lookups == 0) return;
  int* b = sp.bins + ((long long)t * kMaxSortPasses + p) * kSortDigits;
  int v = b[threadIdx.x], x;
  Scan(tmp).ExclusiveSum(v, x);
  b[threadIdx.x] = x;
}

// One digit pass over the tiles of every table that still has digits left.
#ifndef ASB_SORT_MINBLOCKS
#define ASB_SORT_MINBLOCKS 2
#endif
__global__ void __launch_bounds__(ASB_SORT_THREADS, ASB_SORT_MINBLOCKS) sort_onesweep_kernel(SortParams sp, int pass) {
  __shared__ typename OnesweepAgent::TempStorage s;
  // the table of this tile; the agent's per-table tile counter orders the
  // look-back (a tile only waits on tiles of its table that already started)
  const int t = __ldg(sp.tile_tab[pass] + blockIdx.x);
  const DevTable& tb = sp.tabs[t];
  const int np = sort_passes_of(tb.sort_bits);
  // the table's last pass writes the output buffers
  const bool to_out = ((np - 1 - pass) & 1) == 0;
  const unsigned* kin = pass == 0 ? sp.keys_in : (to_out ? sp.keys_tmp : sp.keys_out);
  const int* vin = pass == 0 ? sp.vals_in : (to_out ? sp.vals_tmp : sp.vals_out);
  unsigned* kout = to_out ? sp.keys_out : sp.keys_tmp;
  int* vout = to_out ? sp.vals_out : sp.vals_tmp;
  const long long o = tb.idx_off;
  OnesweepAgent agent(s, sp.lookback + ((long long)pass * sp.n_tiles + tb.sort_tile_off) * kSortDigits,
                      sp.ctrs + pass * sp.T + t, nullptr,
                      sp.bins + ((long long)t * kMaxSortPasses + pass) * kSortDigits, kout + o, kin + o, vout + o,
                      vin + o, (int)tb.n_lookups, pass * kSortBits, min(kSortBits, tb.sort_bits - pass * kSortBits));
  agent.Process();
}

}  // namespace asb
