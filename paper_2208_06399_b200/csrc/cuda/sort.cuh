// K2: stable LSD radix sort of (table-local row, bag) pairs, SEGMENTED BY
// TABLE, hand-written for sm_100a (no library code).
//
// The lookups of a shard are table-major and row ids are table-local
// (< hash_t), so every table is sorted in its own element range with only
// ceil(bits(hash_t - 1) / 8) digit passes: 2 for a 10^4-row table, 3 for
// 10^7 (pool856: 2.62 passes per lookup instead of the 4 a global sort over
// the shard's concatenated row space needs).
//
// Each pass is reduce-then-scan over SUPERBLOCKS (sb_elems elements of one
// table: 1..16 tiles, chosen per batch for several waves of CTAs):
//   upsweep    CTA per superblock: digit counts (per-warp smem histograms)
//   scan       CTA per table: counts -> each superblock's first output
//              position per digit (digit-major, superblock-minor), in place
//   downsweep  CTA per superblock, its tiles in order: warp-stable ranking
//              (match.any peers + per-warp digit counters), warp -> tile
//              prefix per digit, scatter to the running per-digit position
// No CTA waits on another (no look-back chain): every superblock's offsets
// are known before its downsweep starts.
//
// Pass 0 reads the values (bag ids) from K4's bag array; its upsweep and
// scan need only the row ids, so they overlap K4 and only the pass-0
// downsweep waits for it.
//
// Stability: a warp owns a contiguous run of the tile and ranks its items in
// element order; warps, tiles and superblocks are ranked in element order.
// Every table's input is in bag order, so the output is sorted by (row, bag).
// Ping-pong buffers are picked per table so that its LAST pass writes the
// output arrays.
#pragma once

#include "types.hpp"

namespace asb {

static_assert(kSortThreads == kSortDigits, "one thread per digit in the scan / prefix steps");
constexpr int kSortWarps = kSortThreads / 32;

struct SortParams {
  const DevTable* tabs;
  int pass;
  const unsigned* keys_in;  // idx32 (table-local rows, batch order)
  const int* vals_in;       // bag ids (K4)
  unsigned* keys_out;       // sorted (final)
  int* vals_out;
  unsigned* keys_tmp;  // ping-pong
  int* vals_tmp;
  int* hist;           // [n_sb][256]: digit counts of the pass, then the first output position per digit
  const int* sb_tab;   // superblock -> table
  const int* pass_sb;  // superblocks of the tables taking part in this pass
  int sb_elems;        // elements per superblock (a multiple of kSortTile)
  int bag_bits;        // bits of the largest bag id (packed keys: row << bag_bits | bag)
};

struct SortView {
  const unsigned* kin;
  const int* vin;
  unsigned* kout;
  int* vout;
};
__device__ __forceinline__ SortView sort_view(const SortParams& sp, const DevTable& tb) {
  const int np = sort_passes_of(tb.sort_bits);
  const bool to_out = ((np - 1 - sp.pass) & 1) == 0;  // the table's last pass writes the output
  SortView v;
  const long long o = tb.idx_off;
  v.kin = (sp.pass == 0 ? sp.keys_in : (to_out ? sp.keys_tmp : sp.keys_out)) + o;
  v.vin = (sp.pass == 0 ? sp.vals_in : (to_out ? sp.vals_tmp : sp.vals_out)) + o;
  v.kout = (to_out ? sp.keys_out : sp.keys_tmp) + o;
  v.vout = (to_out ? sp.vals_out : sp.vals_tmp) + o;
  return v;
}

// Digit position of this pass in the keys it reads: packed tables carry
// (row << bag_bits | bag) after pass 0, whose input is the plain row.
// Digit width of a table: its ceil(bits / 8) passes split its row bits
// evenly (a 17-bit table sorts 6 + 6 + 5 bits, not 8 + 8 + 1), so every pass
// has at most 2^width buckets: longer runs per bucket and tile in the
// write-out (fewer partial sectors), fewer distinct digits per warp to rank.
__device__ __forceinline__ int sort_width(const DevTable& tb) {
#ifdef ASB_SORT_FULL_DIGITS
  return kSortBits;
#else
  const int np = sort_passes_of(tb.sort_bits);
  return (tb.sort_bits + np - 1) / np;
#endif
}
__device__ __forceinline__ int sort_shift(const SortParams& sp, const DevTable& tb, bool as_read) {
  const bool packed_in = tb.sort_packed && (sp.pass > 0 || !as_read);
  return sp.pass * sort_width(tb) + (packed_in ? sp.bag_bits : 0);
}
__device__ __forceinline__ unsigned sort_mask(const DevTable& tb) { return (1u << sort_width(tb)) - 1u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Digit counts of one superblock.
__global__ void __launch_bounds__(kSortThreads) sort_upsweep_kernel(SortParams sp) {
  __shared__ int h[kSortWarps][kSortDigits];
  const int warp = threadIdx.x >> 5;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) h[w][threadIdx.x] = 0;
  const int sb = __ldg(sp.pass_sb + blockIdx.x);
  const int t = __ldg(sp.sb_tab + sb);
  const DevTable& tb = sp.tabs[t];
  const SortView v = sort_view(sp, tb);
  const long long lo = (long long)(sb - tb.sort_tile_off) * sp.sb_elems;
  const int n = (int)min((long long)sp.sb_elems, tb.n_lookups - lo);
  const int shift = sort_shift(sp, tb, true);
  const unsigned dm = sort_mask(tb);
  const unsigned* k = v.kin + lo;
  __syncthreads();
  int* hw = h[warp];
  constexpr int U = 8;
  for (int j0 = 0; j0 < n; j0 += U * kSortThreads) {
    unsigned x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * kSortThreads + threadIdx.x;
      x[u] = j < n ? __ldcs(k + j) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u * kSortThreads + (int)threadIdx.x < n) atomicAdd(hw + ((x[u] >> shift) & dm), 1);
  }
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) s += h[w][threadIdx.x];
  sp.hist[(long long)sb * kSortDigits + threadIdx.x] = s;
}

// Per table: counts -> first output position of every (superblock, digit),
// digit-major then superblock order (table-local positions).
__global__ void __launch_bounds__(kSortDigits) sort_scan_kernel(SortParams sp) {
  __shared__ int ws[kSortDigits / 32];
  const DevTable& tb = sp.tabs[blockIdx.x];
  if (tb.n_lookups == 0 || sp.pass >= sort_passes_of(tb.sort_bits)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsb = (int)((tb.n_lookups + sp.sb_elems - 1) / sp.sb_elems);
  int* h = sp.hist + (long long)tb.sort_tile_off * kSortDigits + threadIdx.x;
  // 8 superblocks' counts in flight per round trip (a 45-superblock table was
  // 2 x 45 dependent loads: 25 % of the cfg2 sort)
  constexpr int R = 8;
  int tot = 0;
  for (int k = 0; k < nsb; k += R) {
    int v[R];
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = k + u < nsb ? h[(long long)(k + u) * kSortDigits] : 0;
#pragma unroll
    for (int u = 0; u < R; ++u) tot += v[u];
  }
  int x = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  int run = x - tot;
  for (int w = 0; w < warp; ++w) run += ws[w];
  for (int k = 0; k < nsb; k += R) {
    int v[R];
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = k + u < nsb ? h[(long long)(k + u) * kSortDigits] : 0;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (k + u < nsb) h[(long long)(k + u) * kSortDigits] = run;
      run += v[u];
    }
  }
}

#ifndef ASB_SORT_MINBLOCKS
#define ASB_SORT_MINBLOCKS 5
#endif
// Per tile: the keys and values come into registers (warp-striped: a warp
// owns a contiguous run of the tile), are ranked stably, placed in shared
// memory in digit order, and written out from there so consecutive threads
// store consecutive positions of a digit's run (coalesced: the first pass's
// input is in bag order, so a warp's 32 elements would otherwise hit ~24
// different sectors). The next tile's loads are issued before this tile's
// write-out, so their latency overlaps it.
// MODE 0: rows + bag ids in and out; packed tables (tb.sort_packed): 1 = pass
// 0 (rows + bag ids in, packed keys out), 2 = keys alone, 3 = the table's
// last pass (packed keys in, rows + bag ids out) — half the bytes in between.
struct SortSmem {
  unsigned lkey[kSortTile];         // the tile in digit order
  int lval[kSortTile];
  int cnt[kSortWarps][kSortDigits];  // per-warp digit counts, then per-warp tile offsets
  int gbase[kSortDigits];            // running output position per digit
  int gdelta[kSortDigits];           // output position - tile position, per digit
  int wsum[kSortWarps];
};

template <int MODE>
__device__ __forceinline__ void sort_downsweep_body(const SortParams& sp, SortSmem& sm, const SortView& v, int n,
                                                    int shift, unsigned dm) {
  constexpr int I = kSortItems;
  constexpr bool VALS_IN = MODE <= 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int bb = sp.bag_bits;
  const unsigned lt = lanemask_lt();
  const int wb = warp * (I * 32);
  unsigned key[I];
  int val[I];
  auto load = [&](int a) {
    const int nt = min(kSortTile, n - a);
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int e = wb + i * 32 + lane;
      key[i] = e < nt ? __ldcs(v.kin + a + e) : 0u;
      if constexpr (VALS_IN) val[i] = e < nt ? __ldcs(v.vin + a + e) : 0;
      if constexpr (MODE == 1) key[i] = (key[i] << bb) | (unsigned)val[i];
    }
  };
  load(0);
  for (int a = 0; a < n; a += kSortTile) {
    const int nt = min(kSortTile, n - a);
    // warp-stable ranking
#pragma unroll
    for (int q = 0; q < kSortDigits / 32; ++q) sm.cnt[warp][q * 32 + lane] = 0;
    __syncwarp();
    int rk[I];
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const bool ok = wb + i * 32 + lane < nt;
      const unsigned d = ok ? (key[i] >> shift) & dm : kSortDigits + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int before = __popc(peers & lt);
      const int c = ok ? sm.cnt[warp][d] : 0;
      __syncwarp();
      if (ok && (peers >> lane) == 1u) sm.cnt[warp][d] = c + before + 1;  // highest lane of the group
      __syncwarp();
      rk[i] = c + before;
    }
    __syncthreads();
    {
      // digit d: tile count, exclusive scan over digits (tile offset), warp offsets
      const int d = threadIdx.x;
      int c = 0;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) c += sm.cnt[w][d];
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) sm.wsum[warp] = x;
      __syncthreads();
      int toff = x - c;
      for (int w = 0; w < warp; ++w) toff += sm.wsum[w];
      sm.gdelta[d] = sm.gbase[d] - toff;
      sm.gbase[d] += c;
      int run = toff;
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const int cw = sm.cnt[w][d];
        sm.cnt[w][d] = run;
        run += cw;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < I; ++i) {
      if (wb + i * 32 + lane < nt) {
        const int lp = sm.cnt[warp][(key[i] >> shift) & dm] + rk[i];
        sm.lkey[lp] = key[i];
        if constexpr (MODE == 0) sm.lval[lp] = val[i];
      }
    }
    __syncthreads();
    if (a + kSortTile < n) load(a + kSortTile);  // in flight during the write-out
#pragma unroll 4
    for (int i = 0; i < I; ++i) {
      const int lp = i * kSortThreads + threadIdx.x;
      if (lp < nt) {
        const unsigned k = sm.lkey[lp];
        const int pos = lp + sm.gdelta[(k >> shift) & dm];
        if constexpr (MODE == 0) {
          v.kout[pos] = k;
          v.vout[pos] = sm.lval[lp];
        } else if constexpr (MODE == 3) {
          v.kout[pos] = k >> bb;
          v.vout[pos] = (int)(k & ((1u << bb) - 1u));
        } else {
          v.kout[pos] = k;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kSortThreads, ASB_SORT_MINBLOCKS) sort_downsweep_kernel(SortParams sp) {
  __shared__ SortSmem sm;
  const int sb = __ldg(sp.pass_sb + blockIdx.x);
  const int t = __ldg(sp.sb_tab + sb);
  const DevTable& tb = sp.tabs[t];
  SortView v = sort_view(sp, tb);
  const long long lo = (long long)(sb - tb.sort_tile_off) * sp.sb_elems;
  const int n = (int)min((long long)sp.sb_elems, tb.n_lookups - lo);
  v.kin += lo;
  v.vin += lo;
  sm.gbase[threadIdx.x] = sp.hist[(long long)sb * kSortDigits + threadIdx.x];
  const int shift = sort_shift(sp, tb, false);
  const unsigned dm = sort_mask(tb);
  const int mode =
      !tb.sort_packed ? 0 : (sp.pass == 0 ? 1 : (sp.pass == sort_passes_of(tb.sort_bits) - 1 ? 3 : 2));
  switch (mode) {
    case 0: sort_downsweep_body<0>(sp, sm, v, n, shift, dm); break;
    case 1: sort_downsweep_body<1>(sp, sm, v, n, shift, dm); break;
    case 2: sort_downsweep_body<2>(sp, sm, v, n, shift, dm); break;
    default: sort_downsweep_body<3>(sp, sm, v, n, shift, dm); break;
  }
}

}  // namespace asb
