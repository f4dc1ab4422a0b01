// Plain structs shared by the host context and the kernels.
#pragma once

#include <vector_types.h>

#ifndef ASB_SORT_ITEMS
#define ASB_SORT_ITEMS 8
#endif

namespace asb {

// K2 (sort.cuh): 8-bit digits; tiles of 256 threads x kSortItems elements;
// superblocks of 1..kSortMaxSBTiles tiles (the unit of the per-pass digit
// counts; chosen per batch so that there are several waves of CTAs)
constexpr int kSortBits = 8;
constexpr int kSortDigits = 1 << kSortBits;
constexpr int kSortThreads = 256;
constexpr int kSortItems = ASB_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kSortMaxSBTiles = 16;
constexpr int kMaxSortPasses = 4;  // table-local rows < 2^31
__host__ __device__ constexpr int sort_passes_of(int bits) { return (bits + kSortBits - 1) / kSortBits; }

// Per-table device descriptor (host-built, see context.cu).
struct DevTable {
  long long w_base;     // W element offset of the table: row r (table-local) at w_base + r*dim
  long long row_off;    // first global row of the table (momentum M[row_off + r])
  long long hash;       // rows
  long long idx_off;    // first element of the table in the lookup arrays
  long long n_lookups;  // L_t of the loaded batch
  int dim;
  int col;        // first pooled column
  int chunk_off;  // first (global) chunk id; a table owns n_units * (32/GL) chunks
  int chunk_len;  // elements per chunk (multiple of 32)
  int unit_off;   // first warp unit; a warp unit = 32/GL consecutive chunks
  int n_units;
  int table_id;
  int kind;  // lane layout (GL lanes per row, NV float4 per lane), see kind_gl / kind_nv
  int sort_bits;      // bits of the largest table-local row id (K2 passes = ceil(sort_bits / 8))
  int sort_tile_off;  // first K2 superblock of the table (its digit-count rows)
  int sort_packed;    // K2 sorts 32-bit (row << bag_bits | bag) keys alone (rows + bag ids fit 32 bits, >= 2 passes)
};

// Lane layouts: kinds 0..5: GL = 1..32, NV = 1; 6,7,8: GL = 32, NV = 2,4,8;
// 9: GL 8 NV 2; 10: GL 16 NV 2; 11: GL 8 NV 4; 12: GL 16 NV 4 (wider per-lane
// vectors: one warp instruction gathers 2-4 rows).
__host__ __device__ constexpr int kind_gl(int k) {
  return k <= 5 ? 1 << k : (k <= 8 ? 32 : ((k == 9 || k == 11) ? 8 : 16));
}
__host__ __device__ constexpr int kind_nv(int k) { return k <= 5 ? 1 : (k <= 8 ? 1 << (k - 5) : (k <= 10 ? 2 : 4)); }
constexpr int kNumKinds = 13;

// Fused forward exchange (table-wise sharding): pooled row b
// goes straight to the receive buffer of its sample owner q (start[q] <= b <
// start[q+1]; uneven splits allowed), at base[q] + (b - start[q]) * out_stride
// + col_t — on another GPU a peer (NVLink) store, so the all-to-all of the
// pooled rows rides on the K1 epilogue. n = 0: the plain [B, sum_dim] output.
constexpr int kMaxPeers = 8;
struct PeerOut {
  float* base[kMaxPeers];
  int start[kMaxPeers + 1];
  int n;
};

struct SegParams {
  const DevTable* tabs;
  const int* unit_table;  // warp unit -> table position
  int n_units;
  int unit_begin;  // first unit handled by this launch
  const int* seg;  // segment key per element
  const int* src;  // gathered row per element
  // forward
  const float* W_ro;
  float* out;
  long long out_stride;
  double* loss;  // optional: += 1/2 sum of squares of the pooled rows
  PeerOut peers;
  // fp16 weight storage (bytes_per_param 2): W holds
  // __half (W_ro / W reinterpret), fp32 accumulation and update
  int w_half;
  // backward
  const float* grad;
  long long grad_stride;
  float* W;
  float* M;
  float lr, eps;
  // carries: [n_chunks][2][carry_stride] (0 = head, 1 = tail)
  float* carry;
  int carry_stride;
  // index staging per warp and buffer (ints), sized for the shard's widest layout
  int stage_x, stage_s;
  // chunks completing a segment that began in an earlier chunk: {chunk, table}
  int2* completers;
  int* n_completers;
  // completers of long segments: {chunk, table, k0, key}
  int4* completers_long;
  int* n_completers_long;
  // completers the per-lane fixup hands to the warp fixup (segment spans > 2
  // chunks, or rows wider than 32 floats): {chunk, table}
  int2* completers_mid;
  int* n_completers_mid;
};

}  // namespace asb
