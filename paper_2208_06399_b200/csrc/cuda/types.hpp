// Plain structs shared by the host context and the kernels.
#pragma once

#include <vector_types.h>

namespace asb {

// Per-table device descriptor (host-built, see context.cu).
struct DevTable {
  long long w_base;     // W element offset with row r (GLOBAL row id) at w_base + r*dim
  long long row_off;    // first global row of the table
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
  int kind;  // lane layout: 0..5 -> GL = 1<<kind, NV = 1; 6,7,8 -> GL = 32, NV = 2,4,8
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
};

}  // namespace asb
