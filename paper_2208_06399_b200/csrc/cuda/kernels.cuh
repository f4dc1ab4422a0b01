// sm_100a kernels of the embedding-bag hot path.
//
// The forward (sum pooling) and the backward (segment-sum + exact row-wise
// Adagrad) are the SAME segmented gather-reduce over a CSR-like element list:
//
//             element j            segment key seg[j]        gathered row src[j]
//   forward   lookup j             bag id (ascending)        W_t[idx_j, :]
//   backward  j-th sorted lookup   global row (ascending)    G[bag_j, col_t:+dim_t]
//
// The element list of each table is cut into fixed-length chunks (one warp
// each), so a 100k-lookup bag or a 1M-occurrence hot row is spread over many
// warps; partial sums of segments that cross a chunk edge go to per-chunk
// head/tail carries and a fixup pass finishes them in a fixed order
// (deterministic, no float atomics). Inside a warp, D/4 lanes own one 16-byte
// column slice each and 32/(D/4) elements are gathered per round; segments
// inside a round are combined with a shuffle segmented scan.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "types.hpp"

namespace asb {

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float f4dot(float4 a) { return a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w; }
__device__ __forceinline__ float4 shfl4(float4 v, int src) {
  return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                     __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}
__device__ __forceinline__ float4 shfl4_up(float4 v, int d) {
  return make_float4(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d),
                     __shfl_up_sync(0xffffffffu, v.z, d), __shfl_up_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4_streaming(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}

// Group (GL lanes) sum, every lane of the warp participates.
template <int GL>
__device__ __forceinline__ float group_sum(float x) {
#pragma unroll
  for (int m = GL / 2; m >= 1; m >>= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
  return x;
}

// Segment epilogue, executed by the GL lanes of one group (predicated by
// `active`, all lanes call it so the group reduction stays converged).
template <bool FWD, int GL, int NV>
__device__ __forceinline__ void finish_segment(const SegParams& p, const DevTable& tb, bool active,
                                               int seg, const float4 (&v)[NV], int c,
                                               float& loss_acc) {
  const int nvec = tb.dim >> 2;
  if constexpr (FWD) {
    if (active) {
      float* o = p.out + (long long)seg * p.out_stride + tb.col;
#pragma unroll
      for (int w = 0; w < NV; ++w) {
        const int cv = c + w * GL;
        if (cv < nvec) {
          st4_streaming(o + cv * 4, v[w]);
          loss_acc += f4dot(v[w]);
        }
      }
    }
  } else {
    float sq = 0.f;
#pragma unroll
    for (int w = 0; w < NV; ++w)
      if (c + w * GL < nvec) sq += f4dot(v[w]);
    sq = group_sum<GL>(sq);
    if (active) {
      // exact row-wise Adagrad (FBGEMM semantics): m += |g|^2/D; W -= lr*g/(sqrt(m)+eps)
      const float m = p.M[seg] + sq / (float)tb.dim;
      const float mult = p.lr / (sqrtf(m) + p.eps);
      float* wr = p.W + tb.w_base + (long long)seg * tb.dim;
#pragma unroll
      for (int w = 0; w < NV; ++w) {
        const int cv = c + w * GL;
        if (cv < nvec) {
          float4* q = reinterpret_cast<float4*>(wr + cv * 4);
          float4 x = *q;
          x.x -= mult * v[w].x;
          x.y -= mult * v[w].y;
          x.z -= mult * v[w].z;
          x.w -= mult * v[w].w;
          *q = x;
        }
      }
      if (c == 0) p.M[seg] = m;
    }
  }
}

template <int NV>
__device__ __forceinline__ void store_carry(const SegParams& p, int chunk, int which, int nvec, int GL,
                                            int c, const float4 (&v)[NV]) {
  float* dst = p.carry + ((long long)chunk * 2 + which) * p.carry_stride;
#pragma unroll
  for (int w = 0; w < NV; ++w) {
    const int cv = c + w * GL;
    if (cv < nvec) *reinterpret_cast<float4*>(dst + cv * 4) = v[w];
  }
}

// One warp reduces one chunk of one table.
template <bool FWD, int GL, int NV>
__device__ __forceinline__ void seg_chunk(const SegParams& p, const DevTable& tb, int chunk) {
  constexpr int R = 32 / GL;   // elements per round
  constexpr int RS = GL;       // rounds per 32-element super-round
  constexpr int U = (RS < 8 / NV ? RS : (8 / NV > 0 ? 8 / NV : 1));  // rounds per load batch
  const int lane = threadIdx.x & 31;
  const int g = lane / GL;
  const int c = lane % GL;
  const int nvec = tb.dim >> 2;
  const long long t_lo = tb.idx_off, t_hi = tb.idx_off + tb.n_lookups;
  const long long j_lo = t_lo + (long long)(chunk - tb.chunk_off) * tb.chunk_len;
  const long long j_hi = min(j_lo + (long long)tb.chunk_len, t_hi);
  if (j_lo >= j_hi) return;
  const int prev_seg = j_lo > t_lo ? __ldg(p.seg + j_lo - 1) : -1;
  const int next_seg = j_hi < t_hi ? __ldg(p.seg + j_hi) : -2;

  const float* gbase;
  long long gstride;
  if constexpr (FWD) {
    gbase = p.W_ro + tb.w_base;
    gstride = tb.dim;
  } else {
    gbase = p.grad + tb.col;
    gstride = p.grad_stride;
  }

  float4 carry[NV];
#pragma unroll
  for (int w = 0; w < NV; ++w) carry[w] = make_float4(0.f, 0.f, 0.f, 0.f);
  int carry_seg = -3;
  float loss_acc = 0.f;

  for (long long e0 = j_lo; e0 < j_hi; e0 += 32) {
    const long long e = e0 + lane;
    const int my_seg = e < j_hi ? __ldg(p.seg + e) : -4;
    const int my_src = e < j_hi ? __ldg(p.src + e) : 0;
    const int my_nxt = e + 1 < j_hi ? __ldg(p.seg + e + 1) : (e + 1 == j_hi ? next_seg : -5);
    const int n_here = (int)min(32LL, j_hi - e0);

#pragma unroll 1
    for (int rb = 0; rb < RS; rb += U) {
      float4 v[U][NV];
      int s[U], nx[U];
      // issue all gathers of the batch first (memory-level parallelism)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = (rb + u) * R + g;
        s[u] = __shfl_sync(0xffffffffu, my_seg, i);
        nx[u] = __shfl_sync(0xffffffffu, my_nxt, i);
        const int x = __shfl_sync(0xffffffffu, my_src, i);
        const bool ok = i < n_here;
        const float* row = gbase + (long long)x * gstride;
#pragma unroll
        for (int w = 0; w < NV; ++w) {
          const int cv = c + w * GL;
          v[u][w] = (ok && cv < nvec) ? ldg4(row + cv * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = (rb + u) * R + g;
        const bool ok = i < n_here;
        // segmented inclusive scan across the R groups of this round
#pragma unroll
        for (int off = 1; off < R; off <<= 1) {
          const int so = __shfl_up_sync(0xffffffffu, s[u], off * GL);
#pragma unroll
          for (int w = 0; w < NV; ++w) {
            const float4 t = shfl4_up(v[u][w], off * GL);
            if (g >= off && so == s[u]) v[u][w] = f4add(v[u][w], t);
          }
        }
        if (s[u] == carry_seg) {
#pragma unroll
          for (int w = 0; w < NV; ++w) v[u][w] = f4add(v[u][w], carry[w]);
        }
        const bool ends = ok && nx[u] != s[u];
        const bool cont = ok && (e0 + i == j_hi - 1) && nx[u] == s[u];
        const bool split_left = s[u] == prev_seg;
        // complete segments: epilogue; split ones: carries for the fixup
        finish_segment<FWD, GL, NV>(p, tb, ends && !split_left, s[u], v[u], c, loss_acc);
        if ((ends || cont) && split_left) store_carry<NV>(p, chunk, 0, nvec, GL, c, v[u]);
        if (cont && !split_left) store_carry<NV>(p, chunk, 1, nvec, GL, c, v[u]);
        // carry-out from the last group of the round
        const int lsrc = (R - 1) * GL + c;
#pragma unroll
        for (int w = 0; w < NV; ++w) carry[w] = shfl4(v[u][w], lsrc);
        const int cs = __shfl_sync(0xffffffffu, s[u], lsrc);
        const bool ce = __shfl_sync(0xffffffffu, (int)ends, lsrc) != 0;
        carry_seg = ce ? -3 : cs;
      }
    }
  }
  if constexpr (FWD) {
    if (p.loss) {
      float l = loss_acc;
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) l += __shfl_xor_sync(0xffffffffu, l, m);
      if (lane == 0 && l != 0.f) atomicAdd(p.loss, 0.5 * (double)l);
    }
  }
}

template <bool FWD>
__global__ void __launch_bounds__(256) seg_reduce_kernel(SegParams p) {
  const int chunk = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (chunk >= p.n_chunks) return;
  const DevTable tb = p.tabs[__ldg(p.chunk_table + chunk)];
  switch (tb.kind) {
    case 0: seg_chunk<FWD, 1, 1>(p, tb, chunk); break;
    case 1: seg_chunk<FWD, 2, 1>(p, tb, chunk); break;
    case 2: seg_chunk<FWD, 4, 1>(p, tb, chunk); break;
    case 3: seg_chunk<FWD, 8, 1>(p, tb, chunk); break;
    case 4: seg_chunk<FWD, 16, 1>(p, tb, chunk); break;
    case 5: seg_chunk<FWD, 32, 1>(p, tb, chunk); break;
    case 6: seg_chunk<FWD, 32, 2>(p, tb, chunk); break;
    case 7: seg_chunk<FWD, 32, 4>(p, tb, chunk); break;
    default: seg_chunk<FWD, 32, 8>(p, tb, chunk); break;
  }
}

// Fixup: one warp per chunk. The chunk that COMPLETES a segment which began
// in an earlier chunk sums tail[k0] + head[k0+1..k] in chunk order and runs
// the epilogue. Whole-warp lane layout: lane owns float4 columns lane+32*w.
template <bool FWD>
__global__ void __launch_bounds__(256) seg_fixup_kernel(SegParams p) {
  const int chunk = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (chunk >= p.n_chunks) return;
  const int lane = threadIdx.x & 31;
  const DevTable tb = p.tabs[__ldg(p.chunk_table + chunk)];
  const long long t_lo = tb.idx_off, t_hi = tb.idx_off + tb.n_lookups;
  const long long j_lo = t_lo + (long long)(chunk - tb.chunk_off) * tb.chunk_len;
  const long long j_hi = min(j_lo + (long long)tb.chunk_len, t_hi);
  if (j_lo >= j_hi || j_lo == t_lo) return;
  const int first = __ldg(p.seg + j_lo);
  if (__ldg(p.seg + j_lo - 1) != first) return;  // not split on the left
  if (j_hi < t_hi && __ldg(p.seg + j_hi) == first && __ldg(p.seg + j_hi - 1) == first) return;  // middle
  // find k0: walk back over middle chunks (warp-parallel, 32 chunks per probe)
  int k0 = -1;
  for (int base = chunk - 1; k0 < 0; base -= 32) {
    const int k = base - lane;
    bool mid = false;
    if (k >= tb.chunk_off) {
      const long long jl = t_lo + (long long)(k - tb.chunk_off) * tb.chunk_len;
      mid = jl > t_lo && __ldg(p.seg + jl - 1) == first;
    }
    const unsigned notmid = __ballot_sync(0xffffffffu, !mid);
    if (notmid) k0 = base - (__ffs(notmid) - 1);
  }
  const int nvec = tb.dim >> 2;
  float4 v[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) v[w] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k = k0; k <= chunk; ++k) {
    const float* src = p.carry + ((long long)k * 2 + (k == k0 ? 1 : 0)) * p.carry_stride;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int cv = lane + 32 * w;
      if (cv < nvec) v[w] = f4add(v[w], *reinterpret_cast<const float4*>(src + cv * 4));
    }
  }
  float loss_acc = 0.f;
  finish_segment<FWD, 32, 8>(p, tb, true, first, v, lane, loss_acc);
  if constexpr (FWD) {
    if (p.loss) {
      float l = loss_acc;
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) l += __shfl_xor_sync(0xffffffffu, l, m);
      if (lane == 0 && l != 0.f) atomicAdd(p.loss, 0.5 * (double)l);
    }
  }
}

// K4: bag id per lookup from the offsets; empty bags get a zero pooled row
// here (they have no elements for the segmented reduce). One warp per 32
// consecutive (table, bag) pairs.
__global__ void __launch_bounds__(256) bag_expand_kernel(const int* __restrict__ off, int T, int B,
                                                         const DevTable* __restrict__ tabs,
                                                         int* __restrict__ bag, float* __restrict__ out,
                                                         long long out_stride) {
  const long long nb = (long long)T * B;
  const long long w0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  if (w0 >= nb) return;
  const int lane = threadIdx.x & 31;
  const long long gb = w0 + lane;
  int o = 0, len = 0, b = 0, t = 0;
  if (gb < nb) {
    o = __ldg(off + gb);
    len = __ldg(off + gb + 1) - o;
    t = (int)(gb / B);
    b = (int)(gb - (long long)t * B);
  }
  const int n = (int)min(32LL, nb - w0);
  for (int i = 0; i < n; ++i) {
    const int li = __shfl_sync(0xffffffffu, len, i);
    const int oi = __shfl_sync(0xffffffffu, o, i);
    const int bi = __shfl_sync(0xffffffffu, b, i);
    if (li > 0) {
      for (int k = lane; k < li; k += 32) bag[oi + k] = bi;
    } else {
      const int ti = __shfl_sync(0xffffffffu, t, i);
      const int nvec = tabs[ti].dim >> 2;
      float* row = out + (long long)bi * out_stride + tabs[ti].col;
      for (int cv = lane; cv < nvec; cv += 32) st4_streaming(row + cv * 4, make_float4(0.f, 0.f, 0.f, 0.f));
    }
  }
}

// ---- stream packing / validation (load_workload checks on the device) ----
// Error key: (table position << 42) | (kind << 40) | entry; the smallest wins.
// kind 0: offsets[0] != 0, 1: decreasing offset, 2: final offset != count,
// 3: index out of [0, hash).
__global__ void pack_offsets_kernel(const long long* __restrict__ off64, int T, int B,
                                    const DevTable* __restrict__ tabs, int* __restrict__ off32,
                                    unsigned long long* __restrict__ err) {
  const long long n = (long long)T * (B + 1);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(e / (B + 1));
    const int q = (int)(e - (long long)t * (B + 1));
    const long long o = off64[e];
    int kind = -1;
    if (q == 0) {
      if (o != 0) kind = 0;
    } else if (o < off64[e - 1]) {
      kind = 1;
    }
    if (kind < 0 && q == B && o != tabs[t].n_lookups) kind = 2;
    if (kind >= 0) {
      atomicMin(err, ((unsigned long long)t << 42) | ((unsigned long long)kind << 40) | (unsigned long long)q);
    } else if (q < B) {
      off32[(long long)t * B + q] = (int)(tabs[t].idx_off + o);
    } else if (t == T - 1) {
      off32[(long long)T * B] = (int)(tabs[t].idx_off + o);
    }
  }
}

__global__ void __launch_bounds__(256) pack_indices_kernel(const long long* __restrict__ idx64,
                                                           const DevTable* __restrict__ tabs,
                                                           const int* __restrict__ chunk_table,
                                                           int n_chunks, int* __restrict__ idx32,
                                                           unsigned long long* __restrict__ err) {
  const int chunk = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (chunk >= n_chunks) return;
  const int lane = threadIdx.x & 31;
  const int t = chunk_table[chunk];
  const DevTable tb = tabs[t];
  const long long j_lo = tb.idx_off + (long long)(chunk - tb.chunk_off) * tb.chunk_len;
  const long long j_hi = min(j_lo + (long long)tb.chunk_len, tb.idx_off + tb.n_lookups);
  for (long long j = j_lo + lane; j < j_hi; j += 32) {
    const long long v = idx64[j];
    if (v < 0 || v >= tb.hash) {
      atomicMin(err, ((unsigned long long)t << 42) | (3ull << 40) | (unsigned long long)(j - tb.idx_off));
    } else {
      idx32[j] = (int)(tb.row_off + v);
    }
  }
}

// ---- K6: counter-hash init (bit-identical to oracle/oracle.c) -------------
__device__ __forceinline__ unsigned long long dev_splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float grid_value(unsigned long long h) {
  return (float)((int)(h >> 54) - 512) * 0x1.0p-12f;
}

// W_t[r, d] for one table; s0 = splitmix64(seed) precomputed on the host.
__global__ void init_table_kernel(float* __restrict__ W, long long rows, int dim, int table_id,
                                  unsigned long long s0) {
  const long long nv = rows * (dim >> 2);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nv;
       q += (long long)gridDim.x * blockDim.x) {
    const long long r = q / (dim >> 2);
    const int d0 = (int)(q - r * (dim >> 2)) * 4;
    const unsigned long long base =
        ((unsigned long long)(unsigned)table_id << 40) | ((unsigned long long)r << 10);
    float4 x;
    x.x = grid_value(dev_splitmix64(s0 ^ (base | (unsigned long long)(d0 + 0))));
    x.y = grid_value(dev_splitmix64(s0 ^ (base | (unsigned long long)(d0 + 1))));
    x.z = grid_value(dev_splitmix64(s0 ^ (base | (unsigned long long)(d0 + 2))));
    x.w = grid_value(dev_splitmix64(s0 ^ (base | (unsigned long long)(d0 + 3))));
    reinterpret_cast<float4*>(W)[q] = x;
  }
}

}  // namespace asb
