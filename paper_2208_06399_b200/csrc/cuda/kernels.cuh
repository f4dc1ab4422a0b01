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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "types.hpp"

namespace asb {

// Packed fp32 pair add (FADD2 on sm_100a): IEEE round-to-nearest per element,
// bit-identical to two FADDs, half the issue slots.
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 r;
  asm("{\n.reg .b64 a, b, d;\n"
      "mov.b64 a, {%2, %3};\n"
      "mov.b64 b, {%4, %5};\n"
      "add.rn.f32x2 d, a, b;\n"
      "mov.b64 {%0, %1}, d;\n}\n"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
#ifdef ASB_NO_FADD2
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
#else
  const float2 lo = f2add(make_float2(a.x, a.y), make_float2(b.x, b.y));
  const float2 hi = f2add(make_float2(a.z, a.w), make_float2(b.z, b.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
#endif
}
// base + row * stride. ptxas splits a 64-bit-addend mad.wide.u32 into
// IMAD.WIDE.U32 + IADD3 + IMAD.X when the base does not sit in an aligned
// register pair; the carry-chained form (low word with carry-out, high word
// with carry-in) is two IMADs whatever the allocation.
__device__ __forceinline__ const char* row_addr(const char* base, unsigned row, unsigned stride) {
#ifdef ASB_MADWIDE_ADDR
  const char* r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(row), "r"(stride), "l"(base));
  return r;
#else
  const unsigned long long b = reinterpret_cast<unsigned long long>(base);
  unsigned lo, hi;
  asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\t"
      "madc.hi.u32 %1, %2, %3, %5;"
      : "=r"(lo), "=r"(hi)
      : "r"(row), "r"(stride), "r"(static_cast<unsigned>(b)), "r"(static_cast<unsigned>(b >> 32)));
  return reinterpret_cast<const char*>((static_cast<unsigned long long>(hi) << 32) | lo);
#endif
}
// U consecutive staged row ids (16-B aligned when U % 4 == 0) with vector LDS
template <int U>
__device__ __forceinline__ void lds_ids(const int* p, int (&x)[U]) {
  if constexpr (U % 4 == 0) {
#pragma unroll
    for (int i = 0; i < U / 4; ++i) {
      const int4 v = reinterpret_cast<const int4*>(p)[i];
      x[4 * i] = v.x;
      x[4 * i + 1] = v.y;
      x[4 * i + 2] = v.z;
      x[4 * i + 3] = v.w;
    }
  } else if constexpr (U == 2) {
    const int2 v = *reinterpret_cast<const int2*>(p);
    x[0] = v.x;
    x[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < U; ++i) x[i] = p[i];
  }
}
// The same from a 32-bit shared-window address: the staged ids / keys are
// addressed by one register per buffer instead of a generic pointer the
// compiler re-derives from %tid and the CTA's shared window at every batch
// (under the 64-register cap it rematerialised ~19 instructions per batch).
__device__ __forceinline__ int lds32(unsigned a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(unsigned a, int v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
template <int U>
__device__ __forceinline__ void lds_ids_sh(unsigned a, int (&x)[U]) {
  if constexpr (U % 4 == 0) {
#pragma unroll
    for (int i = 0; i < U / 4; ++i)
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(x[4 * i]), "=r"(x[4 * i + 1]), "=r"(x[4 * i + 2]), "=r"(x[4 * i + 3])
                   : "r"(a + 16u * i));
  } else if constexpr (U == 2) {
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(x[0]), "=r"(x[1]) : "r"(a));
  } else {
#pragma unroll
    for (int i = 0; i < U; ++i) x[i] = lds32(a + 4u * i);
  }
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
// fp16 weights: 4 halves (8 B) -> float4, and back with round-to-nearest
__device__ __forceinline__ float4 half4_to_float4(uint2 r) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&r.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&r.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ uint2 float4_to_half4(float4 v) {
  const __half2 a = __floats2half2_rn(v.x, v.y);
  const __half2 b = __floats2half2_rn(v.z, v.w);
  return make_uint2(*reinterpret_cast<const unsigned*>(&a), *reinterpret_cast<const unsigned*>(&b));
}
// 8 halves (16 B) -> two float4; zeros when !ok
__device__ __forceinline__ void gather8h(float4& a, float4& b, bool ok, const char* p) {
  if (ok) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
    a = half4_to_float4(make_uint2(r.x, r.y));
    b = half4_to_float4(make_uint2(r.z, r.w));
  } else {
    a = b = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}
__device__ __forceinline__ float4 ldg_h4(const char* p) {
  return half4_to_float4(__ldg(reinterpret_cast<const uint2*>(p)));
}
#ifdef ASB_L2HINTS
// backward epilogue rows (read once, written once per step): evict-first in L2
// so they do not push the gradient slabs of the tables in flight out
__device__ __forceinline__ float4 ld4_evict_first(const float* p) {
  float4 v;
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], pol;\n}\n"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}
__device__ __forceinline__ void st4_evict_first(float* p, float4 v) {
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, pol;\n}\n" ::"l"(p),
      "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
      : "memory");
}
#endif
// Row slice of W (cv-th float4 of row `seg`) in either storage type.
__device__ __forceinline__ float4 load_w4(const SegParams& p, const DevTable& tb, int seg, int cv) {
  const long long e = tb.w_base + (long long)seg * tb.dim + cv * 4;
  if (p.w_half) return half4_to_float4(*reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(p.W) + e));
#ifdef ASB_L2HINTS
  return ld4_evict_first(p.W + e);
#else
  return *reinterpret_cast<const float4*>(p.W + e);
#endif
}
__device__ __forceinline__ void store_w4(const SegParams& p, const DevTable& tb, int seg, int cv, float4 x) {
  const long long e = tb.w_base + (long long)seg * tb.dim + cv * 4;
  if (p.w_half)
    *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(p.W) + e) = float4_to_half4(x);
  else
#ifdef ASB_L2HINTS
    st4_evict_first(p.W + e, x);
#else
    *reinterpret_cast<float4*>(p.W + e) = x;
#endif
}

// L2 eviction priorities (ASB_L2HINTS): gathered rows (re-read ~L/U times)
// evict_last, the streamed index arrays evict_first.
__device__ __forceinline__ unsigned long long l2_policy_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 ldg4_hint(const float* p, unsigned long long pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
#ifdef ASB_L2HINTS
#define ASB_GPOL , gpol
template <bool HALF>
__device__ __forceinline__ float4 gather4(const char* p, unsigned long long pol) {
  if constexpr (HALF) return ldg_h4(p);
  return ldg4_hint(reinterpret_cast<const float*>(p), pol);
}
#else
#define ASB_GPOL
template <bool HALF>
__device__ __forceinline__ float4 gather4(const char* p) {
  if constexpr (HALF) return ldg_h4(p);
  return ldg4(reinterpret_cast<const float*>(p));
}
#endif
__device__ __forceinline__ void st4_streaming(float* p, float4 v) {
  __stcs(reinterpret_cast<float4*>(p), v);
}

template <int GL>
__device__ __forceinline__ unsigned low_bits() {
  return GL >= 32 ? 0xffffffffu : ((1u << GL) - 1u);
}

// Sum over the GL lanes of a group; `mask` = the group's lanes (all of them
// must be active, the caller's branch is group-uniform).
template <int GL>
__device__ __forceinline__ float group_sum(float x, unsigned mask) {
#pragma unroll
  for (int m = GL / 2; m >= 1; m >>= 1) x += __shfl_xor_sync(mask, x, m);
  return x;
}

// Row `b` of the pooled output: local [B, stride] buffer, or the receive
// buffer of the sample's owner (fused exchange, PeerOut).
__device__ __forceinline__ float* pooled_row(float* out, long long stride, const PeerOut& peers, int b) {
  if (peers.n == 0) return out + (long long)b * stride;
  int q = 0;
#pragma unroll
  for (int i = 1; i < kMaxPeers; ++i) q += (i < peers.n && b >= peers.start[i]) ? 1 : 0;
  return peers.base[q] + (long long)(b - peers.start[q]) * stride;
}

// Column group (4 columns) held in slot w of lane c. Standard layouts stride
// the slots by GL; PAIRED layouts (fp16 tables: one 16-B load = 8 halves per
// lane) hold two adjacent groups per load: slots 2k, 2k+1 = groups
// 2(c + k*GL), 2(c + k*GL) + 1.
template <int GL, bool PAIR>
__device__ __forceinline__ int colv(int c, int w) {
  if constexpr (PAIR) return 2 * (c + (w >> 1) * GL) + (w & 1);
  return c + w * GL;
}

// Segment epilogues, executed by the GL lanes of one group.
// forward : pooled[bag, col_t + :] = v   (+ loss 1/2|v|^2)
template <int GL, int NV, bool PAIR = false, bool EX = false>
__device__ __forceinline__ void store_pooled(const SegParams& p, const DevTable& tb, int seg, const float4 (&v)[NV],
                                             int c, float& loss_acc) {
  const int nvec = EX ? GL * NV : tb.dim >> 2;
  float* o = pooled_row(p.out, p.out_stride, p.peers, seg) + tb.col;
#pragma unroll
  for (int w = 0; w < NV; ++w) {
    const int cv = colv<GL, PAIR>(c, w);
    if (cv < nvec) {
      st4_streaming(o + cv * 4, v[w]);
      loss_acc += f4dot(v[w]);
    }
  }
}

template <int GL, int NV>
__device__ __forceinline__ void load_row_state(const SegParams& p, const DevTable& tb, int seg, int c,
                                               float4 (&w)[NV], float& m) {
  const int nvec = tb.dim >> 2;
  m = p.M[tb.row_off + seg];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const int cv = c + q * GL;
    w[q] = cv < nvec ? load_w4(p, tb, seg, cv) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// backward: m_r += |g|^2/D; W_r -= lr * g / (sqrt(m_r) + eps)  (FBGEMM exact row-wise Adagrad).
// w / m_old: the row's current weights and momentum (prefetched by the caller).
template <int GL, int NV>
__device__ __forceinline__ void adagrad_row(const SegParams& p, const DevTable& tb, unsigned gmask, int seg,
                                            const float4 (&g)[NV], int c, const float4 (&w)[NV], float m_old) {
  const int nvec = tb.dim >> 2;
  float sq = 0.f;
#pragma unroll
  for (int q = 0; q < NV; ++q)
    if (c + q * GL < nvec) sq += f4dot(g[q]);
  sq = group_sum<GL>(sq, gmask);
  const float m = m_old + sq / (float)tb.dim;
  const float mult = p.lr / (sqrtf(m) + p.eps);
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const int cv = c + q * GL;
    if (cv < nvec) {
      float4 x = w[q];
      x.x -= mult * g[q].x;
      x.y -= mult * g[q].y;
      x.z -= mult * g[q].z;
      x.w -= mult * g[q].w;
      store_w4(p, tb, seg, cv, x);
    }
  }
  if (c == 0) p.M[tb.row_off + seg] = m;
}

// Predicated variant for lane groups that run converged (GL < 32): every lane
// of the warp executes it (the group reduction needs them), `active` selects
// the groups whose segment ends here.
// `pre`: the row's state was prefetched into wp / mp (with the batch's gathers).
template <int GL, int NV>
__device__ __forceinline__ void adagrad_row_pred(const SegParams& p, const DevTable& tb, int seg, const float4 (&g)[NV],
                                                 int c, bool active, bool pre = false,
                                                 const float4 (*wp)[NV] = nullptr, float mp = 0.f) {
  const int nvec = tb.dim >> 2;
  float sq = 0.f;
#pragma unroll
  for (int q = 0; q < NV; ++q)
    if (c + q * GL < nvec) sq += f4dot(g[q]);
  sq = group_sum<GL>(sq, 0xffffffffu);
  if (active) {
    float4 w[NV];
    float m_old;
    if (pre) {
#pragma unroll
      for (int q = 0; q < NV; ++q) w[q] = (*wp)[q];
      m_old = mp;
    } else {
      load_row_state<GL, NV>(p, tb, seg, c, w, m_old);
    }
    const float m = m_old + sq / (float)tb.dim;
    const float mult = p.lr / (sqrtf(m) + p.eps);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int cv = c + q * GL;
      if (cv < nvec) {
        float4 x = w[q];
        x.x -= mult * g[q].x;
        x.y -= mult * g[q].y;
        x.z -= mult * g[q].z;
        x.w -= mult * g[q].w;
        store_w4(p, tb, seg, cv, x);
      }
    }
    if (c == 0) p.M[tb.row_off + seg] = m;
  }
}

template <bool FWD, int GL, int NV>
__device__ __forceinline__ void finish_segment(const SegParams& p, const DevTable& tb, unsigned gmask, int seg,
                                               const float4 (&v)[NV], int c, float& loss_acc) {
  if constexpr (FWD) {
    store_pooled<GL, NV>(p, tb, seg, v, c, loss_acc);
  } else {
    float4 w[NV];
    float m;
    load_row_state<GL, NV>(p, tb, seg, c, w, m);
    adagrad_row<GL, NV>(p, tb, gmask, seg, v, c, w, m);
  }
}

template <int GL, int NV, bool PAIR = false>
__device__ __forceinline__ void store_carry(const SegParams& p, int chunk, int which, int nvec, int c,
                                            const float4 (&v)[NV]) {
  float* dst = p.carry + ((long long)chunk * 2 + which) * p.carry_stride;
#pragma unroll
  for (int w = 0; w < NV; ++w) {
    const int cv = colv<GL, PAIR>(c, w);
    if (cv < nvec) *reinterpret_cast<float4*>(dst + cv * 4) = v[w];
  }
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
#ifdef ASB_L2HINTS
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem),
               "l"(l2_policy_first())
               : "memory");
#else
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async4_sh(unsigned s, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// One warp = one "unit" = 32/GL consecutive chunks of one table; each group
// of GL lanes walks its own chunk sequentially: gather a row, add it to the
// running sum, finish the segment when the key changes.
//
// Row ids and keys of each 32-element super-round are staged in shared
// memory with cp.async, double-buffered (the next super-round's indices are
// in flight while this one is gathered). Gathers are issued U at a time
// (U x 16 B per lane in flight, address = base + row * stride in one
// IMAD.WIDE.U32); a batch without a segment end is a plain run of adds, a
// batch with ends walks them with __ffs and ONE copy of the epilogue (small
// SASS, fits the instruction cache). The backward prefetches the weight row
// and momentum of the first segment ending in a batch together with the
// batch's gradient gathers.
#ifndef ASB_GATHER_U
#define ASB_GATHER_U 4
#endif
#ifndef ASB_GATHER_U_NARROW
#define ASB_GATHER_U_NARROW 4
#endif
constexpr int kSegWarps = 8;  // warps per CTA of the segment kernels
#ifdef ASB_IDX64
using EIdx = long long;
#else
using EIdx = int;  // element index inside a shard (< 2^31, enforced at staging)
#endif

// Staged ints per warp and buffer for lane layout `kind`: row ids R*SR, keys R*(SR+1).
__host__ __device__ constexpr int stage_sr(int kind) { return 8 * kind_gl(kind) < 32 ? 8 * kind_gl(kind) : 32; }
__host__ __device__ constexpr int stage_x_ints(int kind) { return (32 / kind_gl(kind)) * stage_sr(kind); }
__host__ __device__ constexpr int stage_s_ints(int kind) { return (32 / kind_gl(kind)) * (stage_sr(kind) + 1); }

// EXACT: dim == 4*GL*NV, so every lane owns a full column slice and the gathers
// need no column predicate.
#ifdef ASB_ABLATE_GATHER  // ablation builds only: every gather hits row 0 (L1-resident)
#define ASB_ROWID(x) (0u * (unsigned)(x))
#else
#define ASB_ROWID(x) ((unsigned)(x))
#endif
template <bool FWD, int GL, int NV, bool EXACT, bool HALF, bool PAIR_>
__device__ __forceinline__ void seg_unit(const SegParams& p, const DevTable& tb, int t, int unit, int* xs, int* ss) {
  // this layout's buffer sizes (compile-time; the warp's smem region is sized
  // by the host for the shard's widest layout, so these always fit)
  constexpr int kStageX = (32 / GL) * ((8 * GL < 32) ? 8 * GL : 32);
  constexpr int kStageS = (32 / GL) * (((8 * GL < 32) ? 8 * GL : 32) + 1);
  constexpr int R = 32 / GL;                       // chunks (groups) per warp
  constexpr int SR = (8 * GL < 32) ? 8 * GL : 32;  // elements per group per super-round
  constexpr int Q = SR / GL;                       // elements staged per lane per super-round
  // gathers in flight per lane (narrow rows: more, their warps walk several chunks)
  constexpr int UG = GL < 32 ? ASB_GATHER_U_NARROW : ASB_GATHER_U;
  constexpr int U = NV >= UG ? 1 : UG / NV;
  const int lane = threadIdx.x & 31;
  const int g = lane / GL;
  const int c = lane % GL;
  const unsigned gmask = low_bits<GL>() << (g * GL);
  // forward, EXACT layouts: the row width is a compile-time constant
  const int nvec = (FWD && EXACT) ? GL * NV : (tb.dim >> 2);
  const int C = tb.chunk_len;
  const int lchunk = (unit - tb.unit_off) * R + g;
  const int chunk = tb.chunk_off + lchunk;
  // element indices of the shard fit 32 bits (stage() rejects >= 2^31 lookups)
  const EIdx t_lo = (EIdx)tb.idx_off, t_hi = (EIdx)(tb.idx_off + tb.n_lookups);
  const EIdx j_lo = t_lo + (EIdx)lchunk * C;
  const EIdx j_hi = min(j_lo + (EIdx)C, t_hi);
  const bool live = j_lo < j_hi;
  const int prev_seg = (live && j_lo > t_lo) ? __ldg(p.seg + j_lo - 1) : -1;

  // gathered row = gbase + row_id * gstride (bytes): one IMAD.WIDE.U32 per gather
  const char* gbase;
  unsigned gstride;
  constexpr int VB = HALF ? 8 : 16;  // bytes of one lane's 4 columns
  // fp16 rows with dim % 8 == 0 get PAIRED layouts (kind_for_dim): one 16-B
  // load = 8 halves = slots w, w+1
  constexpr bool PAIR = FWD && HALF && (NV % 2 == 0) && PAIR_;
  if constexpr (FWD) {
    gbase = HALF ? reinterpret_cast<const char*>(reinterpret_cast<const __half*>(p.W_ro) + tb.w_base)
                 : reinterpret_cast<const char*>(p.W_ro + tb.w_base);
    gstride = EXACT ? (unsigned)(GL * NV * (HALF ? 8 : 16)) : (unsigned)tb.dim * (HALF ? 2u : 4u);
  } else {
    gbase = reinterpret_cast<const char*>(p.grad + tb.col);
    gstride = (unsigned)p.grad_stride * 4u;
  }
  gbase += PAIR ? c * 16 : c * VB;
#ifdef ASB_L2HINTS
  const unsigned long long gpol = l2_policy_last();
#endif

  // this group's staging buffers as 32-bit shared addresses (buffer 0; +kStage*4 B for buffer 1)
  const unsigned xsh = static_cast<unsigned>(__cvta_generic_to_shared(xs)) + 4u * (g * SR);
  const unsigned ssh = static_cast<unsigned>(__cvta_generic_to_shared(ss)) + 4u * (g * (SR + 1));
  // stage the row ids [base, base+SR) and keys [base, base+SR] of one super-round
  auto stage = [&](EIdx base, int buf) {
    const unsigned gx = xsh + 4u * (buf * kStageX);
    const unsigned gs = ssh + 4u * (buf * kStageS);
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int m = q * GL + c;
      const EIdx e = base + m;
      if (e < j_hi) cp_async4_sh(gx + 4u * m, p.src + e);
      if (e < t_hi)
        cp_async4_sh(gs + 4u * m, p.seg + e);
      else
        sts32(gs + 4u * m, -2);
    }
    if (c == 0) {
      const EIdx e = base + SR;
      if (e < t_hi)
        cp_async4_sh(gs + 4u * SR, p.seg + e);
      else
        sts32(gs + 4u * SR, -2);
    }
    cp_async_commit();
  };

  float4 acc[NV];
#pragma unroll
  for (int w = 0; w < NV; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
  float loss_acc = 0.f;
  bool hpend = false;  // this chunk ended a segment that began earlier (head carry stored)

  if (live)
    stage(j_lo, 0);
  else
    cp_async_commit();
  int buf = 0;
#pragma unroll 1
  for (int sr = 0; sr < C; sr += SR, buf ^= 1) {
    const EIdx base = j_lo + sr;
    if (base + SR < j_hi)
      stage(base + SR, buf ^ 1);
    else
      cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const unsigned gxa = xsh + 4u * (buf * kStageX);
    const unsigned gsa = ssh + 4u * (buf * kStageS);
    auto gs = [&](int k) { return lds32(gsa + 4u * k); };
    const int nval = (int)max((EIdx)0, min((EIdx)SR, j_hi - base));
    unsigned endm = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int m = q * GL + c;
      const bool end = m < nval && gs(m) != gs(m + 1);
      const unsigned be = __ballot_sync(0xffffffffu, end);
      endm |= ((be >> (g * GL)) & low_bits<GL>()) << (q * GL);
    }
    if (__ballot_sync(0xffffffffu, nval > 0) == 0) break;
#pragma unroll 1
    for (int m0 = 0; m0 < SR; m0 += U) {
      unsigned ebits = (endm >> m0) & low_bits<U>();
      float4 v[U][NV];
      int ids[U];
      lds_ids_sh<U>(gxa + 4u * m0, ids);
      if (m0 + U <= nval) {  // full batch: no element predicate
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const char* row = row_addr(gbase, ASB_ROWID(ids[u]), gstride);
          if constexpr (PAIR) {
#pragma unroll
            for (int w = 0; w < NV; w += 2)
              gather8h(v[u][w], v[u][w + 1], EXACT || colv<GL, true>(c, w) < nvec, row + (w >> 1) * GL * 16);
          } else {
#pragma unroll
            for (int w = 0; w < NV; ++w)
              v[u][w] = (EXACT || c + w * GL < nvec) ? gather4<HALF>(row + w * GL * VB ASB_GPOL)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = m0 + u < nval;
          const char* row = row_addr(gbase, ASB_ROWID(ids[u]), gstride);
          if constexpr (PAIR) {
#pragma unroll
            for (int w = 0; w < NV; w += 2)
              gather8h(v[u][w], v[u][w + 1], ok && (EXACT || colv<GL, true>(c, w) < nvec), row + (w >> 1) * GL * 16);
          } else {
#pragma unroll
            for (int w = 0; w < NV; ++w)
              v[u][w] = (ok && (EXACT || c + w * GL < nvec)) ? gather4<HALF>(row + w * GL * VB ASB_GPOL)
                                                             : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      if constexpr (GL < 32) {
        // several chunks per warp: stay converged, handle each element's
        // segment end with a warp-uniform test and predicated epilogues.
        // Backward: each group prefetches the row state of the first segment
        // ending in its batch (issued after the batch's gathers, so both
        // latencies overlap).
        float4 wpre[FWD ? 1 : NV];
        float mpre = 0.f;
        int spre = -7;
#ifndef ASB_NO_NARROW_PREFETCH
        if constexpr (!FWD) {
          if (ebits) {
            spre = gs(m0 + __ffs(ebits) - 1);
            if (spre != prev_seg) load_row_state<GL, NV>(p, tb, spre, c, wpre, mpre);
          }
        }
#endif
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int w = 0; w < NV; ++w) acc[w] = f4add(acc[w], v[u][w]);
          const bool endu = (ebits >> u) & 1u;
          if (__any_sync(0xffffffffu, endu)) {
            const int s = gs(m0 + u);
            const bool split = s == prev_seg;
            if (endu && split) {
              store_carry<GL, NV, PAIR>(p, chunk, 0, nvec, c, acc);
              hpend = true;  // finished at the chunk end (inline or via the fixup list)
            }
            if constexpr (FWD) {
              if (endu && !split) store_pooled<GL, NV, PAIR, EXACT>(p, tb, s, acc, c, loss_acc);
            } else {
              if constexpr (!FWD)
                adagrad_row_pred<GL, NV>(p, tb, s, acc, c, endu && !split, s == spre, &wpre, mpre);
            }
            if (endu) {
#pragma unroll
              for (int w = 0; w < NV; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
        }
      } else {
      // backward: the first segment ending in this batch gets its row state
      // fetched together with the gathers
      float4 wpre[FWD ? 1 : NV];
      float mpre = 0.f;
      int spre = -7;
      if constexpr (!FWD) {
        if (ebits) {
          spre = gs(m0 + __ffs(ebits) - 1);
          if (spre != prev_seg) load_row_state<GL, NV>(p, tb, spre, c, wpre, mpre);
        }
      }
        if (ebits == 0) {
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int w = 0; w < NV; ++w) acc[w] = f4add(acc[w], v[u][w]);
        } else {
          int u0 = 0;
          for (;;) {  // group-uniform
            const int e = ebits ? __ffs(ebits) - 1 : U;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (u >= u0 && u <= e)
#pragma unroll
                for (int w = 0; w < NV; ++w) acc[w] = f4add(acc[w], v[u][w]);
            if (e >= U) break;
            const int s = gs(m0 + e);
            if (s == prev_seg) {
              // completes a segment that began in an earlier chunk -> fixup
              store_carry<GL, NV, PAIR>(p, chunk, 0, nvec, c, acc);
              if (c == 0) p.completers[atomicAdd(p.n_completers, 1)] = make_int2(chunk, t);
            } else if constexpr (FWD) {
              store_pooled<GL, NV, PAIR, EXACT>(p, tb, s, acc, c, loss_acc);
            } else {
#ifdef ASB_ABLATE_EPILOGUE  // ablation builds only: write g, skip the row update
              if (c == 0) p.M[tb.row_off + s] = acc[0].x;
              if (false) {
#else
              if (s == spre) {
#endif
                adagrad_row<GL, NV>(p, tb, gmask, s, acc, c, wpre, mpre);
              } else {
                float4 wr[NV];
                float mr;
                load_row_state<GL, NV>(p, tb, s, c, wr, mr);
                adagrad_row<GL, NV>(p, tb, gmask, s, acc, c, wr, mr);
              }
            }
#pragma unroll
            for (int w = 0; w < NV; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
            ebits &= ebits - 1;
            u0 = e + 1;
          }
        }
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  // The chunk's last segment continues into the next chunk: hand the partial on
  // (tail: the segment started in this chunk; through: the whole chunk is
  // inside one segment).
  int ckind = 0;  // 1: tail, 2: through
  if (live && j_hi < t_hi) {
    const int sl = __ldg(p.seg + j_hi - 1);
    if (__ldg(p.seg + j_hi) == sl) {
      store_carry<GL, NV, PAIR>(p, chunk, sl == prev_seg ? 0 : 1, nvec, c, acc);
      ckind = sl == prev_seg ? 2 : 1;
    }
  }
  (void)ckind;
  if constexpr (GL < 32) {
    // A segment that began in the previous chunk and ended in this one, when
    // that chunk is the previous group of THIS warp and left a tail: finish it
    // here (tail[k-1] + head[k], the fixup's order; the warp barrier orders
    // the other group's carry stores) instead of queueing it for the fixups.
    __syncwarp();
    const int pred_kind = __shfl_sync(0xffffffffu, ckind, (lane - GL) & 31);
    const bool ready = hpend && g > 0 && pred_kind == 1;
    if (__any_sync(0xffffffffu, ready)) {
      float4 hv[NV];
      const float* tail = p.carry + ((long long)(chunk - 1) * 2 + 1) * p.carry_stride;
      const float* head = p.carry + ((long long)chunk * 2) * p.carry_stride;
#pragma unroll
      for (int w = 0; w < NV; ++w) {
        const int cv = colv<GL, PAIR>(c, w);
        hv[w] = (ready && cv < nvec) ? f4add(f4add(make_float4(0.f, 0.f, 0.f, 0.f),
                                                   *reinterpret_cast<const float4*>(tail + cv * 4)),
                                             *reinterpret_cast<const float4*>(head + cv * 4))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if constexpr (FWD) {
        if (ready) store_pooled<GL, NV, PAIR, EXACT>(p, tb, prev_seg, hv, c, loss_acc);
      } else {
        adagrad_row_pred<GL, NV>(p, tb, prev_seg, hv, c, ready);
      }
    }
    if (hpend && !ready && c == 0) p.completers[atomicAdd(p.n_completers, 1)] = make_int2(chunk, t);
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

#ifndef ASB_SEG_MINBLOCKS
#define ASB_SEG_MINBLOCKS 4
#endif
#ifndef ASB_SEG_MINBLOCKS_FWD
#define ASB_SEG_MINBLOCKS_FWD ASB_SEG_MINBLOCKS
#endif
#ifndef ASB_SEG_MINBLOCKS_BWD
#define ASB_SEG_MINBLOCKS_BWD ASB_SEG_MINBLOCKS
#endif
// fp16 forward: the paired 16-B layout for rows with dim % 8 == 0 (16-B
// aligned), the 8-B layout otherwise
template <bool FWD, int GL, int NV, bool EXACT, bool HALF>
__device__ __forceinline__ void seg_unit_d(const SegParams& p, const DevTable& tb, int t, int unit, int* x, int* s) {
  if constexpr (FWD && HALF && NV % 2 == 0) {
    if ((tb.dim & 7) == 0) {
      seg_unit<FWD, GL, NV, EXACT, HALF, true>(p, tb, t, unit, x, s);
      return;
    }
  }
  seg_unit<FWD, GL, NV, EXACT, HALF, false>(p, tb, t, unit, x, s);
}

template <bool FWD, bool HALF = false>
__global__ void __launch_bounds__(256, FWD ? ASB_SEG_MINBLOCKS_FWD : ASB_SEG_MINBLOCKS_BWD)
    seg_reduce_kernel(SegParams p) {
  // per warp: [2][stage_x] row ids then [2][stage_s] keys (sized on the host
  // for the widest lane layout present in the shard)
  extern __shared__ int seg_smem[];
  const int warp = threadIdx.x >> 5;
  const int unit = p.unit_begin + blockIdx.x * kSegWarps + warp;
  if (unit >= p.n_units) return;
  const int t = __ldg(p.unit_table + unit);
  const DevTable tb = p.tabs[t];
  int* x = seg_smem + warp * 2 * (p.stage_x + p.stage_s);
  int* s = x + 2 * p.stage_x;
  // lane layouts; "exact" widths (dim = 4*GL*NV) drop the column predicate
  const bool ex = tb.dim == 4 * kind_gl(tb.kind) * kind_nv(tb.kind);
#define ASB_SEG_CASE(K)                                                                  \
  case K:                                                                                \
    if (ex)                                                                              \
      seg_unit_d<FWD, kind_gl(K), kind_nv(K), true, HALF>(p, tb, t, unit, x, s);         \
    else                                                                                 \
      seg_unit_d<FWD, kind_gl(K), kind_nv(K), false, HALF>(p, tb, t, unit, x, s);        \
    break;
#ifdef ASB_ONLY_KIND  // register/spill study builds only
  switch (ASB_ONLY_KIND) {
    ASB_SEG_CASE(ASB_ONLY_KIND)
    default: break;
  }
  return;
#endif
  switch (tb.kind) {
    ASB_SEG_CASE(0)
    ASB_SEG_CASE(1)
    ASB_SEG_CASE(2)
    ASB_SEG_CASE(3)
    ASB_SEG_CASE(4)
    ASB_SEG_CASE(5)
    ASB_SEG_CASE(6)
    ASB_SEG_CASE(7)
    ASB_SEG_CASE(9)
    ASB_SEG_CASE(10)
    ASB_SEG_CASE(11)
    ASB_SEG_CASE(12)
    default:
      if (ex)
        seg_unit_d<FWD, 32, 8, true, HALF>(p, tb, t, unit, x, s);
      else
        seg_unit_d<FWD, 32, 8, false, HALF>(p, tb, t, unit, x, s);
      break;
  }
#undef ASB_SEG_CASE
}

// ---- fixups -----------------------------------------------------------------
// A completer chunk k finishes a segment that began in an earlier chunk k0;
// its value is tail[k0] + head[k0+1] + ... + head[k] (fixed order).
// k0 = k-1 is the common case (checked with one load); otherwise a 32-ary
// lower_bound over the sorted keys finds the segment's first element.
// Segments spanning <= kShortParts chunks are finished by one warp; longer
// ones (hot rows, very long bags) are queued for a CTA-wide reduction.
constexpr int kShortParts = 64;

__device__ __forceinline__ int find_k0(const SegParams& p, const DevTable& tb, int chunk, int first, int lane) {
  const long long t_lo = tb.idx_off;
  const long long jp = t_lo + (long long)(chunk - 1 - tb.chunk_off) * tb.chunk_len;  // start of chunk k-1
  if (jp == t_lo || __ldg(p.seg + jp - 1) != first) return chunk - 1;
  long long lo = t_lo, hi = jp - 1;  // lower_bound(first) lies in [lo, hi]
  while (hi - lo > 32) {
    const long long step = (hi - lo + 31) / 32;
    const long long q = lo + lane * step;
    const bool lt = q < hi && __ldg(p.seg + q) < first;
    const int cnt = __popc(__ballot_sync(0xffffffffu, lt));
    if (cnt == 0) {
      hi = lo;
    } else {
      if (cnt < 32 && lo + (long long)cnt * step < hi) hi = lo + (long long)cnt * step;
      lo = lo + (long long)(cnt - 1) * step + 1;
    }
  }
  const long long q = lo + lane;
  const bool lt = q < hi && __ldg(p.seg + q) < first;
  const long long p0 = lo + __popc(__ballot_sync(0xffffffffu, lt));
  return tb.chunk_off + (int)((p0 - t_lo) / tb.chunk_len);
}

__device__ __forceinline__ const float* carry_of(const SegParams& p, int k, int k0) {
  return p.carry + ((long long)k * 2 + (k == k0 ? 1 : 0)) * p.carry_stride;
}

template <bool FWD>
__device__ __forceinline__ void fixup_loss(const SegParams& p, float loss_acc, int lane) {
  if constexpr (FWD) {
    if (p.loss) {
      float l = loss_acc;
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) l += __shfl_xor_sync(0xffffffffu, l, m);
      if (lane == 0 && l != 0.f) atomicAdd(p.loss, 0.5 * (double)l);
    }
  }
}

// Thread per completer (the common case first): a segment that began in the
// previous chunk (k0 = k-1) of a table with rows of <= 32 floats is finished
// by ONE lane — tail[k-1] + head[k], then the epilogue over the row's <= 8
// float4 — so a warp finishes 32 of them with all their loads in flight.
// Anything else goes to the warp-per-completer kernel below.
template <bool FWD>
__global__ void __launch_bounds__(256, 4) seg_fixup_lane_kernel(SegParams p) {
  const int n = *p.n_completers;
  float loss_acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int2 ct = p.completers[i];
    const int chunk = ct.x;
    const DevTable& tb = p.tabs[ct.y];
    const int nvec = tb.dim >> 2;
    const long long t_lo = tb.idx_off;
    const long long j0 = t_lo + (long long)(chunk - tb.chunk_off) * tb.chunk_len;  // start of chunk k
    const int first = __ldg(p.seg + j0);
    const long long jp = j0 - tb.chunk_len;  // start of chunk k-1
    if (nvec > 8 || (jp != t_lo && __ldg(p.seg + jp - 1) == first)) {
      p.completers_mid[atomicAdd(p.n_completers_mid, 1)] = ct;
      continue;
    }
    const float* tail = carry_of(p, chunk - 1, chunk - 1);
    const float* head = carry_of(p, chunk, chunk - 1);
    float4 v[8];
#pragma unroll
    for (int w = 0; w < 8; ++w)
      v[w] = w < nvec ? f4add(f4add(make_float4(0.f, 0.f, 0.f, 0.f), *reinterpret_cast<const float4*>(tail + 4 * w)),
                              *reinterpret_cast<const float4*>(head + 4 * w))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (FWD) {
      store_pooled<1, 8>(p, tb, first, v, 0, loss_acc);
    } else {
      float4 w[8];
      float m_old;
      load_row_state<1, 8>(p, tb, first, 0, w, m_old);
      adagrad_row<1, 8>(p, tb, 1u << (threadIdx.x & 31), first, v, 0, w, m_old);
    }
  }
  fixup_loss<FWD>(p, loss_acc, threadIdx.x & 31);
}

// Warp per completer. Whole-warp lane layout: lane owns float4 columns lane + 32*w.
template <bool FWD>
__global__ void __launch_bounds__(256) seg_fixup_kernel(SegParams p) {
  const int lane = threadIdx.x & 31;
  const int n = *p.n_completers_mid;
  float loss_acc = 0.f;
  for (int i = blockIdx.x * 8 + (threadIdx.x >> 5); i < n; i += gridDim.x * 8) {
    const int2 ct = p.completers_mid[i];
    const int chunk = ct.x;
    const DevTable tb = p.tabs[ct.y];
    const int first = __ldg(p.seg + tb.idx_off + (long long)(chunk - tb.chunk_off) * tb.chunk_len);
    const int k0 = find_k0(p, tb, chunk, first, lane);
    if (chunk - k0 + 1 > kShortParts) {
      if (lane == 0) p.completers_long[atomicAdd(p.n_completers_long, 1)] = make_int4(chunk, ct.y, k0, first);
      continue;
    }
    const int nvec = tb.dim >> 2;
    float4 v[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) v[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nvec <= 32) {
      const bool on = lane < nvec;
      int k = k0;
      for (; k + 4 <= chunk + 1; k += 4) {  // 4 carries in flight
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        if (on) {
          a0 = *reinterpret_cast<const float4*>(carry_of(p, k, k0) + lane * 4);
          a1 = *reinterpret_cast<const float4*>(carry_of(p, k + 1, k0) + lane * 4);
          a2 = *reinterpret_cast<const float4*>(carry_of(p, k + 2, k0) + lane * 4);
          a3 = *reinterpret_cast<const float4*>(carry_of(p, k + 3, k0) + lane * 4);
        }
        v[0] = f4add(f4add(f4add(f4add(v[0], a0), a1), a2), a3);
      }
      for (; k <= chunk; ++k)
        if (on) v[0] = f4add(v[0], *reinterpret_cast<const float4*>(carry_of(p, k, k0) + lane * 4));
    } else {
      for (int k = k0; k <= chunk; ++k) {
        const float* src = carry_of(p, k, k0);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int cv = lane + 32 * w;
          if (cv < nvec) v[w] = f4add(v[w], *reinterpret_cast<const float4*>(src + cv * 4));
        }
      }
    }
    finish_segment<FWD, 32, 8>(p, tb, 0xffffffffu, first, v, lane, loss_acc);
  }
  fixup_loss<FWD>(p, loss_acc, lane);
}

// CTA per long segment: 8 warps sum contiguous ranges of the partials, then
// warp 0 combines them in warp order and runs the epilogue.
template <bool FWD>
__global__ void __launch_bounds__(256) seg_fixup_long_kernel(SegParams p) {
  __shared__ float4 part[8][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = *p.n_completers_long;
  float loss_acc = 0.f;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int4 ct = p.completers_long[i];
    const int chunk = ct.x, k0 = ct.z, first = ct.w;
    const DevTable tb = p.tabs[ct.y];
    const int nvec = tb.dim >> 2;
    const int nparts = chunk - k0 + 1;
    const int per = (nparts + 7) / 8;
    const int a = k0 + warp * per, b = min(chunk + 1, a + per);
    float4 v[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) v[w] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (nvec <= 32) {
      const bool on = lane < nvec;
      int k = a;
      for (; k + 8 <= b; k += 8) {
        float4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          x[u] = on ? *reinterpret_cast<const float4*>(carry_of(p, k + u, k0) + lane * 4)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u) v[0] = f4add(v[0], x[u]);
      }
      for (; k < b; ++k)
        if (on) v[0] = f4add(v[0], *reinterpret_cast<const float4*>(carry_of(p, k, k0) + lane * 4));
    } else {
      for (int k = a; k < b; ++k) {
        const float* src = carry_of(p, k, k0);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int cv = lane + 32 * w;
          if (cv < nvec) v[w] = f4add(v[w], *reinterpret_cast<const float4*>(src + cv * 4));
        }
      }
    }
#pragma unroll
    for (int w = 0; w < 8; ++w)
      if (lane + 32 * w < nvec) part[warp][lane + 32 * w] = v[w];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const int cv = lane + 32 * w;
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cv < nvec)
          for (int q = 0; q < 8; ++q) s = f4add(s, part[q][cv]);
        v[w] = s;
      }
      finish_segment<FWD, 32, 8>(p, tb, 0xffffffffu, first, v, lane, loss_acc);
    }
    __syncthreads();
  }
  if (warp == 0) fixup_loss<FWD>(p, loss_acc, lane);
}

// K4: bag id per lookup from the offsets; empty bags get a zero pooled row
// here (they have no elements for the segmented reduce). One warp per 32
// consecutive (table, bag) pairs: lane i holds bag i's end offset, and the
// warp walks the bags' element range 32 elements at a time, each lane finding
// its element's bag with a 5-step shuffle binary search over the lanes' ends
// (coalesced stores; no per-bag serial loop).
__global__ void __launch_bounds__(256) bag_expand_kernel(const int* __restrict__ off, int T, int B,
                                                         const DevTable* __restrict__ tabs,
                                                         int* __restrict__ bag, float* __restrict__ out,
                                                         long long out_stride, PeerOut peers) {
#ifdef ASB_K4_OLD
  const long long nb = (long long)T * B;
  const long long w0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  if (w0 >= nb) return;
  const int lane = threadIdx.x & 31;
  const long long gb = min(w0 + lane, nb - 1);  // lanes past the end repeat the last bag
  const int t = (int)(gb / B);
  const int b = (int)(gb - (long long)t * B);
#else
  // T*B + 1 offsets are int32-indexed (staging): 32-bit bag arithmetic
  const int nb = T * B;
  const int w0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  if (w0 >= nb) return;
  const int lane = threadIdx.x & 31;
  const int gb = min(w0 + lane, nb - 1);  // lanes past the end repeat the last bag
  const int t = gb / B;
  const int b = gb - t * B;
#endif
  const int o = __ldg(off + gb);
  const int e = __ldg(off + gb + 1);
  const int first = __shfl_sync(0xffffffffu, o, 0);
  const int last = __shfl_sync(0xffffffffu, e, 31);
  for (int base = first; base < last; base += 32) {
    const int j = base + lane;
    // number of lanes whose bag ends at or before j = j's bag (ends ascending)
    int lo = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
      const int v = __shfl_sync(0xffffffffu, e, lo + step - 1);
      if (v <= j) lo += step;
    }
    const int bj = __shfl_sync(0xffffffffu, b, lo);
    if (j < last) bag[j] = bj;
  }
  if (out == nullptr) return;  // ids only (backward without a forward of this batch)
#ifdef ASB_K4_OLD
  unsigned empty = __ballot_sync(0xffffffffu, w0 + lane < nb && o == e);
#else
  // zero rows of empty bags: rows of <= 32 floats by their own lane (all
  // empty bags of the warp at once), wider rows by the whole warp
  const bool is_empty = w0 + lane < nb && o == e;
  const int nv_mine = is_empty ? (__ldg(&tabs[t].dim) >> 2) : 0;
  if (is_empty && nv_mine <= 8) {
    float* row = pooled_row(out, out_stride, peers, b) + __ldg(&tabs[t].col);
    for (int cv = 0; cv < nv_mine; ++cv) st4_streaming(row + cv * 4, make_float4(0.f, 0.f, 0.f, 0.f));
  }
  unsigned empty = __ballot_sync(0xffffffffu, is_empty && nv_mine > 8);
#endif
  while (empty) {
    const int i = __ffs(empty) - 1;
    empty &= empty - 1;
    const int ti = __shfl_sync(0xffffffffu, t, i);
    const int bi = __shfl_sync(0xffffffffu, b, i);
    const int nvec = tabs[ti].dim >> 2;
    float* row = pooled_row(out, out_stride, peers, bi) + tabs[ti].col;
    for (int cv = lane; cv < nvec; cv += 32) st4_streaming(row + cv * 4, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// ---- cost-model features from the sorted keys ----------
// For every segment end of the sorted (row, bag) list: occurrence count of the
// row = end - lower_bound(row) + 1 within its table, binned like
// detail::frequency_bin (tables.hpp:317-324): (0,1], (1,2], (2,4], ...,
// (32768, inf) -> 17 bins. hist[t][17] counts rows per bin, hist[t][17] is
// unused; distinct[t] counts unique rows.
__global__ void row_count_hist_kernel(const int* __restrict__ skey, const long long* __restrict__ t_start, int T,
                                      long long L, unsigned long long* __restrict__ hist) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < L; j += (long long)gridDim.x * blockDim.x) {
    // table of element j: last t with t_start[t] <= j (t_start ascending, T+1 entries)
    int lo = 0, hi = T;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (t_start[mid] <= j) lo = mid; else hi = mid;
    }
    const long long t_hi = t_start[lo + 1];
    const int k = skey[j];
    if (j + 1 < t_hi && skey[j + 1] == k) continue;  // not the last occurrence
    long long a = t_start[lo], b = j;  // first occurrence of k in [a, b]
    while (a < b) {
      const long long m = (a + b) >> 1;
      if (skey[m] < k) a = m + 1; else b = m;
    }
    const long long c = j - a + 1;
    int bin = 0;
    if (c > 1) {
      bin = 64 - __clzll((unsigned long long)(c - 1));
      if (bin > 16) bin = 16;
    }
    atomicAdd(hist + (long long)lo * 18 + bin, 1ull);
    atomicAdd(hist + (long long)lo * 18 + 17, 1ull);
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
// The grid values k*2^-12, |k| <= 512, are exact in fp16 too (HALF storage).
template <bool HALF>
__global__ void init_table_kernel(void* __restrict__ Wv, long long rows, int dim, int table_id,
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
    if constexpr (HALF)
      reinterpret_cast<uint2*>(Wv)[q] = float4_to_half4(x);
    else
      reinterpret_cast<float4*>(Wv)[q] = x;
  }
}

}  // namespace asb
