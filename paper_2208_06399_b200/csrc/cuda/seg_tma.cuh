// TMA-gather variant of the segmented reduce for rows of 100..1024 floats
// (lane layouts GL = 32, NV = 1/2/4/8): the whole warp walks one chunk.
//
// Rows are fetched with bulk async copies (cp.async.bulk ... complete_tx,
// the TMA engine; one lane issues one row) into a ring of kSlots slots of
// kRows(NV) rows in shared memory, completion tracked by one mbarrier per
// slot. The warp consumes slot k (LDS.128 per lane, adds, segment epilogues)
// while slots k+1 .. k+kSlots-1 are in flight, so memory-level parallelism
// no longer costs registers: ~16 KB per warp in flight versus 2 KB with
// register-held LDG batches. Row ids / keys of the batch after next are
// prefetched into registers one iteration ahead. Semantics (segments, carries,
// completers, epilogues) are identical to seg_unit (kernels.cuh).
#pragma once

#include "kernels.cuh"

namespace asb {

constexpr int kTmaWarps = 4;   // warps per CTA of the TMA kernels
constexpr int kTmaSlots = 3;   // ring depth per warp
__host__ __device__ constexpr int tma_rows(int nv) { return 16 / nv; }  // rows per slot: 8 KB at dim 128 * nv
constexpr int kTmaSlotBytes = 8192;
// per warp: ring + keys [slots][rows+1] + end masks [slots] + mbarriers [slots]
constexpr int kTmaWarpBytes = kTmaSlots * kTmaSlotBytes + 256;
constexpr int kTmaSmemBytes = kTmaWarps * kTmaWarpBytes;

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <bool FWD, int NV>
__device__ __forceinline__ void seg_unit_tma(const SegParams& p, const DevTable& tb, int t, int unit, char* wsm) {
  constexpr int GL = 32;
  constexpr int B = tma_rows(NV);
  constexpr int NS = kTmaSlots;
  const int lane = threadIdx.x & 31;
  const int nvec = tb.dim >> 2;
  const unsigned rb = (unsigned)tb.dim * 4u;  // row bytes (multiple of 16)
  const int C = tb.chunk_len;
  const int chunk = tb.chunk_off + (unit - tb.unit_off);
  const long long t_lo = tb.idx_off, t_hi = tb.idx_off + tb.n_lookups;
  const long long j_lo = t_lo + (long long)(unit - tb.unit_off) * C;
  const long long j_hi = min(j_lo + (long long)C, t_hi);
  if (j_lo >= j_hi) return;
  const int prev_seg = j_lo > t_lo ? __ldg(p.seg + j_lo - 1) : -1;
  const int nb = (int)((j_hi - j_lo + B - 1) / B);

  float* ring = reinterpret_cast<float*>(wsm);
  int* keys = reinterpret_cast<int*>(wsm + NS * kTmaSlotBytes);  // [NS][B+1]
  unsigned* masks = reinterpret_cast<unsigned*>(keys + NS * (B + 1));
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(wsm + NS * kTmaSlotBytes + 256 - NS * sizeof(unsigned long long));

  const char* gbase;
  size_t gstride;  // bytes
  if constexpr (FWD) {
    gbase = reinterpret_cast<const char*>(p.W_ro + tb.w_base);
    gstride = rb;
  } else {
    gbase = reinterpret_cast<const char*>(p.grad + tb.col);
    gstride = (size_t)p.grad_stride * 4u;
  }

  if (lane < NS) mbar_init(&bars[lane], 1);
  fence_mbar_init();
  __syncwarp();

  // ids of one batch: lane u < B holds element u's row id and key
  int rx = 0, rs = -4, rsn = -5;
  auto load_ids = [&](int b) {
    const long long e = j_lo + (long long)b * B + lane;
    rx = 0;
    rs = -4;
    rsn = -5;
    if (lane < B && b < nb && e < j_hi) {
      rx = __ldg(p.src + e);
      rs = __ldg(p.seg + e);
      rsn = e + 1 < t_hi ? __ldg(p.seg + e + 1) : -2;
    }
  };
  auto issue = [&](int b) {  // batch b -> slot b % NS, ids in rx/rs/rsn
    const int sl = b % NS;
    const long long e = j_lo + (long long)b * B + lane;
    const bool ok = lane < B && e < j_hi;
    const unsigned em = __ballot_sync(0xffffffffu, ok && rs != rsn);
    const int nval = (int)min((long long)B, j_hi - (j_lo + (long long)b * B));
    if (lane < B) keys[sl * (B + 1) + lane] = rs;
    if (lane == 0) {
      masks[sl] = em;
      mbar_arrive_expect(&bars[sl], (unsigned)nval * rb);
    }
    __syncwarp();
    if (ok) bulk_g2s(ring + (size_t)(sl * B + lane) * tb.dim, gbase + (size_t)(unsigned)rx * gstride, rb, &bars[sl]);
  };

  // prologue: slots 0..NS-1 in flight, ids of batch NS in registers
  load_ids(0);
  for (int b = 0; b < NS; ++b) {
    if (b < nb) issue(b);
    load_ids(b + 1);
  }

  float4 acc[NV];
#pragma unroll
  for (int w = 0; w < NV; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
  float loss_acc = 0.f;

#pragma unroll 1
  for (int k = 0; k < nb; ++k) {
    const int sl = k % NS;
    mbar_wait(&bars[sl], (unsigned)((k / NS) & 1));
    const float* rows = ring + (size_t)sl * B * tb.dim;
    const int* ks = keys + sl * (B + 1);
    unsigned ebits = masks[sl];
    const int nval = (int)min((long long)B, j_hi - (j_lo + (long long)k * B));
    // backward: fetch the row state of the first segment ending in this batch early
    float4 wpre[FWD ? 1 : NV];
    float mpre = 0.f;
    int spre = -7;
    if constexpr (!FWD) {
      if (ebits) {
        spre = ks[__ffs(ebits) - 1];
        if (spre != prev_seg) load_row_state<GL, NV>(p, tb, spre, lane, wpre, mpre);
      }
    }
    int u0 = 0;
    for (;;) {
      const int e = ebits ? __ffs(ebits) - 1 : nval - 1;
#pragma unroll 4
      for (int u = u0; u <= e; ++u) {
        const float* r = rows + (size_t)u * tb.dim;
#pragma unroll
        for (int w = 0; w < NV; ++w) {
          const int cv = lane + w * GL;
          if (cv < nvec) acc[w] = f4add(acc[w], *reinterpret_cast<const float4*>(r + cv * 4));
        }
      }
      if (!ebits) break;
      const int s = ks[e];
      if (s == prev_seg) {
        store_carry<GL, NV>(p, chunk, 0, nvec, lane, acc);
        if (lane == 0) p.completers[atomicAdd(p.n_completers, 1)] = make_int2(chunk, t);
      } else if constexpr (FWD) {
        store_pooled<GL, NV>(p, tb, s, acc, lane, loss_acc);
      } else {
        if (s == spre) {
          adagrad_row<GL, NV>(p, tb, 0xffffffffu, s, acc, lane, wpre, mpre);
        } else {
          float4 wr[NV];
          float mr;
          load_row_state<GL, NV>(p, tb, s, lane, wr, mr);
          adagrad_row<GL, NV>(p, tb, 0xffffffffu, s, acc, lane, wr, mr);
        }
      }
#pragma unroll
      for (int w = 0; w < NV; ++w) acc[w] = make_float4(0.f, 0.f, 0.f, 0.f);
      ebits &= ebits - 1;
      u0 = e + 1;
      if (u0 >= nval) break;
    }
    // slot consumed: hand it to the async proxy again
    fence_proxy_async_smem();
    __syncwarp();
    if (k + NS < nb) issue(k + NS);
    load_ids(k + NS + 1);
  }
  // The chunk's last segment continues into the next chunk: hand the partial on.
  if (j_hi < t_hi) {
    const int sl = __ldg(p.seg + j_hi - 1);
    if (__ldg(p.seg + j_hi) == sl) store_carry<GL, NV>(p, chunk, sl == prev_seg ? 0 : 1, nvec, lane, acc);
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

// Units [unit_begin, unit_begin + n) of GL = 32 tables (ordered first by the host).
template <bool FWD>
__global__ void __launch_bounds__(kTmaWarps * 32, 1) seg_reduce_tma_kernel(SegParams p, int n) {
  extern __shared__ __align__(128) char tma_smem[];
  const int warp = threadIdx.x >> 5;
  const int unit = blockIdx.x * kTmaWarps + warp;
  if (unit >= n) return;
  const int t = __ldg(p.unit_table + unit);
  const DevTable tb = p.tabs[t];
  char* wsm = tma_smem + warp * kTmaWarpBytes;
  switch (tb.kind) {
    case 5: seg_unit_tma<FWD, 1>(p, tb, t, unit, wsm); break;
    case 6: seg_unit_tma<FWD, 2>(p, tb, t, unit, wsm); break;
    case 7: seg_unit_tma<FWD, 4>(p, tb, t, unit, wsm); break;
    default: seg_unit_tma<FWD, 8>(p, tb, t, unit, wsm); break;
  }
}

}  // namespace asb
