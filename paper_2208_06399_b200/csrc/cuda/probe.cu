// Live roofline denominators for bench.py: the B200's random-row gather
// bandwidth over a given footprint (an L2-resident footprint gives the L2
// gather ceiling of the cache-resident embedding kernels; a multi-GB one the
// HBM gather ceiling). Same access shape as the seg_reduce kernels: each
// group of row_bytes/16 lanes loads one random row, 8 rows in flight per lane.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../host/host.hpp"
#include "context.hpp"

namespace asb {
namespace {

template <int GL>
__global__ void __launch_bounds__(256) probe_gather_kernel(const float4* __restrict__ src, unsigned rows,
                                                           unsigned iters, unsigned seed, float4* sink) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned g = lane / GL, c = lane % GL;
  unsigned x = seed ^ ((blockIdx.x * 256 + threadIdx.x - c) * 2654435761u);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (unsigned it = 0; it < iters; ++it) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const unsigned r = (x >> 6) % rows;
      v[u] = __ldg(src + (size_t)r * GL + c);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  (void)g;
  if (acc.x == 1234.5f) sink[0] = acc;
}

template <int GL>
double run_probe(const float4* buf, size_t footprint, float4* sink, int sms) {
  const unsigned rows = (unsigned)std::max<size_t>(1, footprint / (GL * 16));
  double best = 0.0;
  cudaEvent_t a, b;
  cuda_check(cudaEventCreate(&a), "event");
  cuda_check(cudaEventCreate(&b), "event");
  for (int ctas_per_sm : {4, 8}) {
    const unsigned blocks = (unsigned)(sms * ctas_per_sm), iters = 64;
    probe_gather_kernel<GL><<<blocks, 256>>>(buf, rows, 4, 1, sink);  // warm-up
    cuda_check(cudaEventRecord(a), "event");
    probe_gather_kernel<GL><<<blocks, 256>>>(buf, rows, iters, 7, sink);
    cuda_check(cudaEventRecord(b), "event");
    cuda_check(cudaEventSynchronize(b), "probe");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, a, b), "elapsed");
    const double bytes = (double)blocks * 256 * iters * 8 * 16;
    best = std::max(best, bytes / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

}  // namespace

double probe_gather_bw(int device, int64_t footprint, int row_bytes) {
  if (footprint < 4096) fail(AS_CONFIG, "as_probe_gather_bw: footprint must be >= 4096 bytes");
  int dev0 = 0;
  cuda_check(cudaGetDevice(&dev0), "cudaGetDevice");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  int sms = 148;
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "SM count");
  float4* buf = nullptr;
  float4* sink = nullptr;
  cuda_check(cudaMalloc(&buf, (size_t)footprint), "cudaMalloc");
  cuda_check(cudaMalloc(&sink, 64), "cudaMalloc");
  cuda_check(cudaMemset(buf, 0, (size_t)footprint), "memset");
  double gbs = 0.0;
  switch (row_bytes) {
    case 16: gbs = run_probe<1>(buf, footprint, sink, sms); break;
    case 32: gbs = run_probe<2>(buf, footprint, sink, sms); break;
    case 64: gbs = run_probe<4>(buf, footprint, sink, sms); break;
    case 128: gbs = run_probe<8>(buf, footprint, sink, sms); break;
    case 256: gbs = run_probe<16>(buf, footprint, sink, sms); break;
    case 512: gbs = run_probe<32>(buf, footprint, sink, sms); break;
    default:
      cudaFree(buf);
      cudaFree(sink);
      fail(AS_CONFIG, "as_probe_gather_bw: row_bytes must be 16..512 (power of two), got " + std::to_string(row_bytes));
  }
  cudaFree(buf);
  cudaFree(sink);
  cudaSetDevice(dev0);
  return gbs;
}

}  // namespace asb
