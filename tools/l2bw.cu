// Microbenchmark: B200 bandwidth of 16-byte loads that hit L2 (and, for the
// small footprint, L1), and of HBM, with random 512-B row gathers like the
// embedding kernels. Prints GB/s. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2bw.cu -o tools/l2bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gather_rows(const float4* __restrict__ src, unsigned rows, unsigned iters, unsigned seed,
                            float4* sink) {
  // each warp gathers random 512-B rows (32 lanes x 16 B), 8 in flight
  const unsigned lane = threadIdx.x & 31;
  unsigned x = seed ^ (blockIdx.x * 1024 + (threadIdx.x >> 5)) * 2654435761u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (unsigned it = 0; it < iters; ++it) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const unsigned r = (x >> 8) % rows;
      v[u] = __ldg(src + (size_t)r * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc.x += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc.x == 1234.5f) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = 8ull << 30;  // 8 GB: HBM
  float4* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  float4* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t foot[] = {1ull << 20, 16ull << 20, 64ull << 20, 96ull << 20, 256ull << 20, big};
  for (size_t f : foot) {
    const unsigned rows = (unsigned)(f / 512);
    for (int occ : {8, 16, 32}) {
      const unsigned blocks = sms * occ / 8, iters = 256;
      gather_rows<<<blocks, 256>>>(buf, rows, 4, 1, sink);
      cudaEventRecord(a);
      gather_rows<<<blocks, 256>>>(buf, rows, iters, 7, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)blocks * 8 * iters * 8 * 512;
      printf("footprint %8.1f MB  warps/SM %2d  %8.1f GB/s\n", f / 1048576.0, occ, bytes / ms / 1e6);
    }
  }
  return 0;
}
