// Microbenchmark (experiment, not product code): the L2 -> SMEM ingress cap for the SpMM's
// gather pattern.  One CTA per SM, W warps; every warp streams random 512-byte rows (one
// 16-byte cp.async.cg per lane) out of an L2-resident region of R rows into a 128 KB smem ring
// (contents are never read: bandwidth only), keeping G commit groups of 8 rows in flight.
// Prints delivered TB/s and B/clk/SM for a sweep of (region, warps, depth).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/l2_cap scripts/l2_cap.cu
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int G>
__global__ void gather(const uint4* __restrict__ src, const int* __restrict__ idx, int rows_per_warp) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int* my = idx + ((size_t)blockIdx.x * nw + warp) * rows_per_warp;
  const uint32_t ring = smem_u32(sm) + (warp % 16) * 8192 + lane * 16;
  int k = 0;
  for (int r0 = 0; r0 < rows_per_warp; r0 += 32) {
    const int mine = __ldg(my + r0 + lane);
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const int row = __shfl_sync(0xffffffffu, mine, j);
      asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(ring + (j & 15) * 512),
                   "l"(src + (size_t)row * 32 + lane)
                   : "memory");
      if (++k == 8) {
        k = 0;
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(G) : "memory");
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

template <int G>
void run(const uint4* src, int* d_idx, int region_rows, int warps, int sms) {
  const int rows_per_warp = 4096;
  const size_t n = (size_t)sms * warps * rows_per_warp;
  int* h = (int*)malloc(n * 4);
  uint32_t s = 12345u + region_rows;
  for (size_t i = 0; i < n; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = (s >> 8) % region_rows;
  }
  cudaMemcpy(d_idx, h, n * 4, cudaMemcpyHostToDevice);
  free(h);
  cudaFuncSetAttribute(gather<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<G><<<sms, 32 * warps, 131072>>>(src, d_idx, rows_per_warp);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather<G><<<sms, 32 * warps, 131072>>>(src, d_idx, rows_per_warp);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = (double)n * 512;
  printf("region %6.1f MB  warps %2d  depth %2d groups (%3d KB/SM in flight)  %7.3f ms  %6.2f TB/s  %5.1f B/clk/SM\n",
         region_rows * 512.0 / 1048576, warps, G, warps * (G + 1) * 8 * 512 / 1024, ms,
         bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1.965e9 / sms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int max_rows = 262144;  // 128 MB
  uint4* src;
  cudaMalloc(&src, (size_t)max_rows * 512);
  cudaMemset(src, 1, (size_t)max_rows * 512);
  int* d_idx;
  cudaMalloc(&d_idx, (size_t)sms * 16 * 4096 * 4);
  const int regions[] = {4096, 8192, 16384, 65536, 262144};  // 2, 4, 8, 32, 128 MB
  for (int r : regions) run<4>(src, d_idx, r, 8, sms);
  for (int w : {4, 8, 12, 16}) {
    run<1>(src, d_idx, 8192, w, sms);
    run<2>(src, d_idx, 8192, w, sms);
    run<4>(src, d_idx, 8192, w, sms);
    run<6>(src, d_idx, 8192, w, sms);
  }
  return 0;
}
