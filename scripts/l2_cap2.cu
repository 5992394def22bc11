// Microbenchmark (experiment, not product code): L2 -> SMEM ingress for random 512-byte rows,
// comparing issue mechanisms beyond scripts/l2_cap.cu:
//   cpasync W : W warps, one 16-byte cp.async.cg per lane (the SpMM's gather), 8-row commit groups
//   bulk    W : W warps, every lane issues its own 1-D cp.async.bulk of one 512-byte row
//               (32 rows per warp instruction), completion on a per-warp mbarrier ring
//   mix     W : half the warps cp.async, half bulk
// One CTA per SM; contents are never read (bandwidth only).  Region 4 MB (L2 resident).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/l2_cap2 scripts/l2_cap2.cu
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}

// mode 0 = cp.async, 1 = bulk, 2 = mix (even warps cp.async, odd warps bulk)
template <int MODE, int DEPTH>
__global__ void gather(const uint4* __restrict__ src, const int* __restrict__ idx, int rows_per_warp,
                       int seg_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int* my = idx + ((size_t)blockIdx.x * nw + warp) * rows_per_warp;
  // per warp: 4 KB of "ring" for cp.async (rows overwrite each other) / DEPTH slots x 32 rows for bulk
  __shared__ __align__(8) uint64_t bars[32][DEPTH];
  const bool bulk = MODE == 1 || (MODE == 2 && (warp & 1));
  if (bulk && lane == 0)
    for (int d = 0; d < DEPTH; ++d)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][d])));
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const char* s8 = reinterpret_cast<const char*>(src);
  if (!bulk) {
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
          asm volatile("cp.async.wait_group 4;" ::: "memory");
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    // each lane copies one segment per round; DEPTH rounds in flight per warp
    const uint32_t dst = smem_u32(sm) + (warp % 16) * 8192 + (lane % 16) * 512;
    uint32_t phase = 0;
    int slot = 0;
    for (int r0 = 0; r0 < rows_per_warp; r0 += 32) {
      const uint32_t bar = smem_u32(&bars[warp][slot]);
      if (r0 >= 32 * DEPTH) mbar_wait(bar, phase ^ 1);   // previous use of this slot completed
      const int row = __ldg(my + r0 + lane);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(32 * seg_bytes)
                     : "memory");
      __syncwarp();
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(s8 + (size_t)row * 512), "r"(seg_bytes), "r"(bar)
                   : "memory");
      if (++slot == DEPTH) { slot = 0; phase ^= 1; }
    }
    // drain
    for (int d = 0; d < DEPTH; ++d) {
      const int r0 = rows_per_warp - 32 * DEPTH + 32 * d;
      if (r0 < 0) continue;
      const int s = (r0 / 32) % DEPTH;
      const uint32_t ph = ((r0 / 32) / DEPTH) & 1;
      mbar_wait(smem_u32(&bars[warp][s]), ph);
    }
  }
}

template <int MODE, int DEPTH>
void run(const uint4* src, int* d_idx, int region_rows, int warps, int sms, int seg_bytes, const char* name) {
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
  cudaFuncSetAttribute(gather<MODE, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<MODE, DEPTH><<<sms, 32 * warps, 131072>>>(src, d_idx, rows_per_warp, seg_bytes);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather<MODE, DEPTH><<<sms, 32 * warps, 131072>>>(src, d_idx, rows_per_warp, seg_bytes);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  // bytes: cp.async rows are 512 B; bulk rows seg_bytes
  double bytes = 0;
  for (int w = 0; w < warps; ++w) {
    const bool bulk = MODE == 1 || (MODE == 2 && (w & 1));
    bytes += (double)sms * rows_per_warp * (bulk ? seg_bytes : 512);
  }
  printf("%-8s warps %2d depth %2d seg %4d B  %7.3f ms  %6.2f TB/s  %5.1f B/clk/SM\n", name, warps, DEPTH, seg_bytes, ms,
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
  cudaMalloc(&d_idx, (size_t)sms * 32 * 4096 * 4);
  const int region = 8192;  // 4 MB
  for (int w : {8, 16, 24, 32}) run<0, 4>(src, d_idx, region, w, sms, 512, "cpasync");
  for (int w : {1, 2, 4, 8, 16}) run<1, 2>(src, d_idx, region, w, sms, 512, "bulk");
  for (int w : {1, 2, 4, 8, 16}) run<1, 4>(src, d_idx, region, w, sms, 512, "bulk");
  for (int w : {4, 8}) run<1, 4>(src, d_idx, region, w, sms, 256, "bulk");
  for (int w : {16, 24, 32}) run<2, 4>(src, d_idx, region, w, sms, 512, "mix");
  run<0, 4>(src, d_idx, 262144, 16, sms, 512, "cp128MB");
  run<1, 4>(src, d_idx, 262144, 8, sms, 512, "bk128MB");
  return 0;
}
