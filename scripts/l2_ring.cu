// Microbenchmark (experiment, not product code): the SpMM gather pipeline in isolation.
// One CTA per SM.  GW producer warps fill a ring of S stages of R random 512-byte rows each
// (16-byte cp.async.cg per lane, completion signalled with cp.async.mbarrier.arrive.noinc on the
// stage's full barrier, exactly as k_hinm_spmm does); one consumer warp waits full -> arrives
// empty.  Optionally a second warp adds a bulk copy of ABYTES per stage into the same full
// barrier (the compressed-A / metadata stream).  Prints delivered TB/s for a sweep.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/l2_ring scripts/l2_ring.cu
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

struct Cfg { int GW, R, S, abytes, stages; int stride16; };  // row pitch in 16-byte units

__global__ void ring(const uint4* __restrict__ src, const int* __restrict__ idx, const uint8_t* __restrict__ asrc,
                     Cfg c) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[32]);
  const uint32_t sB = smem_u32(sm), sA = sB + c.S * c.R * 512;
  if (threadIdx.x == 0) {
    for (int s = 0; s < c.S; ++s) {
      mbar_init(full0 + 8 * s, 32 * c.GW + 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int* my = idx + (size_t)blockIdx.x * c.stages * c.R;
  if (warp < c.GW) {
    const int gw = warp, rpw = c.R / c.GW;
    int stage = 0;
    uint32_t phase = 0;
    // gather indices prefetched PF stages ahead (as in k_hinm_spmm)
    constexpr int PF = 8;
    int pre[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) pre[j] = lane < rpw && j < c.stages ? __ldg(my + (size_t)j * c.R + gw + lane * c.GW) : 0;
    for (int i0 = 0; i0 < c.stages; i0 += PF) {
#pragma unroll
     for (int jj = 0; jj < PF; ++jj) {
      const int i = i0 + jj;
      if (i >= c.stages) break;
      const int myrow = pre[jj];
      pre[jj] = lane < rpw && i + PF < c.stages ? __ldg(my + (size_t)(i + PF) * c.R + gw + lane * c.GW) : 0;
      mbar_wait(empty0 + 8 * stage, phase ^ 1);
      const uint32_t dst = sB + stage * c.R * 512 + lane * 16;
      for (int j = 0; j < rpw; ++j) {
        const int row = __shfl_sync(0xffffffffu, myrow, j);
        asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst + (gw + j * c.GW) * 512),
                     "l"(src + (size_t)row * c.stride16 + lane) : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full0 + 8 * stage) : "memory");
      if (++stage == c.S) { stage = 0; phase ^= 1; }
     }
    }
  } else if (warp == c.GW) {
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < c.stages; ++i) {
      mbar_wait(empty0 + 8 * stage, phase ^ 1);
      if (lane == 0) {
        const uint32_t fb = full0 + 8 * stage;
        if (c.abytes) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(c.abytes) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(sA + stage * c.abytes), "l"(asrc + ((size_t)blockIdx.x * 977 + i) % 4096 * c.abytes),
                       "r"(c.abytes), "r"(fb) : "memory");
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fb) : "memory");
        }
      }
      __syncwarp();
      if (++stage == c.S) { stage = 0; phase ^= 1; }
    }
  } else if (warp == c.GW + 1) {
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < c.stages; ++i) {
      mbar_wait(full0 + 8 * stage, phase);
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * stage) : "memory");
      __syncwarp();
      if (++stage == c.S) { stage = 0; phase ^= 1; }
    }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int region = 8192;  // rows of 512 B (an LLaMA down-projection token block is 11008 rows)
  uint4* src;
  cudaMalloc(&src, (size_t)region * 32768);
  cudaMemset(src, 1, (size_t)region * 32768);
  uint8_t* asrc;
  cudaMalloc(&asrc, 4096 * 8192);
  const size_t total_rows = (size_t)sms * 2048 * 64;
  int* h = (int*)malloc(total_rows * 4);
  uint32_t s = 777;
  for (size_t i = 0; i < total_rows; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % region; }
  int* idx;
  cudaMalloc(&idx, total_rows * 4);
  cudaMemcpy(idx, h, total_rows * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  // region rows of 512 B: pitch 512 B (contiguous 4 MB) or 32 KB (a 16384-token channel-major X:
  // the same 8192 rows spread over 256 MB, i.e. the SpMM's real source pattern)
  Cfg cfgs[] = {
      {16, 64, 5, 0, 0, 32},   {16, 64, 5, 0, 0, 2048},  {16, 64, 5, 0, 0, 256},  {16, 64, 5, 0, 0, 1024},
      {16, 128, 3, 0, 0, 32},  {16, 128, 3, 0, 0, 2048}, {8, 64, 5, 0, 0, 2048},
  };
  for (Cfg c : cfgs) {
    c.stages = (int)(total_rows / sms / c.R);
    const int smem = c.S * c.R * 512 + c.S * c.abytes;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    ring<<<sms, 32 * (c.GW + 2), smem>>>(src, idx, asrc, c);
    cudaEventRecord(a);
    ring<<<sms, 32 * (c.GW + 2), smem>>>(src, idx, asrc, c);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)sms * c.stages * (c.R * 512.0 + c.abytes);
    printf("GW %2d  rows/stage %3d  stages %2d  A %5d B/stage  pitch %6d B  smem %3d KB  %7.3f ms  %6.2f TB/s  %5.1f B/clk/SM\n",
           c.GW, c.R, c.S, c.abytes, c.stride16 * 16, smem / 1024, ms, bytes / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1.965e9 / sms);
  }
  return 0;
}
