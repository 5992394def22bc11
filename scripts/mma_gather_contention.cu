// Microbenchmark (experiment, not product code): do the SpMM's cp.async gather writes into
// shared memory and the tcgen05.mma operand reads compete for the same SMEM bandwidth?
//
// One CTA per SM.  Warp 0 issues back-to-back tcgen05.mma (sparse M=64 N=256 K=32, the V=64
// SpMM instruction; or dense M=128 N=256 K=16) on static smem operands for ITERS instructions;
// G gather warps meanwhile stream random 512-byte rows (16-byte cp.async.cg per lane) out of an
// L2-resident 4 MB region into a disjoint 128 KB smem ring until warp 0 is done.  Reported per
// configuration: MMA cycles per instruction and the gather's delivered bytes per SM clock.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/mma_gather_contention scripts/mma_gather_contention.cu
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

constexpr int SB = 65536, SA = 16384, SG = 131072;

// SPARSE: 1 = sparse M=64 N=256 K=32, 0 = dense M=128 N=256 K=16; do_mma = 0: gather alone
template <int SPARSE>
__global__ void bench(const uint4* __restrict__ src, const int* __restrict__ idx, int iters, int do_mma,
                      unsigned long long* out, int gap_cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  __shared__ unsigned long long rows_done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sB = sm;
  uint8_t* sA = sm + SB;
  const uint32_t sG = smem_u32(sm + SB + SA);
  for (int i = threadIdx.x; i < (SB + SA) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    stop = 0;
    rows_done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (warp < 4) {
    const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanebase + 504 + c), "r"(0x44444444u));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const long long t0 = clock64();
  if (warp == 0) {
    const int M = SPARSE ? 64 : 128, N = 256;
    const uint32_t idesc = (SPARSE ? (1u << 2) : 0u) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sA), 128, 256, 0);
    const uint64_t bd = desc(smem_u32(sB), 16384, 1024, 2);
    const uint32_t te = tmem + 504;
    if (do_mma) {
      for (int i = 0; i < iters; i += 8) {
        if (elect_one()) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (SPARSE)
              asm volatile("tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%4], %3, 1;\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(te));
            else
              asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc));
          }
        }
        __syncwarp();
        // duty < 100 %: after each batch of 8 MMAs, hold the issue for gap_cycles
        if (gap_cycles) {
          const long long tg = clock64();
          while (clock64() - tg < gap_cycles) {}
        }
      }
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      __syncwarp();
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar)));
    } else {
      // gather alone: a fixed wall of cycles
      while (clock64() - t0 < (long long)iters * 144) {}
    }
    const long long t1 = clock64();
    if (lane == 0) {
      stop = 1;
      out[blockIdx.x * 2 + 0] = (unsigned long long)(t1 - t0);
    }
  } else if (warp >= 4) {
    const int gw = warp - 4, ngw = (blockDim.x >> 5) - 4;
    const int* my = idx + ((size_t)blockIdx.x * ngw + gw) * 65536;
    const uint32_t ring = sG + (gw % 16) * 8192 + lane * 16;
    unsigned long long rows = 0;
    int k = 0, r0 = 0;
    while (!stop) {
      const int mine = __ldg(my + (r0 & 65535) + lane);
      r0 += 32;
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
      rows += 32;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == 0) atomicAdd(&rows_done, rows);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x * 2 + 1] = rows_done;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int SPARSE>
void run(const uint4* src, const int* idx, int gwarps, int do_mma, int sms, unsigned long long* d,
         int gap = 0) {
  const int iters = 16384;
  const int smem = SB + SA + SG;
  cudaFuncSetAttribute(bench<SPARSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bench<SPARSE><<<sms, 32 * (4 + gwarps), smem>>>(src, idx, 64, do_mma, d, gap);
  bench<SPARSE><<<sms, 32 * (4 + gwarps), smem>>>(src, idx, gap ? iters / 2 : iters, do_mma, d, gap);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[512];
  cudaMemcpy(h, d, sms * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, rows = 0;
  for (int i = 0; i < sms; ++i) {
    cyc += h[2 * i];
    rows += h[2 * i + 1];
  }
  cyc /= sms;
  rows /= sms;
  const int n_mma = gap ? iters / 2 : iters;
  printf("%-14s gather_warps %2d  mma %s gap %5d  cycles/mma %7.1f  gather %6.1f B/clk/SM (%5.2f TB/s at 1.965 GHz)\n",
         SPARSE ? "sparse_m64" : "dense_m128", gwarps, do_mma ? "on " : "off", gap, do_mma ? cyc / n_mma : 0.0,
         rows * 512 / cyc, rows * 512 / cyc * sms * 1.965e9 / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int region_rows = 8192;  // 4 MB
  uint4* src;
  cudaMalloc(&src, (size_t)region_rows * 512);
  cudaMemset(src, 1, (size_t)region_rows * 512);
  const size_t nidx = (size_t)sms * 28 * 65536;
  int* h = (int*)malloc(nidx * 4);
  uint32_t s = 777u;
  for (size_t i = 0; i < nidx; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = (s >> 8) % region_rows;
  }
  int* idx;
  cudaMalloc(&idx, nidx * 4);
  cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
  unsigned long long* d;
  cudaMalloc(&d, sms * 16);
  for (int g : {0, 8, 16, 24}) run<1>(src, idx, g, 1, sms, d);
  for (int g : {8, 16, 24}) run<1>(src, idx, g, 0, sms, d);
  for (int g : {0, 8, 16}) run<0>(src, idx, g, 1, sms, d);
  // ~50 % MMA duty (the SpMM's tensor pipe is busy about half the time): 8 MMAs, then 2304 idle
  for (int g : {8, 16, 24, 28}) run<1>(src, idx, g, 1, sms, d, 2304);
  return 0;
}
