// Microbenchmark (experiment, not product code): sustained tcgen05.mma rate per SM on B200 for
// the operand shapes a HiNM SpMM can use.  Warp-uniform issue loop (descriptors in uniform
// registers), elected lane issues, unrolled x8, one commit at the end.  Static smem operands.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/mma_rate scripts/mma_rate.cu
#include <stdint.h>
#include <stdio.h>

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

// kind: 0 dense SS, 1 sparse SS, 2 sparse TS (A in TMEM), 3 dense TS (A in TMEM)
template <int KIND>
__global__ void bench(int M, int N, int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  uint8_t* sB = sm;             // 64 KB
  uint8_t* sA = sm + 65536;     // 16 KB
  for (int i = threadIdx.x; i < (65536 + 16384) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
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
  {
    const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanebase + 504 + c), "r"(0x44444444u));
    for (int c = 0; c < 16; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanebase + 256 + c), "r"(0x3c003c00u));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const bool sparse = KIND == 1 || KIND == 2;
    const uint32_t idesc = (sparse ? (1u << 2) : 0u) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sA), 128, 256, 0);
    const uint64_t bd = desc(smem_u32(sB), 16384, 1024, 2);
    const uint32_t te = tmem + 504;
    const uint32_t ta = tmem + 256;
    const long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (KIND == 0)
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc));
          else if (KIND == 1)
            asm volatile("tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%4], %3, 1;\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(te));
          else if (KIND == 2)
            asm volatile("tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%4], %3, 1;\n" ::"r"(tmem), "r"(ta), "l"(bd), "r"(idesc), "r"(te));
          else
            asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n" ::"r"(tmem), "r"(ta), "l"(bd), "r"(idesc));
        }
      }
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    const long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND>
void run(int M, int N, int sms, unsigned long long* d) {
  const int iters = 8192;
  cudaFuncSetAttribute(bench<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 16384);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bench<KIND><<<sms, 128, 65536 + 16384>>>(M, N, 64, d);
  cudaEventRecord(a);
  bench<KIND><<<sms, 128, 65536 + 16384>>>(M, N, iters, d);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const int K = (KIND == 1 || KIND == 2) ? 32 : 16;
  const double flops = 2.0 * M * N * K * (double)iters * sms;
  const char* names[] = {"dense_ss", "sparse_ss", "sparse_ts", "dense_ts"};
  printf("%s,%d,%d,%d,%.1f,%.3f,%.1f\n", names[KIND], M, N, K, avg / iters, ms, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  printf("kind,M,N,K_logical,cycles_per_mma,ms,chip_TFLOPs_logical\n");
  int Ns[] = {64, 128, 256};
  for (int N : Ns) run<0>(128, N, sms, d);
  for (int N : Ns) run<0>(64, N, sms, d);
  for (int N : Ns) run<1>(128, N, sms, d);
  for (int N : Ns) run<1>(64, N, sms, d);
  for (int N : Ns) run<2>(128, N, sms, d);
  for (int N : Ns) run<3>(128, N, sms, d);
  return 0;
}
