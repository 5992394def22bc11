// Microbenchmark (experiment, not product code): back-to-back tcgen05.mma throughput on B200 for
// the shapes the HiNM SpMM can use.  One CTA per SM; thread 0 issues ITERS MMAs on static smem
// operands, commits once, and the kernel time gives cycles per MMA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o mma_bench scripts/mma_bench.cu
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

// sparse: 0 dense kind::f16 (K=16), 1 sparse (K=32), 2 sparse with A in TMEM
__global__ void bench(int M, int N, int sparse, int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  uint8_t* sB = sm;             // 64 KB: K=32 rows x 256 tokens, SW128 MN-major
  uint8_t* sA = sm + 65536;     // 8 KB: 128 rows x 32 B (K-major, no swizzle)
  for (int i = threadIdx.x; i < (65536 + 8192) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
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
  // metadata 0x44444444 in columns 384..391, A-in-TMEM in columns 256..383 (all lanes)
  {
    const uint32_t lanebase = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < 8; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanebase + 384 + c), "r"(0x44444444u));
    for (int c = 0; c < 16; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lanebase + 256 + c), "r"(0x3c003c00u));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (sparse ? (1u << 2) : 0u) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sA), 128, 256, 0);
    const uint64_t bd = desc(smem_u32(sB), 16384, 1024, 2);
    const uint32_t te = tmem + 384;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (sparse == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(i));
      } else if (sparse == 1) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(ad), "l"(bd), "r"(idesc), "r"(i), "r"(te));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], [%1], %2, [%5], %3, p;\n\t}\n" ::"r"(tmem),
                     "r"(tmem + 256), "l"(bd), "r"(idesc), "r"(i), "r"(te));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)));
    const long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 8192);
  const int iters = 4096;
  printf("kind,M,N,K_logical,cycles_per_mma,ms,chip_TFLOPs_logical\n");
  for (int sparse = 0; sparse < 3; ++sparse)
    for (int M : {64, 128})
      for (int N : {64, 128, 256}) {
        if (sparse == 2 && M == 64) continue;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        bench<<<sms, 128, 65536 + 8192>>>(M, N, sparse, 64, d);  // warm
        cudaEventRecord(a);
        bench<<<sms, 128, 65536 + 8192>>>(M, N, sparse, iters, d);
        cudaEventRecord(b);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s (sparse=%d M=%d N=%d)\n", cudaGetErrorString(e), sparse, M, N); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[256];
        cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += h[i];
        avg /= sms;
        const int K = sparse ? 32 : 16;
        const double flops = 2.0 * M * N * K * (double)iters * sms;
        printf("%s,%d,%d,%d,%.1f,%.3f,%.1f\n", sparse == 0 ? "dense" : (sparse == 1 ? "sparse_ss" : "sparse_ts"),
               M, N, K, avg / iters, ms, flops / (ms * 1e-3) / 1e12);
      }
  return 0;
}
