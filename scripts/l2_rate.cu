// Microbenchmark (experiment, not product code): L2 -> SM ingress rate on B200 for the access
// patterns an activation gather can use.  148 CTAs x 256 threads; a 64 MB L2-resident source
// (n rows x 256 tokens bf16 = 512 B per row); each CTA streams `rows` random rows.
//   mode 0: cp.async.cg 16 B (L2 only) into a 32 KB smem ring
//   mode 1: cp.async.ca 16 B (L1 allocate)
//   mode 2: LDG.128 (ld.global.nc.L1::no_allocate) into registers, xor-accumulated
//   mode 3: cp.async.bulk 512 B rows (one bulk copy per row) into smem
//   mode 4: same as 0 but every CTA reads the SAME row sequence (max L1/L2 locality)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/l2_rate scripts/l2_rate.cu
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ src, const int* __restrict__ idx,
                                              int rows, int nrows, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* myidx = idx + (MODE == 4 ? 0 : (size_t)blockIdx.x * rows);
  uint4 acc = make_uint4(0, 0, 0, 0);
  if (MODE == 5) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t phase = 0;
      const size_t chunks = (size_t)nrows * 512 / 16384;
      for (int r0 = 0; r0 < rows * 512 / 16384; r0 += 2) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * 16384));
        for (int r = 0; r < 2; ++r) {
          const size_t c = ((size_t)blockIdx.x * 977 + r0 + r) % chunks;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                       ::"r"(smem_u32(sm + r * 16384)), "l"((const char*)src + c * 16384), "r"(smem_u32(&bar)) : "memory");
        }
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase));
        phase ^= 1;
      }
    }
    __syncthreads();
  } else if (MODE == 3) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t phase = 0;
      for (int r0 = 0; r0 < rows; r0 += 64) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(64 * 512));
        for (int r = 0; r < 64; ++r) {
          const uint4* s = src + (size_t)myidx[r0 + r] * 32;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];"
                       ::"r"(smem_u32(sm + r * 512)), "l"(s), "r"(smem_u32(&bar)) : "memory");
        }
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase));
        phase ^= 1;
      }
    }
    __syncthreads();
  } else {
    // warp w handles rows w, w+8, ...; lane = 16 B chunk of the 512 B row
    int k = 0;
    int ibuf = 0;
    for (int r = warp; r < rows; r += 8) {
      if (((r - warp) >> 3) % 32 == 0) ibuf = __ldg(myidx + r + 8 * lane);  // 32 rows of indices per warp
      const int row = __shfl_sync(0xffffffffu, ibuf, ((r - warp) >> 3) % 32);
      const uint4* s = src + (size_t)row * 32 + lane;
      const uint32_t d = smem_u32(sm + ((r & 63) * 512) + lane * 16);
      if (MODE == 0 || MODE == 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
      else if (MODE == 1)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
      else {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s));
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
      }
      if (MODE != 2 && ++k == 8) {
        asm volatile("cp.async.commit_group;");
        asm volatile("cp.async.wait_group 6;");
        k = 0;
      }
    }
    if (MODE != 2) asm volatile("cp.async.wait_all;");
  }
  if (acc.x == 0x12345678u) out[blockIdx.x] = acc.y;  // keep loads alive
}

template <int MODE>
void run(const char* name, const uint4* src, const int* idx, int rows, int nrows, int sms, unsigned long long* d) {
  cudaFuncSetAttribute(gather<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 512);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<MODE><<<sms, 256, 64 * 512>>>(src, idx, rows, nrows, d);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) gather<MODE><<<sms, 256, 64 * 512>>>(src, idx, rows, nrows, d);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = (double)sms * rows * 512;
  printf("%-28s %8.3f ms  %8.2f TB/s  %6.1f B/clk/SM @1.965GHz\n", name, ms, bytes / (ms * 1e-3) / 1e12,
         bytes / (ms * 1e-3) / 1.965e9 / sms);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int nrows = 131072;  // 64 MB of 512 B rows
  const int rows = 16384;    // per CTA: 8 MB
  uint4* src;
  int* idx;
  cudaMalloc(&src, (size_t)nrows * 512);
  cudaMemset(src, 1, (size_t)nrows * 512);
  int* h = (int*)malloc((size_t)sms * rows * 4);
  uint32_t s = 12345;
  for (size_t i = 0; i < (size_t)sms * rows; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = (s >> 8) % nrows;
  }
  cudaMalloc(&idx, (size_t)sms * rows * 4);
  cudaMemcpy(idx, h, (size_t)sms * rows * 4, cudaMemcpyHostToDevice);
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  run<0>("cp.async.cg 16B", src, idx, rows, nrows, sms, d);
  run<1>("cp.async.ca 16B", src, idx, rows, nrows, sms, d);
  run<2>("ldg.nc no_allocate 16B", src, idx, rows, nrows, sms, d);
  run<3>("cp.async.bulk 512B rows", src, idx, rows, nrows, sms, d);
  run<4>("cp.async.cg same rows/CTA", src, idx, rows, nrows, sms, d);
  run<5>("bulk 2x16KB contiguous", src, idx, rows, nrows, sms, d);
  return 0;
}
