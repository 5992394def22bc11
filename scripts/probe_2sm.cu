// Hardware probe + microbenchmark (experiment, not product code): the CTA-pair sparse MMA
// (tcgen05.mma.sp.cta_group::2.kind::f16, M = 256, N = 256) that a union-group HiNM SpMM would use.
//
// Part 1 (probe): operand split and metadata placement.  Each CTA of a 2-CTA cluster holds
// 128 rows of A (2:4 compressed, the product's K-major SWIZZLE_NONE image) and 128 of the 256
// tokens of B (the product's SWIZZLE_128B MN-major gathered-row stage); the leader copies both
// CTAs' metadata into their TMEM with one tcgen05.cp.cta_group::2 and issues four MMAs (128
// logical K, the product's id2 / E-column stepping).  Each CTA reads its 128 x 256 accumulator
// back; the host compares with D = A_dense @ B_full (small integers: exact in fp32).
//
// Part 2 (rate): back-to-back MMAs on static operands while G warps per CTA stream 512-byte rows
// into shared memory with cp.async (the SpMM's gather), for
//   2sm_m256  tcgen05.mma.sp.cta_group::2 M=256 N=256 K=32  (per SM: 128 rows, half of B)
//   1sm_m128  tcgen05.mma.sp.cta_group::1 M=128 N=256 K=32
//   1sm_m64   tcgen05.mma.sp.cta_group::1 M=64  N=256 K=32  (today's V = 64 instruction)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/probe_2sm scripts/probe_2sm.cu
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

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

__host__ __device__ constexpr uint32_t idesc_sp(int M, int N) {
  return (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

constexpr int A_BYTES = 128 * 64 * 2;     // 128 rows x 64 compressed (128 logical K)
constexpr int B_BYTES = 2 * 128 * 128;    // 2 chunks of 64 tokens x 128 K-rows x 128 B
constexpr int E_BYTES = 128 * 16;         // 128 lanes x 4 words
constexpr int E_COL = 256;

// ------------------------------------------------------------------------------ part 1
constexpr int A_COL = 320;  // TMEM columns of the A copies (TS variant): 4 MMA steps x 8 columns
template <bool ATMEM>
__global__ void __cluster_dims__(2, 1, 1) probe(const uint8_t* __restrict__ a_img, const uint8_t* __restrict__ b_img,
                                                const uint8_t* __restrict__ e_img, float* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  uint8_t* g = smem + (base - smem_u32(smem));
  const uint32_t r = cta_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < A_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(g)[i] = reinterpret_cast<const uint4*>(a_img + r * A_BYTES)[i];
  for (int i = tid; i < B_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(g + A_BYTES)[i] = reinterpret_cast<const uint4*>(b_img + r * B_BYTES)[i];
  for (int i = tid; i < E_BYTES / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(g + A_BYTES + B_BYTES)[i] = reinterpret_cast<const uint4*>(e_img + r * E_BYTES)[i];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (r == 0 && warp == 0) {
    if (elect_one()) {
      const uint64_t ed = desc(base + A_BYTES + B_BYTES, 0, 128, 0);
      asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(tmem + E_COL), "l"(ed) : "memory");
      const uint64_t ad0 = desc(base, 128, 256, 0);
      const uint64_t bd0 = desc(base + A_BYTES, B_BYTES / 2, 1024, 2);
      const uint32_t idesc = idesc_sp(256, 256);
      for (int i = 0; i < 4; ++i) {
        const uint64_t ad = ad0 + (uint64_t)((i * 32 * 128) >> 4);
        const uint64_t bd = bd0 + (uint64_t)((i * 4096) >> 4);
        const uint32_t ecol = tmem + E_COL + (i >> 1) * 2;
        if (ATMEM) {  // A of this step: smem image -> TMEM (128 lanes x 256 bits), then the TS MMA
          asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(tmem + A_COL + 8 * i), "l"(ad) : "memory");
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%5], %3, p;\n\t}\n" ::"r"(tmem),
              "r"(tmem + A_COL + 8 * i), "l"(bd), "r"(idesc | (uint32_t)(i & 1)), "r"(i), "r"(ecol)
              : "memory");
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc | (uint32_t)(i & 1)), "r"(i), "r"(ecol)
              : "memory");
        }
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    }
    __syncwarp();
  }
  wait_bar(smem_u32(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < 256; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v)
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[((size_t)r * 128 + warp * 32 + lane) * 256 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------------------------------ part 2
constexpr int RING = 131072;
// KIND 0 = 2sm M=256, 1 = 1sm M=128, 2 = 1sm M=64
template <int KIND>
__global__ void __launch_bounds__(32 * 32, 1) rate(const uint4* __restrict__ src, const int* __restrict__ idx,
                                                  int iters, int do_mma, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  __shared__ unsigned long long rows_done;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  uint8_t* g = smem + (base - smem_u32(smem));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t r = KIND == 0 ? cta_rank() : 0;
  for (int i = tid; i < (A_BYTES + B_BYTES) / 4; i += blockDim.x) ((uint32_t*)g)[i] = 0x3c003c00u;
  for (int i = tid; i < E_BYTES / 4; i += blockDim.x) ((uint32_t*)(g + A_BYTES + B_BYTES))[i] = 0x44444444u;
  if (tid == 0) {
    stop = 0;
    rows_done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (KIND == 0) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (KIND == 0) cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const long long t0 = clock64();
  if (warp == 0) {
    if (do_mma) {
      if (r == 0) {
        const uint64_t ed = desc(base + A_BYTES + B_BYTES, 0, 128, 0);
        const uint64_t ad = desc(base, 128, 256, 0);
        const uint64_t bd = desc(base + A_BYTES, B_BYTES / 2, 1024, 2);
        const uint32_t idesc = idesc_sp(KIND == 0 ? 256 : KIND == 1 ? 128 : 64, 256);
        if (elect_one()) {
          if (KIND == 0)
            asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(tmem + E_COL), "l"(ed) : "memory");
          else
            asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(tmem + E_COL), "l"(ed) : "memory");
        }
        __syncwarp();
        for (int i = 0; i < iters; i += 8) {
          if (elect_one()) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (KIND == 0)
                asm volatile("tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%4], %3, 1;\n" ::"r"(tmem), "l"(ad),
                             "l"(bd), "r"(idesc), "r"(tmem + E_COL));
              else
                asm volatile("tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%4], %3, 1;\n" ::"r"(tmem), "l"(ad),
                             "l"(bd), "r"(idesc), "r"(tmem + E_COL));
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          if (KIND == 0)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar)),
                "h"((uint16_t)3)
                : "memory");
          else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        }
        __syncwarp();
      }
      wait_bar(smem_u32(&bar), 0);
    } else {
      while (clock64() - t0 < (long long)iters * 160) {}
    }
    const long long t1 = clock64();
    if (lane == 0) {
      stop = 1;
      out[blockIdx.x * 2 + 0] = (unsigned long long)(t1 - t0);
    }
  } else if (warp >= 4) {
    const int gw = warp - 4, ngw = (blockDim.x >> 5) - 4;
    const int* my = idx + ((size_t)blockIdx.x * ngw + gw) * 65536;
    const uint32_t ring = base + A_BYTES + B_BYTES + E_BYTES + (gw % 16) * 8192 + lane * 16;
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
  if (tid == 0) out[blockIdx.x * 2 + 1] = rows_done;
  if (KIND == 0) cluster_sync_all();
  if (warp == 0) {
    if (KIND == 0)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int KIND>
void run_rate(const uint4* src, const int* idx, int gw, int do_mma, int sms, unsigned long long* d) {
  const int iters = 16384, smem = A_BYTES + B_BYTES + E_BYTES + RING + 1024;
  cudaFuncSetAttribute(rate<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(32 * (4 + gw));
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = KIND == 0 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, rate<KIND>, src, idx, rep ? iters : 64, do_mma, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("rate kind %d error %s\n", KIND, cudaGetErrorString(e));
      exit(1);
    }
  }
  std::vector<unsigned long long> h(2 * sms);
  cudaMemcpy(h.data(), d, sms * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, rows = 0;
  for (int i = 0; i < sms; ++i) {
    cyc += h[2 * i];
    rows += h[2 * i + 1];
  }
  cyc /= sms;
  rows /= sms;
  static const char* names[] = {"2sm_m256", "1sm_m128", "1sm_m64"};
  printf("%-9s gather_warps %2d mma %s  cycles/mma %7.1f  fill %6.1f B/clk/SM (%5.2f TB/s at 1.965 GHz)\n", names[KIND], gw,
         do_mma ? "on " : "off", do_mma ? cyc / iters : 0.0, rows * 512 / cyc, rows * 512 / cyc * sms * 1.965e9 / 1e12);
}

// ------------------------------------------------------------------------------ host packing (part 1)
static uint32_t lcg(uint32_t& s) {
  s = s * 1664525u + 1013904223u;
  return s >> 8;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // ---- part 1
  const int KL = 128, NT = 256;
  std::vector<float> Ad(2 * 128 * KL, 0.f), Bf((size_t)KL * NT);
  std::vector<uint16_t> aimg(2 * A_BYTES / 2, 0);
  std::vector<uint8_t> bimg(2 * B_BYTES, 0), eimg(2 * E_BYTES, 0);
  uint32_t s = 12345u;
  auto bf = [](float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16);
  };
  static const int pats[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  std::vector<uint8_t> nib(2 * 128 * (KL / 4));
  for (int r = 0; r < 2; ++r)
    for (int m = 0; m < 128; ++m)
      for (int c = 0; c < KL / 4; ++c) {
        const int pi = lcg(s) % 6;
        const int p0 = pats[pi][0], p1 = pats[pi][1];
        const float v0 = (float)((int)(lcg(s) % 7) - 3), v1 = (float)((int)(lcg(s) % 7) - 3);
        Ad[((size_t)r * 128 + m) * KL + 4 * c + p0] = v0;
        Ad[((size_t)r * 128 + m) * KL + 4 * c + p1] = v1;
        nib[((size_t)r * 128 + m) * (KL / 4) + c] = (uint8_t)(p0 | (p1 << 2));
        // compressed kc = 2c, 2c+1 -> aval_offset(0, V=128, m, kc)
        for (int q = 0; q < 2; ++q) {
          const int kc = 2 * c + q;
          const int b = kc >> 5, kcb = kc & 31, j = kcb >> 4, kcs = kcb & 15;
          const size_t off = (size_t)b * 32 * 128 + (size_t)j * 16 * 128 + (m >> 3) * 128 + (kcs >> 3) * 64 +
                             (m & 7) * 8 + (kcs & 7);
          aimg[(size_t)r * (A_BYTES / 2) + off] = bf(q ? v1 : v0);
        }
      }
  // metadata words (compress.cu k_pack_meta with V = 128, one 128-K block)
  for (int r = 0; r < 2; ++r)
    for (int lane = 0; lane < 128; ++lane)
      for (int w = 0; w < 4; ++w) {
        const int m0 = lane & 7, k1 = (lane >> 3) & 1, m2 = lane >> 4;
        uint32_t word = 0;
        for (int m1 = 0; m1 < 2; ++m1)
          for (int c = 0; c < 4; ++c) {
            const int row = m0 + 8 * m1 + 16 * m2, gch = 8 * w + 4 * k1 + c;
            word |= (uint32_t)nib[((size_t)r * 128 + row) * (KL / 4) + gch] << (16 * m1 + 4 * c);
          }
        memcpy(&eimg[(size_t)r * E_BYTES + lane * 16 + w * 4], &word, 4);
      }
  for (int k = 0; k < KL; ++k)
    for (int n = 0; n < NT; ++n) {
      const float v = (float)((int)(lcg(s) % 5) - 2);
      Bf[(size_t)k * NT + n] = v;
      const int r = n / 128, nn = n % 128, chunk = nn / 64, t = nn % 64;
      const size_t off = (size_t)chunk * (B_BYTES / 2) + (size_t)k * 128 + ((((t / 8) ^ (k & 7))) * 16) + (t % 8) * 2;
      const uint16_t h = bf(v);
      memcpy(&bimg[(size_t)r * B_BYTES + off], &h, 2);
    }
  uint8_t *da, *db, *de;
  float* dout;
  cudaMalloc(&da, 2 * A_BYTES);
  cudaMalloc(&db, 2 * B_BYTES);
  cudaMalloc(&de, 2 * E_BYTES);
  cudaMalloc(&dout, 2 * 128 * 256 * 4);
  cudaMemcpy(da, aimg.data(), 2 * A_BYTES, cudaMemcpyHostToDevice);
  cudaMemcpy(db, bimg.data(), 2 * B_BYTES, cudaMemcpyHostToDevice);
  cudaMemcpy(de, eimg.data(), 2 * E_BYTES, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 2 * 128 * 256 * 4);
  const int psmem = A_BYTES + B_BYTES + E_BYTES + 1024;
  for (int variant = 0; variant < 2; ++variant) {
  auto pk = variant ? probe<true> : probe<false>;
  cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, psmem);
  cudaMemset(dout, 0, 2 * 128 * 256 * 4);
  pk<<<2, 128, psmem>>>(da, db, de, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("probe error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> D(2 * 128 * 256);
  cudaMemcpy(D.data(), dout, D.size() * 4, cudaMemcpyDeviceToHost);
  // hypothesis H1: CTA r rows x all 256 tokens, tokens [128 r', 128 r'+128) from CTA r' smem
  long bad = 0, zero = 0;
  for (int r = 0; r < 2; ++r)
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double ref = 0;
        for (int k = 0; k < KL; ++k) ref += (double)Ad[((size_t)r * 128 + m) * KL + k] * Bf[(size_t)k * NT + n];
        const float got = D[((size_t)r * 128 + m) * 256 + n];
        if (got != (float)ref) {
          if (bad < 8) printf("mismatch cta %d row %d tok %d: got %g want %g\n", r, m, n, got, ref);
          ++bad;
        }
        zero += got == 0.f;
      }
  printf("probe 2sm M=256 N=256 sparse, A %s (B split by N, metadata via tcgen05.cp.cta_group::2): %ld / %d mismatches (%ld zeros)\n",
         variant ? "in TMEM (tcgen05.cp 128x256b of the smem image, TS MMA)" : "in smem (SS MMA)", bad, 2 * 128 * 256, zero);
  }
  // ---- part 2
  const int region_rows = 8192;
  uint4* src;
  cudaMalloc(&src, (size_t)region_rows * 512);
  cudaMemset(src, 1, (size_t)region_rows * 512);
  const size_t nidx = (size_t)sms * 28 * 65536;
  std::vector<int> h(nidx);
  for (size_t i = 0; i < nidx; ++i) h[i] = lcg(s) % region_rows;
  int* idx;
  cudaMalloc(&idx, nidx * 4);
  cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
  unsigned long long* d;
  cudaMalloc(&d, sms * 16);
  for (int gw : {0, 8, 16, 24}) run_rate<0>(src, idx, gw, 1, sms, d);
  for (int gw : {0, 8, 16, 24}) run_rate<1>(src, idx, gw, 1, sms, d);
  for (int gw : {0, 8, 16, 24}) run_rate<2>(src, idx, gw, 1, sms, d);
  for (int gw : {8, 16, 24}) run_rate<0>(src, idx, gw, 0, sms, d);
  return 0;
}
