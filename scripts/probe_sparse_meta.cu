// Hardware probe (experiment, not product code): recover the TMEM layout of the 2:4 sparse
// metadata read by tcgen05.mma.sp.kind::f16 for M=64 and M=128.
//
// A (M x 16 compressed, K-major) holds a[m][kc] = kc + 1; B (K=32 x N=64, MN-major SW128) is
// the identity, so D[m][n] = A_decompressed[m][n] reveals the two positions selected in every
// 4-wide chunk.  Metadata slot (lane L, nibble j) carries one of the six valid 2:4 patterns
// chosen by base-6 digit r of its slot id; four runs (r = 0..3) identify, for every (row,
// chunk), the slot the tensor core used.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o probe scripts/probe_sparse_meta.cu
#include <cuda_bf16.h>
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

__constant__ uint32_t PAT[6] = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE};

// out: [M][64] floats for each run
__global__ void probe(int M, int run, int id2, int dlane, int elane, int ecol0, float* out) {
  __shared__ __align__(1024) uint8_t sB[4096];
  __shared__ __align__(1024) uint8_t sA[4096];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B: identity 32 x 64, SW128 MN-major: row k at (k/8)*1024 + (k%8)*128, chunk (n/8)^(k%8)
  for (int i = tid; i < 4096 / 2; i += blockDim.x) ((uint16_t*)sB)[i] = 0;
  __syncthreads();
  if (tid < 32) {
    const int k = tid, n = tid;
    const int off = (k / 8) * 1024 + (k % 8) * 128 + (((n / 8) ^ (k % 8)) * 16) + (n % 8) * 2;
    *(__nv_bfloat16*)(sB + off) = __float2bfloat16(1.0f);
  }
  // A: M rows x 16 compressed (K-major, core matrices 8x16B, LBO=128 (K), SBO=256 (rows))
  for (int i = tid; i < M * 16; i += blockDim.x) {
    const int m = i / 16, kc = i % 16;
    const int off = (m / 8) * 256 + (kc / 8) * 128 + (m % 8) * 16 + (kc % 8) * 2;
    *(__nv_bfloat16*)(sA + off) = __float2bfloat16((float)(kc + 1));
  }
  if (tid == 0) {
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
  const uint32_t ECOL = ecol0;
  // metadata: columns ECOL .. ECOL+3, every lane; slot id = (L * 8 + j) + 1024 * col
  {
    const int L = warp * 32 + lane;
    for (int c = 0; c < 4; ++c) {
      uint32_t w = 0;
      for (int j = 0; j < 8; ++j) {
        int slot = (L * 8 + j) + 1024 * c;
        int d = slot;
        for (int r = 0; r < run; ++r) d /= 6;
        w |= PAT[d % 6] << (4 * j);
      }
      uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + ECOL + c;
      if (((lane >> 4) << 4) != elane && elane != 0) w = 0x44444444u;  // only lanes 16-31 carry the pattern
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(w));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                           ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(M >> 4) << 24) | (uint32_t)id2;
    const uint64_t ad = desc(smem_u32(sA), 128, 256, 0);
    const uint64_t bd = desc(smem_u32(sB), 8192, 1024, 2);
    const uint32_t te = tmem + ((uint32_t)elane << 16) + ECOL;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%3], %4, p;\n\t}\n" ::"r"(tmem + ((uint32_t)dlane << 16)),
        "l"(ad), "l"(bd), "r"(te), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // read D: all 128 lanes x 64 columns; store lanes as rows
  for (int c = 0; c < 64; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v)
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[(warp * 32 + lane) * 64 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  static float h[4][128 * 64];
  const int pats[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  struct Cfg { int M, id2, dlane, elane, ecol; } cfgs[] = {
      {64, 0, 0, 16, 256}, {64, 0, 0, 16, 0}, {64, 1, 0, 16, 0}, {128, 0, 0, 0, 256},
      {64, 0, 16, 0, 256}};
  for (auto cf : cfgs) {

    for (int run = 0; run < 4; ++run) {
      cudaMemset(d, 0, 128 * 64 * 4);
      probe<<<1, 128>>>(cf.M, run, cf.id2, cf.dlane, cf.elane, cf.ecol, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("M=%d dlane=%d elane=%d ecol=%d: error %s\n", cf.M, cf.dlane, cf.elane, cf.ecol, cudaGetErrorString(e));
        return 0;  // context is dead after an error
      }
      cudaMemcpy(h[run], d, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    }
    printf("=== M=%d id2=%d dlane=%d elane=%d ecol=%d\n", cf.M, cf.id2, cf.dlane, cf.elane, cf.ecol);
    for (int L = 0; L < 128; ++L) {
      char line[4096];
      int pos = snprintf(line, sizeof line, "lane %3d:", L);
      bool any = false;
      for (int c = 0; c < 8; ++c) {
        int slot = 0, mul = 1;
        bool ok = true;
        for (int run = 0; run < 4; ++run) {
          const float* row = h[run] + L * 64;
          int p0 = -1, p1 = -1;
          for (int q = 0; q < 4; ++q) {
            float v = row[4 * c + q];
            if (v == (float)(2 * c + 1)) p0 = q;
            if (v == (float)(2 * c + 2)) p1 = q;
          }
          int pi = -1;
          for (int k = 0; k < 6; ++k)
            if (pats[k][0] == p0 && pats[k][1] == p1) pi = k;
          if (pi < 0) { ok = false; break; }
          slot += pi * mul;
          mul *= 6;
        }
        if (ok) {
          any = true;
          pos += snprintf(line + pos, sizeof line - pos, " c%d->(col%d,L%d,n%d)", c, slot / 1024,
                          (slot % 1024) / 8, slot % 8);
        } else {
          pos += snprintf(line + pos, sizeof line - pos, " c%d->?", c);
        }
      }
      if (any && (L % 16 == 0 || L % 16 == 8)) printf("%s\n", line);
    }
  }

  return 0;
}
