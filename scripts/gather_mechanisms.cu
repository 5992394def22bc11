// Microbenchmark (experiment, not product code): L2 -> SMEM fill rate of the SpMM's gather with
// the two mechanisms sm_100a offers -- 16-byte cp.async per lane vs TMA tile::gather4 -- with and
// without tcgen05.mma.sp (M=64 N=256 K=32, the V=64 SpMM instruction) streaming on the same SM,
// for two source layouts of the activation rows:
//
//   compact : 8192 rows x 512 B packed (a 4 MB region)  -- what round 1's microbenchmarks used
//   pitched : the SpMM's X (4096 channels x 16384 tokens bf16, 32 KB row pitch, 128 MB), each
//             warp gathering 512-byte row segments of one 256-token block at a time (all SMs
//             walk the token blocks in step, as the SpMM's token-block-major unit order does)
//   blocked : the same X stored token-block-major ([64 blocks][4096 channels][256 tokens]), so a
//             token block is 2 MB contiguous
//
// One CTA per SM.  Warp 0 issues back-to-back MMAs on static operands (or idles for a fixed wall
// of cycles); G gather warps stream random rows until warp 0 is done.
//   cpasync  : lane = 16-byte chunk, one 512-byte row per warp instruction, 8 rows per commit group
//   g4lanes  : every lane issues one gather4 (4 rows x 64 tokens, SWIZZLE_128B box {64,1}),
//              32 per warp step = 16 KB, mbarrier complete_tx per 16 KB slot (2 slots per warp)
//   g4one    : the same 32 gather4 per step issued by one elected lane
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o scripts/bin/gather_mechanisms scripts/gather_mechanisms.cu -lcuda
#include <cuda.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

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

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

enum { CPASYNC = 0, G4LANES = 1, G4ONE = 2, MIX = 3 };  // MIX: warps < ncp cp.async, the rest g4lanes
enum { COMPACT = 0, PITCHED = 1, BLOCKED = 2 };
constexpr int SB = 65536, SA = 16384, SG = 131072;
constexpr int TOK = 16384, NCH = 4096, BLK = 256;

struct Args {
  const uint8_t* src;     // cp.async source base
  const int* idx;         // random row ids
  int rows;               // rows in the row space (8192 compact, 4096 otherwise)
  int layout;
  int iters;
  int do_mma;
  int ncp;
  unsigned long long* out;
};

// byte offset of (row, token block blk, 16-byte chunk c of the 512-byte segment)
__device__ __forceinline__ uint64_t src_off(int layout, int row, int blk, int c) {
  if (layout == COMPACT) return (uint64_t)row * 512 + c * 16;
  if (layout == PITCHED) return (uint64_t)row * (TOK * 2) + (uint64_t)blk * 512 + c * 16;
  return (uint64_t)blk * NCH * 512 + (uint64_t)row * 512 + c * 16;
}

template <int MECH, int SLOTB = 16384, int NSLOT = 2>
__global__ void bench(Args a, const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint64_t gbar[32][8];
  __shared__ uint32_t tmem_base;
  __shared__ volatile int stop;
  __shared__ unsigned long long bytes_done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sB = sm;
  uint8_t* sA = sm + SB;
  const uint32_t sG = smem_u32(sm + SB + SA);
  for (int i = threadIdx.x; i < (SB + SA) / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    stop = 0;
    bytes_done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int w = 0; w < 32; ++w)
      for (int s = 0; s < 8; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&gbar[w][s])));
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
    const uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                           ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sA), 128, 256, 0);
    const uint64_t bd = desc(smem_u32(sB), 16384, 1024, 2);
    const uint32_t te = tmem + 504;
    if (a.do_mma) {
      for (int i = 0; i < a.iters; i += 8) {
        if (elect_one()) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%4], %3, 1;\n" ::"r"(tmem), "l"(ad),
                         "l"(bd), "r"(idesc), "r"(te));
        }
        __syncwarp();
      }
      if (elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      __syncwarp();
      mbar_wait(smem_u32(&bar), 0);
    } else {
      while (clock64() - t0 < (long long)a.iters * 144) {}
    }
    const long long t1 = clock64();
    if (lane == 0) {
      stop = 1;
      a.out[blockIdx.x * 2 + 0] = (unsigned long long)(t1 - t0);
    }
  } else if (warp >= 4) {
    const int gw = warp - 4, ngw = (blockDim.x >> 5) - 4;
    const int* my = a.idx + ((size_t)blockIdx.x * ngw + gw) * 65536;
    unsigned long long bytes = 0;
    int r0 = 0;
    // every SM walks the token blocks in step: one block per 2048 rows gathered by the SM (a unit)
    if (MECH == CPASYNC || (MECH == MIX && gw < a.ncp)) {
      const uint32_t ring = sG + (MECH == MIX ? gw % 8 : gw % 16) * 8192 + lane * 16;
      int k = 0;
      while (!stop) {
        const int mine = __ldg(my + (r0 & 65535) + lane);
        const int blk = ((r0 * ngw) >> 11) & 63;
        r0 += 32;
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const int row = __shfl_sync(0xffffffffu, mine, j);
          asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(ring + (j & 15) * 512),
                       "l"(a.src + src_off(a.layout, row, blk, lane))
                       : "memory");
          if (++k == 8) {
            k = 0;
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 4;" ::: "memory");
          }
        }
        bytes += 32 * 512;
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
      // NSLOT slots of SLOTB bytes per warp; lane l < SLOTB/512 issues gather4 l of a fill (quad l/4 of
      // 4 rows, 64-token chunk l%4); G4ONE: lane 0 issues all of them
      constexpr int NG4 = SLOTB / 512;
      const int tw = MECH == MIX ? gw - a.ncp : gw;  // TMA warp index
      const uint32_t slot0 = sG + (MECH == MIX ? 65536 : 0) + tw * NSLOT * SLOTB;
      int s = 0;
      int uses[NSLOT];
#pragma unroll
      for (int q = 0; q < NSLOT; ++q) uses[q] = 0;
      while (!stop) {
        const uint32_t b = smem_u32(&gbar[gw][s]);
        if (uses[s] >= 1) mbar_wait(b, (uses[s] - 1) & 1);  // this slot's previous fill landed
        const int mine = __ldg(my + (r0 & 65535) + lane);  // row ids: quad q = lanes 4q..4q+3
        const int blk = ((r0 * ngw) >> 11) & 63;
        r0 += NG4;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(SLOTB) : "memory");
        __syncwarp();
        // gather4 coordinates {token, row0..row3} of 2-D maps (tokens, rows)
        const int tok_base = a.layout == PITCHED ? blk * BLK : 0;
        const int radd = a.layout == BLOCKED ? blk * NCH : 0;
        int rr[NG4];
#pragma unroll
        for (int l = 0; l < NG4; ++l) rr[l] = __shfl_sync(0xffffffffu, mine, l) + radd;
        auto issue = [&](int l) {
          const int quad = l >> 2, chunk = l & 3;
          const uint32_t dst = slot0 + s * SLOTB + chunk * (SLOTB / 4) + quad * 512;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(&map), "r"(b), "r"(tok_base + chunk * 64),
              "r"(rr[quad * 4]), "r"(rr[quad * 4 + 1]), "r"(rr[quad * 4 + 2]), "r"(rr[quad * 4 + 3])
              : "memory");
        };
        if (MECH == G4LANES || MECH == MIX) {
#pragma unroll
          for (int l = 0; l < NG4; ++l)
            if (lane == l) issue(l);
        } else if (lane == 0) {
#pragma unroll
          for (int l = 0; l < NG4; ++l) issue(l);
        }
        __syncwarp();
        ++uses[s];
        bytes += SLOTB;
        if (++s == NSLOT) s = 0;
      }
#pragma unroll
      for (int q = 0; q < NSLOT; ++q)  // drain the outstanding fills
        if (uses[q] >= 1) mbar_wait(smem_u32(&gbar[gw][q]), (uses[q] - 1) & 1);
    }
    if (lane == 0) atomicAdd(&bytes_done, bytes);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x == 0) a.out[blockIdx.x * 2 + 1] = bytes_done;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(void* base, int layout) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  memset(&m, 0, sizeof m);
  cuuint64_t dims[2], strides[1];
  if (layout == COMPACT) { dims[0] = 256; dims[1] = 8192; strides[0] = 512; }
  else if (layout == PITCHED) { dims[0] = TOK; dims[1] = NCH; strides[0] = TOK * 2; }
  else { dims[0] = 256; dims[1] = (cuuint64_t)NCH * (TOK / 256); strides[0] = 512; }
  cuuint32_t box[2] = {64, 1}, estr[2] = {1, 1};
  CUresult r = ((EncodeTiledFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tensor map failed %d\n", (int)r); exit(1); }
  return m;
}

static bool g_quiet = false;
static double g_last = 0;
static const char* MECH_NAME[] = {"cpasync", "g4lanes", "g4one", "mix"};
static const char* LAYOUT_NAME[] = {"compact", "pitched", "blocked"};

template <int MECH, int SLOTB = 16384, int NSLOT = 2>
void run(uint8_t* x, int* idx, int layout, int gwarps, int do_mma, int sms, unsigned long long* d, int ncp = 0) {
  Args a;
  a.ncp = ncp;
  a.src = x;
  a.idx = idx;
  a.rows = layout == COMPACT ? 8192 : NCH;
  a.layout = layout;
  a.do_mma = do_mma;
  a.out = d;
  CUtensorMap map = make_map(x, layout);
  const int smem = SB + SA + SG + 1024;
  cudaFuncSetAttribute(bench<MECH, SLOTB, NSLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  a.iters = 64;
  bench<MECH, SLOTB, NSLOT><<<sms, 32 * (4 + gwarps), smem>>>(a, map);
  a.iters = 16384;
  bench<MECH, SLOTB, NSLOT><<<sms, 32 * (4 + gwarps), smem>>>(a, map);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[1024];
  cudaMemcpy(h, d, sms * 16, cudaMemcpyDeviceToHost);
  double cyc = 0, bytes = 0;
  for (int i = 0; i < sms; ++i) { cyc += h[2 * i]; bytes += h[2 * i + 1]; }
  cyc /= sms;
  bytes /= sms;
  g_last = bytes / cyc;
  if (g_quiet) return;
  printf("%-8s ncp %2d slot %5d x %d  %-8s gather_warps %2d  mma %s  cycles/mma %7.1f  fill %6.1f B/clk/SM (%5.2f TB/s at 1.965 GHz)\n",
         MECH_NAME[MECH], ncp, MECH == CPASYNC ? 0 : SLOTB, MECH == CPASYNC ? 0 : NSLOT, LAYOUT_NAME[layout], gwarps, do_mma ? "on " : "off", do_mma ? cyc / 16384 : 0.0,
         bytes / cyc, bytes / cyc * sms * 1.965e9 / 1e12);
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* x;
  const size_t xbytes = (size_t)NCH * TOK * 2;   // 128 MB
  cudaMalloc(&x, xbytes);
  cudaMemset(x, 1, xbytes);
  const size_t nidx = (size_t)sms * 28 * 65536;
  int* h = (int*)malloc(nidx * 4);
  int* idx;
  cudaMalloc(&idx, nidx * 4);
  unsigned long long* d;
  cudaMalloc(&d, sms * 16);
  if (argc > 1 && !strcmp(argv[1], "--ceiling")) {
    // the SpMM's own layout (pitched X rows): cp.async fill with and without the M=64 MMA stream,
    // best of 16 / 24 / 28 issuing warps; one JSON line for bench.py
    uint32_t s = 777u;
    for (size_t i = 0; i < nidx; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % NCH; }
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    g_quiet = true;
    double best[2] = {0, 0};
    for (int mma : {0, 1})
      for (int g : {16, 24, 28}) {
        run<CPASYNC>(x, idx, PITCHED, g, mma, sms, d);
        if (g_last > best[mma]) best[mma] = g_last;
      }
    printf("{\"fill_alone_bclk_sm\": %.1f, \"fill_under_mma_bclk_sm\": %.1f, \"sms\": %d, "
           "\"mechanism\": \"cp.async 16 B/lane, 16-28 warps, 512-byte rows of a 32 KB-pitched X\"}\n",
           best[0], best[1], sms);
    return 0;
  }
  for (int layout : {COMPACT, PITCHED}) {
    const int rows = layout == COMPACT ? 8192 : NCH;
    uint32_t s = 777u;
    for (size_t i = 0; i < nidx; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) % rows; }
    cudaMemcpy(idx, h, nidx * 4, cudaMemcpyHostToDevice);
    for (int mma : {0, 1}) {
      for (int g : {16, 24, 28}) run<CPASYNC>(x, idx, layout, g, mma, sms, d);
      // TMA gather4: warps x slots x slot bytes <= 128 KB
      run<G4LANES, 16384, 8>(x, idx, layout, 1, mma, sms, d);
      run<G4LANES, 16384, 2>(x, idx, layout, 4, mma, sms, d);
      run<G4LANES, 16384, 1>(x, idx, layout, 8, mma, sms, d);
      run<G4LANES, 8192, 2>(x, idx, layout, 8, mma, sms, d);
      run<G4LANES, 8192, 1>(x, idx, layout, 16, mma, sms, d);
      run<G4LANES, 4096, 2>(x, idx, layout, 16, mma, sms, d);
      run<G4LANES, 4096, 1>(x, idx, layout, 28, mma, sms, d);
      run<G4LANES, 2048, 2>(x, idx, layout, 28, mma, sms, d);
      run<G4ONE, 16384, 1>(x, idx, layout, 8, mma, sms, d);
      // cp.async warps (ring in the first 64 KB) + TMA warps (the other 64 KB)
      run<MIX, 4096, 2>(x, idx, layout, 24, mma, sms, d, 16);
      run<MIX, 4096, 1>(x, idx, layout, 28, mma, sms, d, 12);
      run<MIX, 8192, 1>(x, idx, layout, 24, mma, sms, d, 16);
    }
  }
  return 0;
}
