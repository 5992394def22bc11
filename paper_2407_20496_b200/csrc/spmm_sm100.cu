// HiNM SpMM on Blackwell (sm_100a): TMA gather4 of the kept activation rows + 2:4 sparse
// tcgen05.mma.sp into TMEM + fused sigma_o row-scatter epilogue.
//
//   Y[sigma_o[tV + r], b] = sum_k A_t[r, k] * X[gidx_t[k], b]      (spmm.py:88-98 + pruning.py:356)
//
// Work unit = (tile t, block of BN=256 tokens).  Persistent grid (one CTA per SM), units
// distributed round-robin in token-block-major order so the X token block stays L2 resident
// while every tile consumes it.
//
// Warp roles (192 threads):
//   warp 0      producer: per 64-K stage, one bulk copy of the compressed A block (V x 64 B),
//               one bulk copy of the 2:4 metadata every other stage (V x 16 B for 128 K), and
//               64 TMA gather4 (16 lanes x 4 token sub-blocks) of X rows -> SWIZZLE_128B
//               MN-major B operand (64 K-rows x 256 tokens)
//   warp 1      TMEM allocator + single-thread MMA issuer: tcgen05.cp of the metadata into a
//               TMEM ring, 2 x tcgen05.mma.sp (M=128, N=256, K=32) per stage, tcgen05.commit
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 -> bf16 -> 16 B stores to row sigma_o[tV+r]
//
// V = 64 (and 32) use the M=128 instruction with rows >= V ignored: the A descriptor's upper
// row groups alias neighbouring smem and those accumulator lanes are never read.  The M=128
// and M=64 instructions cost the same tensor-pipe cycles (B300_MICROARCH.md: floor =
// max(M,128)*N/256), so this costs smem read bandwidth only.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace hinm {
namespace sm100 {

constexpr int BN = 256;                        // tokens per unit (UMMA N)
constexpr int BK = 64;                         // logical K per pipeline stage
constexpr int STAGES = 5;
constexpr int B_STAGE = BK * BN * 2;           // 32 KB of gathered X per stage
constexpr int E_STAGE = 128 * 16;              // 128 lanes x 16 B metadata image per stage slot
constexpr int TMEM_COLS = 512;
constexpr int E_COL = 256;                     // metadata ring after the 256-column accumulator
constexpr int E_SLOTS = 4;
constexpr uint32_t META_PAD = 0x44444444u;     // 2:4 nibble {0,1} for rows >= V

struct Params {
  const int32_t* tile_kofs;
  const int32_t* tile_eofs;
  const int32_t* gidx;
  const uint16_t* a_vals;
  const uint32_t* a_meta;
  const int32_t* sigma_o;
  uint16_t* Y;
  int64_t ldy;
  int B;
  int T;
  int V;
  int units;
  int out_order;
};

struct SmemLayout {
  uint32_t a, e, bar, tmem, total;
};

__host__ __device__ inline SmemLayout smem_layout(int V) {
  SmemLayout L;
  L.a = STAGES * B_STAGE;
  L.e = L.a + STAGES * V * 64 + 4096;          // 4 KB slack: M=128 descriptor over-read
  L.bar = L.e + STAGES * E_STAGE;
  L.tmem = L.bar + (2 * STAGES + 4) * 8;
  L.total = L.tmem + 16 + 1024;                // + alignment slack for the 1 KB base
  return L;
}

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Parity wait with a watchdog: a protocol bug traps (kernel error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(done)
      : "r"(bar), "r"(parity)
      : "memory");
  if (done) return;
  const uint64_t t0 = globaltimer();
  while (true) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (globaltimer() - t0 > 4000000000ull) __trap();
  }
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int col, int4 rows,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(col), "r"(rows.x), "r"(rows.y), "r"(rows.z), "r"(rows.w), "r"(bar)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// parity to wait on for the n-th (0-based) use of a buffer guarded by an "empty" barrier
__device__ __forceinline__ uint32_t phase_acc_empty_parity(uint32_t n) { return (n & 1) ^ 1; }

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// UMMA shared-memory matrix descriptor (tcgen05 format, version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                      // descriptor version (Blackwell)
  d |= (uint64_t)(layout & 7) << 61;           // 0 = none, 2 = 128B swizzle
  return d;
}

// Instruction descriptor: sparse kind::f16, BF16 x BF16 -> F32, A K-major, B MN-major.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 2)                 // sparse
         | (1u << 4)               // D = F32
         | (1u << 7)               // A = BF16
         | (1u << 10)              // B = BF16
         | (0u << 15)              // A K-major
         | (1u << 16)              // B MN-major
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_sp(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t tmem_e, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(tmem_e)
      : "memory");
}

__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo_f32, uint32_t hi_f32) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo_f32), __uint_as_float(hi_f32));
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------------------------ the kernel
// Warp layout: warps 0-3 epilogue (TMEM lane quadrant = warp), warp 4 MMA issuer + TMEM owner,
// warp 5 A/metadata producer (bulk copies), warps 6.. gather producers.
constexpr int EPI_WARPS = 4;
constexpr int MMA_WARP = 4;
constexpr int AE_WARP = 5;
constexpr int GATHER_WARP0 = 6;

enum GatherMode : int { GATHER_CPASYNC = 0, GATHER_TMA = 1, GATHER_LDG = 2 };

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}

// Per-unit parameters.  Each role loads the NEXT unit's parameters while it works on the
// current one: under load the SM's L1tex queue is full of gather traffic and a dependent
// global load at a unit boundary would otherwise stall ~3k cycles.
struct UnitParams {
  int t, nb, k0, kp, e0;
};

__device__ __forceinline__ UnitParams unit_params(const Params& p, int u) {
  UnitParams q;
  if (u >= p.units) {
    q.t = q.nb = q.k0 = q.kp = q.e0 = 0;
    return q;
  }
  q.t = u % p.T;
  q.nb = u / p.T;
  q.k0 = __ldg(p.tile_kofs + q.t);
  q.kp = __ldg(p.tile_kofs + q.t + 1) - q.k0;
  q.e0 = __ldg(p.tile_eofs + q.t);
  return q;
}

// DBG (experiments only): 1 = skip the MMAs (measure the gather pipeline alone),
// 2 = skip the gather (measure the MMA pipeline alone).  Results are garbage when DBG != 0.
// M64: V <= 64 on the M=64 instruction (half the A-operand shared-memory reads of M=128).  Its
// accumulator row 16q+l sits in TMEM lane 32q+l and its metadata where M=128 row 32q+l would
// (lanes 32q+0..15) -- measured with scripts/probe_sparse_meta.cu, which also shows that an
// M=64 accumulator at lane offset 16 faults (misaligned address), so one accumulator is used.
template <int MODE, int GW, int DBG = 0, bool M64 = false>
__global__ void __launch_bounds__(32 * (GATHER_WARP0 + GW), 1)
    k_hinm_spmm(const __grid_constant__ CUtensorMap xmap, const uint16_t* __restrict__ X,
                int64_t ldx, Params p) {
  constexpr int NT = 32 * (GATHER_WARP0 + GW);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const SmemLayout L = smem_layout(p.V);
  const int V = p.V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sB = base, sA = base + L.a, sE = base + L.e;
  const uint32_t bar_full = base + L.bar, bar_empty = bar_full + STAGES * 8;
  constexpr int NACC = 1;  // accumulator buffers
  const uint32_t bar_acc_full = bar_empty + STAGES * 8;   // [NACC]
  const uint32_t bar_acc_empty = bar_acc_full + 16;       // [NACC]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + L.tmem);
  // warps (= TMEM lane quadrants) that hold real rows
  const int n_epi_warps = M64 ? V / 16 : (V >= 128 ? 4 : V / 32);

  // constant metadata for lanes the producer never writes (rows >= V, M=64 gap lanes)
  if (M64) {
    for (int i = threadIdx.x; i < STAGES * E_STAGE / 4; i += NT)
      reinterpret_cast<uint32_t*>(gbase + L.e)[i] = META_PAD;
  } else {
    for (int i = threadIdx.x; i < STAGES * (128 - V) * 4; i += NT) {
      const int s = i / ((128 - V) * 4), w = i % ((128 - V) * 4);
      reinterpret_cast<uint32_t*>(gbase + L.e + s * E_STAGE + V * 16)[w] = META_PAD;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // cp.async mode: 1 expect_tx arrive + one noinc arrive per gather thread
      mbar_init(bar_full + 8 * s, MODE != GATHER_TMA ? 1 + 32 * GW : 1);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(bar_acc_full + 8 * a, 1);
      mbar_init(bar_acc_empty + 8 * a, n_epi_warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (MODE == GATHER_TMA) asm volatile("prefetch.tensormap [%0];" ::"l"(&xmap) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int T = p.T;

  if (warp == AE_WARP) {
    // ============================================================ A / metadata producer
    // warp-uniform loop; one elected lane issues the bulk copies (see the MMA issuer note)
    int stage = 0;
    uint32_t phase = 0;
    UnitParams nxt = unit_params(p, blockIdx.x);
    const uint32_t a_bytes = V * 64;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const UnitParams cur = nxt;
      nxt = unit_params(p, u + gridDim.x);
      const int nst = cur.kp / BK;
      const uint16_t* asrc = p.a_vals + (int64_t)cur.k0 * V / 2;
      const uint32_t* esrc0 = p.a_meta + (int64_t)cur.e0 * V * 4;
      for (int s = 0; s < nst; ++s) {
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        const uint32_t fb = bar_full + 8 * stage;
        if (elect_one()) {
          if (DBG == 3) {  // experiment: no operand loads at all
            mbar_arrive(fb);
          } else {
            const uint32_t e_bytes = (s & 1) ? 0 : V * 16;
            mbar_expect_tx(fb, a_bytes + e_bytes + (MODE == GATHER_TMA ? B_STAGE : 0));
            bulk_g2s(sA + stage * a_bytes, asrc + (int64_t)s * BK * V / 2, a_bytes, fb);
            if (e_bytes) {
              const uint32_t* esrc = esrc0 + (int64_t)(s / 2) * V * 4;
              if (M64) {  // 16-lane groups of the stored (M=128 order) image -> lanes 32q + 0..15
                for (int q = 0; q < V / 16; ++q)
                  bulk_g2s(sE + stage * E_STAGE + q * 512, esrc + q * 64, 256, fb);
              } else {
                bulk_g2s(sE + stage * E_STAGE, esrc, e_bytes, fb);
              }
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= GATHER_WARP0) {
    // ============================================================ gather producers
    // Flattened stream over (unit, stage) with the gather indices of stage i+PF loaded while
    // stage i is issued (the dependent index load never sits on the critical path).  The
    // issue loop is kept to ~4 instructions per 512-byte row: warp gw owns the K-rows
    // r = gw + GW*i of every stage, lane = 16-byte chunk of the row.
    const int gw = warp - GATHER_WARP0;
    constexpr int PF = 8;
    constexpr int RPW = BK / GW;  // K-rows per warp per stage
    static_assert(MODE == GATHER_TMA || GW == 8, "cp.async/LDG producers assume 8 gather warps");
    const int dt = gridDim.x % T, dnb = gridDim.x / T;
    // prefetch cursor: unit (pt, pnb) with running index pu, stage ps of pnst
    int pu = blockIdx.x, pt = blockIdx.x % T, pnb = blockIdx.x / T, ps = 0, pk0 = 0, pnst = 0;
    auto next_unit = [&]() {  // advance to the next unit with work
      while (pu < p.units) {
        pk0 = __ldg(p.tile_kofs + pt);
        pnst = (__ldg(p.tile_kofs + pt + 1) - pk0) / BK;
        if (pnst > 0) break;
        pu += gridDim.x;
        pt += dt;
        pnb += dnb;
        if (pt >= T) { pt -= T; ++pnb; }
      }
      ps = 0;
    };
    next_unit();
    int r_row[PF], r_col[PF];
    int4 r_quad[PF];
    bool r_ok[PF];
    auto prefetch = [&](int slot) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        if (j != slot) continue;
        r_ok[j] = pu < p.units;
        if (!r_ok[j]) return;
        r_col[j] = pnb * BN;
        const int* gi = p.gidx + pk0 + ps * BK;
        if (MODE != GATHER_TMA) {
          r_row[j] = lane < RPW ? __ldg(gi + gw + lane * GW) : 0;
        } else {
          const int g = gw * 32 + lane;
          r_quad[j] = g < 64 ? __ldg(reinterpret_cast<const int4*>(gi) + (g >> 2)) : make_int4(0, 0, 0, 0);
        }
        if (++ps == pnst) {
          pu += gridDim.x;
          pt += dt;
          pnb += dnb;
          if (pt >= T) { pt -= T; ++pnb; }
          next_unit();
        }
      }
    };
#pragma unroll
    for (int j = 0; j < PF; ++j) prefetch(j);
    // per-warp constant part of the SWIZZLE_128B destination (row r = gw + 8 i: r & 7 = gw)
    const uint32_t dst_lane = (lane >> 3) * (B_STAGE / 4) + gw * 128 + (((lane & 7) ^ gw) << 4);
    const char* xbase = reinterpret_cast<const char*>(X);
    const int64_t ldx2 = ldx * 2;
    int stage = 0;
    uint32_t phase = 0;
    bool done = false;
    if (MODE == GATHER_LDG) {
      // register-staged gather: the rows of stage i+1 are loaded (LDG) before waiting for the
      // stage-i slot, adding one stage of in-flight data held in registers
      uint4 bufA[RPW], bufB[RPW];
      auto ldg_rows = [&](uint4 (&buf)[RPW], int slot) {
#pragma unroll
        for (int jj = 0; jj < PF; ++jj) {
          if (jj != slot) continue;
          const int tok = r_col[jj] + lane * 8;
          const bool in = r_ok[jj] && tok < p.B;
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            const int row = __shfl_sync(0xffffffffu, r_row[jj], i);
            buf[i] = in ? __ldg(reinterpret_cast<const uint4*>(xbase + row * ldx2 + (int64_t)tok * 2))
                        : make_uint4(0, 0, 0, 0);
          }
        }
      };
      ldg_rows(bufA, 0);
      while (!done) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
          if (!r_ok[j]) { done = true; break; }
          uint4(&cur)[RPW] = (j & 1) ? bufB : bufA;
          uint4(&nxt)[RPW] = (j & 1) ? bufA : bufB;
          ldg_rows(nxt, (j + 1) % PF);
          mbar_wait(bar_empty + 8 * stage, phase ^ 1);
          const uint32_t dst0 = sB + stage * B_STAGE + dst_lane;
#pragma unroll
          for (int i = 0; i < RPW; ++i)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst0 + i * 1024),
                         "r"(cur[i].x), "r"(cur[i].y), "r"(cur[i].z), "r"(cur[i].w)
                         : "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(bar_full + 8 * stage);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          prefetch(j);
        }
      }
    }
    while (MODE != GATHER_LDG && !done) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        if (!r_ok[j]) { done = true; break; }
        const int col0 = r_col[j];
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        if (MODE == GATHER_CPASYNC) {
          const int tok = col0 + lane * 8;
          const uint32_t src_bytes = tok < p.B ? 16u : 0u;
          const char* xs = xbase + (src_bytes ? (int64_t)tok * 2 : 0);
          const uint32_t dst0 = sB + stage * B_STAGE + dst_lane;
          const int my_row = r_row[j];
#pragma unroll
          for (int i = 0; i < RPW; ++i) {
            const int row = __shfl_sync(0xffffffffu, my_row, i);
            if (DBG != 2 && DBG != 3) cp_async_16(dst0 + i * 1024, xs + row * ldx2, src_bytes);
          }
          cp_async_arrive_noinc(bar_full + 8 * stage);
        } else {
          const int g = gw * 32 + lane;
          if (g < 64) {
            const int quad = g >> 2, q = g & 3;
            tma_gather4(sB + stage * B_STAGE + q * (B_STAGE / 4) + quad * 512, &xmap,
                        col0 + q * 64, r_quad[j], bar_full + 8 * stage);
          }
        }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        prefetch(j);
      }
    }
  } else if (warp == MMA_WARP) {
    // ============================================================ MMA issuer
    // The whole warp runs the loop (warp-uniform control flow keeps every descriptor in uniform
    // registers); one elected lane issues the tcgen05 instructions.  A single-lane loop forced
    // R2UR conversions of every operand per MMA and measured 2.6x slower MMA issue
    // (scripts/mma_bench.cu vs mma_bench_v1.cu).
    const uint32_t idesc = make_idesc(M64 ? 64 : 128, BN);
    // descriptors at stage 0; the start-address field (16 B units, bits 0-13) is advanced by
    // adding byte offsets >> 4
    const uint64_t a_desc0 = smem_desc(sA, 128, 256, 0);
    const uint64_t b_desc0 = smem_desc(sB, B_STAGE / 4, 1024, 2);
    const uint64_t e_desc0 = smem_desc(sE, 0, 128, 0);
    const uint32_t a_step = (uint32_t)(V * 64) >> 4, a_half = (uint32_t)(32 * V) >> 4;
    int stage = 0;
    uint32_t phase = 0, eslot = 0, acc_uses = 0;
    UnitParams nxt = unit_params(p, blockIdx.x);
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
      const int kp = nxt.kp;
      nxt = unit_params(p, u + gridDim.x);
      if (kp == 0) continue;
      const uint32_t acc = 0;
      mbar_wait(bar_acc_empty, phase_acc_empty_parity(acc_uses));
      ++acc_uses;
      tc_fence_after();
      const int nst = kp / BK;
      for (int s = 0; s < nst; ++s) {
        mbar_wait(bar_full + 8 * stage, phase);
        tc_fence_after();
        if (elect_one()) {
          if ((s & 1) == 0) {
            eslot = (eslot + 1) & (E_SLOTS - 1);
            tmem_cp_128x128b(tmem + E_COL + eslot * 4, e_desc0 + (uint64_t)((stage * E_STAGE) >> 4));
          }
          const uint32_t ecol = tmem + E_COL + eslot * 4 + (s & 1) * 2;
          const uint64_t ad = a_desc0 + (uint64_t)(stage * a_step);
          const uint64_t bd = b_desc0 + (uint64_t)((stage * B_STAGE) >> 4);
          if (DBG != 1) {
            mma_sp(tmem, ad, bd, idesc, ecol, s ? 1u : 0u);                       // id2 = 0
            mma_sp(tmem, ad + a_half, bd + (4096 >> 4), idesc | 1u, ecol, 1u);    // id2 = 1
          }
          tc_commit(bar_empty + 8 * stage);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) tc_commit(bar_acc_full);
      __syncwarp();
      (void)acc;
    }
  } else {
    // ============================================================ epilogue (warps 0-3)
    const int q = warp;  // TMEM lane quadrant of this warp
    if (q < n_epi_warps) {
      uint32_t ucount = 0;
      // row of this thread: M=128 -> lane; M=64 -> lanes 0-15 hold rows 16q + 0..15
      const int r = M64 ? q * 16 + (lane & 15) : q * 32 + lane;
      auto out_row = [&](const UnitParams& q) -> int64_t {
        const int64_t prow = (int64_t)q.t * V + r;
        return p.out_order == HINM_ORDER_ORIGINAL ? (int64_t)__ldg(p.sigma_o + prow) : prow;
      };
      UnitParams nxt = unit_params(p, blockIdx.x);
      int64_t nxt_row = blockIdx.x < p.units ? out_row(nxt) : 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const UnitParams cur = nxt;
        const int64_t orow = nxt_row;
        nxt = unit_params(p, u + gridDim.x);
        if (u + (int)gridDim.x < p.units) nxt_row = out_row(nxt);
        const int nb = cur.nb, kp = cur.kp;
        uint16_t* yrow = p.Y + orow * p.ldy;
        const int col_base = nb * BN;
        if (kp == 0) {  // empty tile: zero rows (spmm.py:89-90)
          if (M64 && lane >= 16) continue;
          for (int c = 0; c < BN; c += 8)
            if (col_base + c < p.B)
              *reinterpret_cast<uint4*>(yrow + col_base + c) = make_uint4(0, 0, 0, 0);
          continue;
        }
        const uint32_t acc = ucount % NACC, use = ucount / NACC;
        ++ucount;
        const bool mine = !M64 || lane < 16;
        mbar_wait(bar_acc_full + 8 * acc, use & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c * 32, v);
          const int col = col_base + c * 32;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            if (mine && col + h * 8 < p.B) {
              uint4 o;
              o.x = pack_bf16x2(v[h * 8 + 0], v[h * 8 + 1]);
              o.y = pack_bf16x2(v[h * 8 + 2], v[h * 8 + 3]);
              o.z = pack_bf16x2(v[h * 8 + 4], v[h * 8 + 5]);
              o.w = pack_bf16x2(v[h * 8 + 6], v[h * 8 + 7]);
              *reinterpret_cast<uint4*>(yrow + col + h * 8) = o;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_acc_empty + 8 * acc);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace sm100
}  // namespace hinm

// ------------------------------------------------------------------------------ host side
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)ptr;
  }
  return fn;
}

thread_local int g_last_launches = 0;

int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

extern "C" int hinm_last_launch_count(void) { return g_last_launches; }

extern "C" int hinm_spmm_bf16(const hinm_pack_t* pk, const uint16_t* X, int64_t ldx, int B,
                              uint16_t* Y, int64_t ldy, int out_order, void* stream) {
  using namespace hinm::sm100;
  g_last_launches = 0;
  if (!pk || !X || !Y) return HINM_ERR_VALUE;
  if (pk->N != 2 || pk->M != 4) return HINM_ERR_UNSUPPORTED;
  if (pk->V != 32 && pk->V != 64 && pk->V != 128) return HINM_ERR_UNSUPPORTED;
  if (!pk->gidx || !pk->a_vals || !pk->a_meta || !pk->tile_kofs) return HINM_ERR_VALUE;
  if (B < 0 || (B % 8) || (ldx % 8) || (ldy % 8) || ldx < B || ldy < B) return HINM_ERR_VALUE;
  if (((uintptr_t)X & 15) || ((uintptr_t)Y & 15)) return HINM_ERR_VALUE;
  if (B == 0 || pk->m == 0) return HINM_OK;
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return HINM_ERR_CUDA;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)pk->n};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)X, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    fprintf(stderr, "[hinm] cuTensorMapEncodeTiled failed (%d)\n", (int)cr);
    return HINM_ERR_CUDA;
  }
  Params prm;
  prm.tile_kofs = pk->tile_kofs;
  prm.tile_eofs = pk->tile_eofs;
  prm.gidx = pk->gidx;
  prm.a_vals = pk->a_vals;
  prm.a_meta = pk->a_meta;
  prm.sigma_o = pk->sigma_o;
  prm.Y = Y;
  prm.ldy = ldy;
  prm.B = B;
  prm.T = pk->T;
  prm.V = pk->V;
  const int nbk = (B + BN - 1) / BN;
  prm.units = nbk * pk->T;
  prm.out_order = out_order;
  const SmemLayout L = smem_layout(pk->V);
  const int grid = std::min(prm.units, sm_count());
  // variant: cp.async gather with 4 (default) or 8 warps, or TMA gather4 with 2 / 4 warps
  static const int variant = [] {
    const char* e = getenv("HINM_GATHER");
    if (!e) return 0;
    if (!strcmp(e, "cp8")) return 1;
    if (!strcmp(e, "tma") || !strcmp(e, "tma2")) return 2;
    if (!strcmp(e, "tma4")) return 3;
    if (!strcmp(e, "dbg_nomma")) return 4;
    if (!strcmp(e, "dbg_nogather")) return 5;
    if (!strcmp(e, "m128")) return 6;
    if (!strcmp(e, "ldg8")) return 9;
    if (!strcmp(e, "dbg_noload")) return 7;
    if (!strcmp(e, "dbg_noload128")) return 8;
    return 0;
  }();
  cudaStream_t st = (cudaStream_t)stream;
  auto launch = [&](auto kern, int gw) -> int {
    HINM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    kern<<<grid, 32 * (GATHER_WARP0 + gw), L.total, st>>>(map, X, ldx, prm);
    return HINM_OK;
  };
  int rc;
  switch (variant) {
    case 1: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8>, 8); break;
    case 2: rc = launch(k_hinm_spmm<GATHER_TMA, 2>, 2); break;
    case 3: rc = launch(k_hinm_spmm<GATHER_TMA, 4>, 4); break;
    case 4: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8, 1>, 8); break;
    case 5: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8, 2>, 8); break;
    case 6: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8, 0, false>, 8); break;  // M=128 for any V
    case 7: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8, 3, true>, 8); break;
    case 8: rc = launch(k_hinm_spmm<GATHER_CPASYNC, 8, 3, false>, 8); break;
    case 9: rc = launch(k_hinm_spmm<GATHER_LDG, 8, 0, true>, 8); break;
    default:
      rc = pk->V <= 64 ? launch(k_hinm_spmm<GATHER_CPASYNC, 8, 0, true>, 8)
                       : launch(k_hinm_spmm<GATHER_CPASYNC, 8, 0, false>, 8);
      break;
  }
  if (rc) return rc;
  HINM_LAUNCH_CHECK();
  g_last_launches = 1;
  return HINM_OK;
}
