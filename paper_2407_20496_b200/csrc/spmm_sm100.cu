// HiNM SpMM on Blackwell (sm_100a): cp.async gather of the kept activation rows + 2:4 sparse
// tcgen05.mma.sp into TMEM + fused sigma_o row-scatter epilogue.
//
//   Y[sigma_o[tV + r], b] = sum_k A_t[r, k] * X[gidx_t[k], b]      (spmm.py:88-98 + pruning.py:356)
//
// Work unit = (tile t, block of BN = 256 tokens).  Persistent grid (one CTA per SM), units
// distributed round-robin in token-block-major order so the X token block stays L2 resident
// while every tile consumes it.
//
// Warp roles (32 * (6 + GW) threads):
//   warps 0-3   epilogue: TMEM lane quadrant = warp; paired tcgen05.ld (16x32bx2 for M=64) ->
//               bf16 -> 16-byte stores to row sigma_o[tV + r] (L2 evict_first)
//   warp 4      TMEM owner + MMA issuer (one elected lane, warp-uniform loop): per X stage the
//               metadata tcgen05.cp into a TMEM ring and 2 or 4 tcgen05.mma.sp (M = 64 for
//               V <= 64, else 128; N = 256; K = 32)
//   warp 5      A / metadata producer: one bulk copy per X stage (L2 evict_last) into its own
//               deeper ring with its own barriers
//   warps 6..   GW gather producers: 16-byte cp.async per lane, one 512-byte X row per warp
//               instruction, SWIZZLE_128B MN-major B operand, completion via
//               cp.async.mbarrier.arrive.noinc; indices prefetched 8 stages ahead
//
// One accumulator: a second one (to overlap a unit's drain with the next unit's MMAs) does not
// fit next to the metadata ring at N = 256, and N = 240 units break the 512-byte alignment of
// the gathered row segments (gather-only time 0.72 -> 0.97 ms on the LLaMA up projection).
// Design measurements behind this layout: profiles/r01_gather_microbench.txt.
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <initializer_list>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace hinm {
namespace sm100 {

// Tokens per unit (UMMA N), a template parameter BNT of the kernel: 256 (one accumulator; the
// default) or 128 (two accumulators so the next unit's MMAs overlap this unit's drain; an
// experiment, see hinm_spmm_bf16).
constexpr int BK = 64;                         // logical K per A / metadata stage (2 MMAs)
constexpr int MAX_ASTAGES = 12;                // compressed-A / metadata ring (own barriers)
// Gathered-X ring: KS K-rows (x 256 tokens) per stage.  The cp.async gather pays a fixed
// per-stage cost in every producer warp (barrier wait + arrive), so 128-row stages
// (16 warps x 8 rows) stream markedly faster than 64-row ones (scripts/l2_ring.cu on B200:
// 20.4 vs 16.6 TB/s).
#ifndef HINM_PAIR_STAGES
#define HINM_PAIR_STAGES 4
#endif
__host__ __device__ constexpr int b_stages(int KS, int BNT, bool pair = false) {
  return pair ? (KS == 128 ? HINM_PAIR_STAGES : 2 * HINM_PAIR_STAGES) : (KS == 128 ? 3 : 5) * (256 / BNT);
}
__host__ __device__ constexpr int b_stage_bytes(int KS, int BNT) { return KS * BNT * 2; }
constexpr int MAX_XSTAGES = 10;
constexpr int E_STAGE = 128 * 16;              // 128 lanes x 16 B metadata image per stage slot
constexpr int TMEM_COLS = 512;
constexpr int E_COL = 256;                     // metadata ring after the accumulator(s)
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
  int rows;           // output rows (pseudo rows >= rows of a union-group pack are padding)
  int tdiv;           // unit -> (tile, token block) divisor: T, or T / 2 groups on the CTA-pair path
  int y_align32;      // Y rows 32-byte aligned: 256-bit stores
  uint32_t xpitch;    // bytes between consecutive K-rows (channels) of X
  int64_t xblk;       // bytes between consecutive BNT-token blocks of X
};

struct SmemLayout {
  uint32_t a, e, bar, tmem, total, ast;
};

// The A / metadata ring has its own barriers: its bulk copies see a much longer latency than the
// cp.async gather under load, and with a shared barrier they held every X stage hostage
// (scripts/l2_ring.cu).  One A stage covers one X stage (KS logical K: V*KS bytes of compressed
// values + one metadata slot); depth = whatever fits next to the X ring.
__host__ __device__ inline SmemLayout smem_layout(int V, int KS, bool m64, int BNT, bool pair = false) {
  SmemLayout L;
  const uint32_t slack = m64 || pair ? 0 : 4096;   // M=128 descriptor over-read past V rows
  const uint32_t budget = 227 * 1024 - 1024 - 512 - 128 - slack;
  const uint32_t per = V * KS + E_STAGE;
  const uint32_t xring = b_stages(KS, BNT, pair) * b_stage_bytes(KS, BNT);
  const uint32_t fit = (budget - xring) / per;
  L.ast = fit < (uint32_t)MAX_ASTAGES ? fit : MAX_ASTAGES;
  L.a = xring;
  L.e = L.a + L.ast * V * KS + slack;
  L.bar = L.e + L.ast * E_STAGE;
  L.tmem = L.bar + (3 * MAX_XSTAGES + 2 * MAX_ASTAGES + 4) * 8;
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

// L2 eviction-priority policies.  The compressed A / metadata image of every tile is re-read once
// per token block and must survive the streaming Y stores: A loads are evict_last, Y stores
// evict_first (run-to-run variance of the 4096x11008 layer came from A being evicted).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_hint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void st_global_v4_hint(void* ptr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.b32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// 32-byte store (one full L2 sector per thread; half the LSU requests of two 16-byte stores)
__device__ __forceinline__ void st_global_v8_hint(void* ptr, uint4 a, uint4 b, uint64_t pol) {
  asm volatile(
      "st.global.L1::no_allocate.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;" ::"l"(ptr),
      "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "l"(pol)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---- CTA pair (cluster of 2) helpers
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Relaxed: a release arrive compiles to MEMBAR.GPU (+ the waiter's acquire.cluster to CCTL.IVALL),
// ~1-2 k cycles on the per-stage critical path (ncu source view, profiles/r02_pair.txt).  What the
// leader needs is already established before the arrive: the peer's cp.async / bulk writes have
// completed (its local full barrier), its TMEM loads have completed (tcgen05.wait::ld).
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Per-stage event trace of CTA pair 0 (experiments build with -DHINM_TRACE; scripts/pair_trace.py):
// clock64 of each role's barrier completions, per running stage index; slot 10 = the two CTAs'
// clocks right after the start-up cluster barrier (offset calibration).
#ifdef HINM_TRACE
__device__ unsigned long long g_trace[11][1024];
__device__ unsigned long long g_utrace[160][72];  // per CTA: globaltimer at start, then per unit (MMA warp)
#define TRACE(ev, i)                                                                     \
  do {                                                                                   \
    if (blockIdx.x < 2 && (i) < 1024) g_trace[ev][i] = (unsigned long long)clock64();    \
  } while (0)
#else
#define TRACE(ev, i) \
  do {               \
  } while (0)
#endif

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
// CTA pair: the leader's commit arrives on the barrier at the same offset in both CTAs
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
template <bool PAIR>
__device__ __forceinline__ void tc_commit_x(uint32_t bar) {
  if (PAIR) tc_commit_pair(bar); else tc_commit(bar);
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

template <bool PAIR = false>
__device__ __forceinline__ void mma_sp(uint32_t tmem_d, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t tmem_e, uint32_t accumulate) {
  if (PAIR)  // CTA pair, M = 256: each CTA's 128 rows of A x the pair's B (N split over the CTAs)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t"
        "}\n" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(tmem_e)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%5], %3, p;\n\t"
        "}\n" ::"r"(tmem_d),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(tmem_e)
        : "memory");
}

template <bool PAIR = false>
__device__ __forceinline__ void tmem_cp_128x128b(uint32_t taddr, uint64_t sdesc) {
  if (PAIR)  // both CTAs: own shared memory -> own TMEM (scripts/probe_2sm.cu)
    asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
  else
    asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// 16 lanes x (32 + 32) columns: thread l < 16 gets lane l, columns c..c+31; thread l >= 16 gets
// lane l-16, columns c+128..c+159.
template <bool WAIT = true, int SPLIT = 128>
__device__ __forceinline__ void tmem_ld_16x32bx2_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {"
      "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], %33;"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr), "n"(SPLIT));
  if (WAIT) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 columns: thread l gets lane l, columns c..c+31.
template <bool WAIT = true>
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {"
      "%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  if (WAIT) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo_f32, uint32_t hi_f32) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo_f32), __uint_as_float(hi_f32));
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------------------------ the kernel
// Warp layout: warps 0-3 epilogue (TMEM lane quadrant = warp), warp 4 MMA issuer + TMEM owner,
// warp 5 A/metadata producer (bulk copies), warps 6.. gather producers.  The gather rate scales
// with the number of warps issuing cp.async, not with the bytes in flight (scripts/l2_cap.cu on
// B200: 8 warps/SM 15.6 TB/s, 12 -> 19.2, 16 -> 21.0 TB/s at any depth), so the default runs
// 16 gather warps.
constexpr int EPI_WARPS = 8;  // 2 per TMEM lane quadrant (column halves)
static_assert(EPI_WARPS == 8, "epilogue warps: quadrant = warp & 3, column half = warp >> 2");
constexpr int MMA_WARP = 8;
constexpr int AE_WARP = 9;
// First gather warp.  With 8 gather warps the kernel runs 18 warps on the launch register budget.
// With 16 (experiment HINM_GW=16) the 832+ threads would cap every role at 72 registers (the
// epilogue and gather loops spilled, which is what made 16 warps look slower), so the gather
// warps start on a warpgroup boundary (warp 12; warps 10-11 idle) and the warpgroups rebalance
// registers with setmaxnreg: gather 16 x 56, epilogue 8 x 104.  Spill-free, it runs exactly as
// fast as 8 warps (LLaMA up 0.741 vs 0.740 ms): under a running MMA the gather is capped by the
// SM's L2->SMEM fill rate, not by issuing warps (scripts/mma_gather_contention.cu).
__host__ __device__ constexpr int gather_warp0(int GW) { return GW == 8 ? 10 : 12; }
// CTA pair, 8 gather warps: the gather warps avoid the MMA warp's SM sub-partition (warp % 4 == 0).
// On the leader the issue of tcgen05.mma.cta_group::2 / commit held back the gather warps that share
// its sub-partition and, through the barrier, the whole stage: the leader's stage fill took ~700
// cycles longer than the peer's, also with the gather itself disabled (scripts/pair_trace.py).
// Warps 12 and 16 stay idle.
#ifdef HINM_SPREAD_ALL
__host__ __device__ constexpr bool gather_spread(int GW, bool) { return GW == 8; }
#else
__host__ __device__ constexpr bool gather_spread(int GW, bool pair) { return pair && GW == 8; }
#endif
__host__ __device__ constexpr int kernel_warps(int GW, bool pair) {
  return gather_spread(GW, pair) ? 20 : gather_warp0(GW) + GW;
}
constexpr int GATHER_REGS = 56, EPI_REGS = 104;

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

// CTA pair: unit u = (group u % tdiv, token block u / tdiv); CTA r works on pseudo tile 2g + r.
template <bool PAIR = false>
__device__ __forceinline__ UnitParams unit_params(const Params& p, int u, int crank = 0) {
  UnitParams q;
  if (u >= p.units) {
    q.t = q.nb = q.k0 = q.kp = q.e0 = 0;
    return q;
  }
  q.t = PAIR ? 2 * (u % p.tdiv) + crank : u % p.T;
  q.nb = u / p.tdiv;
  q.k0 = __ldg(p.tile_kofs + q.t);
  q.kp = __ldg(p.tile_kofs + q.t + 1) - q.k0;
  q.e0 = __ldg(p.tile_eofs + q.t);
  return q;
}

// DBG (experiments only): 1 = skip the MMAs (measure the gather pipeline alone),
// 2 = skip the gather (measure the MMA pipeline alone), 3 = no epilogue, 4 = no A / metadata
// loads, 5 = gather only with every 4th row left unfetched (ring slots vs bytes), 6 = the full
// kernel with every 4th row unfetched (a tile-pair image's zero-filled padding), 7 = the full kernel
// loading the A image on even token blocks only (A shared by two token blocks).  Results are
// garbage when DBG != 0.
// M64: V <= 64 on the M=64 instruction (half the A-operand shared-memory reads of M=128).  Its
// accumulator row 16q+l sits in TMEM lane 32q+l and its metadata where M=128 row 32q+l would
// (lanes 32q+0..15) -- measured with scripts/probe_sparse_meta.cu, which also shows that an
// M=64 accumulator at lane offset 16 faults (misaligned address), so one accumulator is used.
// PAIR (union-group pseudo packs, hinm_group_build): a cluster of two CTAs computes one 256-row
// group with tcgen05.mma.sp.cta_group::2 (M = 256, N = 256).  CTA r holds pseudo tile 2g + r (128
// rows of A, V = 128 image) and gathers tokens [256 nb + 128 r, +128) of the shared K-rows
// (BNT = 128 per CTA); its TMEM accumulator is its 128 rows x all 256 tokens.  The leader (rank
// 0) issues the MMAs once both CTAs' stages have landed: the peer's MMA warp relays each stage
// (local full + A barriers) to the leader's pfull barrier; the leader's commits multicast to the
// empty / accumulator barriers of both CTAs; the peer's epilogue releases the accumulator to the
// leader's acc_empty barrier.
template <int KS, int GW, int DBG = 0, bool M64 = false, int BNT = 256, bool PAIR = false>
__global__ void __launch_bounds__(32 * kernel_warps(GW, PAIR), 1)
    k_hinm_spmm(const uint16_t* __restrict__ X, int64_t ldx, Params p) {
  constexpr int GATHER_WARP0 = gather_warp0(GW);
  constexpr bool REBALANCE = GATHER_WARP0 % 4 == 0 && GW % 4 == 0;
  constexpr int NT = 32 * kernel_warps(GW, PAIR);
  constexpr bool SPREAD = gather_spread(GW, PAIR);
  constexpr int STAGES = b_stages(KS, BNT, PAIR), B_STAGE = b_stage_bytes(KS, BNT);
  constexpr int NCHUNK = BNT / 64;            // 64-token SWIZZLE_128B chunks of a stage
  constexpr int NACC = BNT == 128 && !PAIR ? 2 : 1;  // accumulators (TMEM columns 0 and 128)
  constexpr int NTOK = PAIR ? 256 : BNT;      // tokens per unit (accumulator columns)
  static_assert(STAGES <= MAX_XSTAGES, "X ring");
  static_assert(!PAIR || (BNT == 128 && !M64), "CTA pair: 128 tokens per CTA, M = 256");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const SmemLayout L = smem_layout(p.V, KS, M64, BNT, PAIR);
  const int V = p.V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const int ublk = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;    // first unit of this CTA (pair)
  const int ugrid = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;     // unit stride
  const uint32_t sB = base, sA = base + L.a, sE = base + L.e;
  const uint32_t bar_full = base + L.bar, bar_empty = bar_full + STAGES * 8;
  const uint32_t bar_afull = bar_empty + STAGES * 8, bar_aempty = bar_afull + MAX_ASTAGES * 8;
  const uint32_t bar_acc_full = bar_aempty + MAX_ASTAGES * 8;   // [NACC]
  const uint32_t bar_acc_empty = bar_acc_full + 16;             // [NACC]
  const uint32_t bar_pfull = bar_acc_empty + 16;                // [STAGES] (PAIR, leader)
  const int AST = (int)L.ast;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + L.tmem);
  // TMEM lane quadrants that hold real rows; two epilogue warps (column halves) per quadrant
  const int n_quads = M64 ? V / 16 : (V >= 128 ? 4 : V / 32);
  const int n_epi_warps = 2 * n_quads;

  // constant metadata for lanes the producer never writes (rows >= V, M=64 gap lanes)
  if (M64) {
    for (int i = threadIdx.x; i < AST * E_STAGE / 4; i += NT)
      reinterpret_cast<uint32_t*>(gbase + L.e)[i] = META_PAD;
  } else {
    for (int i = threadIdx.x; i < AST * (128 - V) * 4; i += NT) {
      const int s = i / ((128 - V) * 4), w = i % ((128 - V) * 4);
      reinterpret_cast<uint32_t*>(gbase + L.e + s * E_STAGE + V * 16)[w] = META_PAD;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 32 * GW);       // one cp.async noinc arrive per gather thread
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int s = 0; s < AST; ++s) {
      mbar_init(bar_afull + 8 * s, 1);
      mbar_init(bar_aempty + 8 * s, 1);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(bar_acc_full + 8 * a, 1);
      mbar_init(bar_acc_empty + 8 * a, n_epi_warps * (PAIR ? 2 : 1));  // PAIR: both CTAs' epilogues
    }
    if (PAIR)
      for (int s = 0; s < STAGES; ++s) mbar_init(bar_pfull + 8 * s, 1);  // one relay per peer stage
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == MMA_WARP) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_holder)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_holder)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // barrier inits visible to the peer before any remote arrive
  if (threadIdx.x == 0) TRACE(10, crank);
#ifdef HINM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_utrace[blockIdx.x][0] = globaltimer();
  if (threadIdx.x == 0 && blockIdx.x < 160) g_trace[8][blockIdx.x] = clock64();
#endif
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int T = p.T;
  // Programmatic dependent launch: everything above (barrier init, TMEM allocation, metadata pad)
  // touches only this CTA's shared memory / TMEM, so it overlaps the previous kernel's tail; no
  // global memory is read or written before the previous grid has completed.  The next kernel
  // may start its own prologue as soon as this grid's CTAs start exiting.
  // Only the roles that touch activations wait for the previous grid (gather: X reads, epilogue:
  // Y writes); the weight streams (A / metadata, gather indices, unit parameters) start during its
  // tail -- the previous kernel never writes them (hinm_stream_fence, include/hinm_b200.h).  BERT
  // and cfg1 shapes under CUDA graphs: 5-12 % per launch (profiles/r02_pair.txt).
  const bool waits = warp < EPI_WARPS || (warp >= GATHER_WARP0 && !(SPREAD && (warp & 3) == 0));
  if (!waits) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == AE_WARP) {
    // ============================================================ A / metadata producer
    // warp-uniform loop; one elected lane issues the bulk copies (see the MMA issuer note)
    int aslot = 0;
    uint32_t aphase = 0;
    UnitParams nxt = unit_params<PAIR>(p, ublk, crank);
    int a_count = 0;
    const uint32_t a_slot = V * KS;
    const uint64_t pol_a = l2_policy_evict_last();
    for (int u = ublk; u < p.units; u += ugrid) {
      const UnitParams cur = nxt;
      nxt = unit_params<PAIR>(p, u + ugrid, crank);
      const int nst = cur.kp / BK;                         // 64-K steps of the unit
      const uint16_t* asrc = p.a_vals + (int64_t)cur.k0 * V / 2;
      const uint32_t* esrc0 = p.a_meta + (int64_t)cur.e0 * V * 4;
      for (int s = 0; s < nst; s += KS / BK) {             // one A stage per X stage
        mbar_wait(bar_aempty + 8 * aslot, aphase ^ 1);
        if (DBG == 8) mbar_wait(bar_afull + 8 * aslot, aphase ^ 1);  // experiment: previous copy landed
        if (lane == 0) TRACE(7 + crank, a_count);
        ++a_count;
        const uint32_t fb = bar_afull + 8 * aslot;
        if (DBG == 4 || (DBG == 7 && (cur.nb & 1))) {  // experiments: no A / metadata loads
          // (DBG 7: on every other token block, i.e. the A image read once per 512 tokens)
          if (elect_one()) mbar_arrive(fb);
        } else if (elect_one()) {
          // (experiment 9: ~58 % of the A bytes -- what a compact A image would move; garbage)
          const uint32_t a_bytes = DBG == 9 ? (V * 64 * min(KS / BK, nst - s) * 9 / 16) & ~15u
                                            : V * 64 * min(KS / BK, nst - s);
          const uint32_t e_bytes = (s & 1) || DBG == 10 ? 0 : V * 16;   // metadata per 128-K block (10: skipped)
          mbar_expect_tx(fb, a_bytes + e_bytes);
          if (DBG == 11) {  // experiment: the A stage as one copy per 32-K MMA step
            for (uint32_t o = 0; o < a_bytes; o += 32 * V)
              bulk_g2s_hint(sA + aslot * a_slot + o, reinterpret_cast<const char*>(asrc + (int64_t)s * BK * V / 2) + o,
                            32 * V, fb, pol_a);
          } else {
            bulk_g2s_hint(sA + aslot * a_slot, asrc + (int64_t)s * BK * V / 2, a_bytes, fb, pol_a);
          }
          if (e_bytes) {
            const uint32_t* esrc = esrc0 + (int64_t)(s / 2) * V * 4;
            if (M64) {  // 16-lane groups of the stored (M=128 order) image -> lanes 32q + 0..15
              for (int q = 0; q < V / 16; ++q)
                bulk_g2s_hint(sE + aslot * E_STAGE + q * 512, esrc + q * 64, 256, fb, pol_a);
            } else {
              bulk_g2s_hint(sE + aslot * E_STAGE, esrc, e_bytes, fb, pol_a);
            }
          }
        }
        __syncwarp();
        if (++aslot == AST) { aslot = 0; aphase ^= 1; }
      }
    }
    if (PAIR)  // producer tail: the leader's last commits have landed before this CTA may exit
      for (int i = 0; i < AST; ++i) {
        mbar_wait(bar_aempty + 8 * aslot, aphase ^ 1);
        if (++aslot == AST) { aslot = 0; aphase ^= 1; }
      }
  } else if (warp >= GATHER_WARP0 && !(SPREAD && (warp & 3) == 0)) {
    // ============================================================ gather producers
    if (REBALANCE) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(GATHER_REGS));
    // Flattened stream over (unit, X stage) with the gather indices of stage i+PF loaded while
    // stage i is issued (the dependent index load never sits on the critical path).  The
    // issue loop is kept to ~4 instructions per 512-byte row: warp gw owns the K-rows
    // r = gw + GW*i of every stage, lane = 16-byte chunk of the row.  The last stage of a unit
    // may be partial (kp is a multiple of 64, KS may be 128).
    const int gw = SPREAD ? warp - 10 - (warp > 12) - (warp > 16) : warp - GATHER_WARP0;
    constexpr int PF = 8;
    constexpr int RPW = KS / GW;  // K-rows per warp per stage
    static_assert(KS % GW == 0 && GW >= 8 && RPW <= 32, "gather producers: GW | KS, GW >= 8");
    const int TD = p.tdiv;  // tiles (groups on the CTA-pair path) per token block
    const int dt = ugrid % TD, dnb = ugrid / TD;
    // prefetch cursor: unit (pt, pnb) with running index pu, stage ps, kp of the unit
    int pu = ublk, pt = ublk % TD, pnb = ublk / TD, ps = 0, pk0 = 0, pkp = 0;
    auto next_unit = [&]() {  // advance to the next unit with work
      while (pu < p.units) {
        const int tt = PAIR ? 2 * pt + (int)crank : pt;
        pk0 = __ldg(p.tile_kofs + tt);
        pkp = __ldg(p.tile_kofs + tt + 1) - pk0;
        if (pkp > 0) break;
        pu += ugrid;
        pt += dt;
        pnb += dnb;
        if (pt >= TD) { pt -= TD; ++pnb; }
      }
      ps = 0;
    };
    next_unit();
    const uint32_t ldx2 = p.xpitch;  // row pitch in bytes (host: < 2^32)
    uint32_t r_row[PF];
    int r_col[PF], r_n[PF];
    bool r_ok[PF];
    auto prefetch = [&](int slot) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        if (j != slot) continue;
        r_ok[j] = pu < p.units;
        if (!r_ok[j]) return;
        r_col[j] = PAIR ? pnb * 256 + (int)crank * 128 : pnb * BNT;
        const int n = min(KS, pkp - ps * KS);
        r_n[j] = n;
        const int* gi = p.gidx + pk0 + ps * KS;
        // raw row index: it is consumed PF stages later, so the load never stalls the warp here
        r_row[j] = lane < RPW && gw + lane * GW < n ? (uint32_t)__ldg(gi + gw + lane * GW) : 0u;
        if (++ps * KS >= pkp) {
          pu += ugrid;
          pt += dt;
          pnb += dnb;
          if (pt >= TD) { pt -= TD; ++pnb; }
          next_unit();
        }
      }
    };
#pragma unroll
    for (int j = 0; j < PF; ++j) prefetch(j);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // X is the previous kernel's output
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // A row segment is BNT tokens = LPR lanes x 16 B; one warp instruction covers RPI rows.
    // Per-warp constant part of the SWIZZLE_128B destination (row r = gw + GW i: r & 7 = gw & 7)
    constexpr int LPR = BNT / 8, RPI = 32 / LPR;
    const int lpos = lane % LPR, rsub = lane / LPR;
    const uint32_t dst_lane = (lpos >> 3) * (B_STAGE / NCHUNK) + (gw + rsub * GW) * 128 +
                              (((lpos & 7) ^ (gw & 7)) << 4);
    const char* xbase = reinterpret_cast<const char*>(X);
    int stage = 0, g_count = 0;
    uint32_t phase = 0;
    bool done = false;
    while (!done) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        if (!r_ok[j]) { done = true; break; }
        // per row: SHFL + IMAD.WIDE + LDGSTS (the issue slots of the gather warps are the
        // scarce resource, ncu source view); rows < 64 always exist, the rest only in full stages
        const int tok = r_col[j] + lpos * 8;
        const uint32_t src_bytes = tok < p.B ? 16u : 0u;
        const char* xs = xbase + (src_bytes ? (PAIR ? (int64_t)r_col[j] * 2 : (int64_t)(r_col[j] / BNT) * p.xblk) +
                                                  lpos * 16
                                            : 0);
        const uint32_t my_row = r_row[j];
        const bool full = r_n[j] == KS;
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        if (gw == 0 && lane == 0) TRACE(5 + crank, g_count);
        ++g_count;
        const uint32_t dst0 = sB + stage * B_STAGE + dst_lane;
#pragma unroll
        for (int k = 0; k < RPW / RPI; ++k) {
          const int i = k * RPI + rsub;  // this lane's row (of the warp's RPW)
          const uint32_t row = __shfl_sync(0xffffffffu, my_row, i);
          if (DBG != 2 && (i * GW < 64 || full) && !((DBG == 5 || DBG == 6) && (i & 3) == 3))
            cp_async_16(dst0 + k * RPI * GW * 128, xs + (uint64_t)row * ldx2, src_bytes);  // IMAD.WIDE.U32
        }
        cp_async_arrive_noinc(bar_full + 8 * stage);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        prefetch(j);
      }
    }
    if (PAIR)  // producer tail (see the A producer)
      for (int i = 0; i < STAGES; ++i) {
        mbar_wait(bar_empty + 8 * stage, phase ^ 1);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
  } else if (PAIR && warp == MMA_WARP && crank != 0) {
    // ============================================================ peer relay (CTA pair, rank 1)
    // The peer's X stage and A / metadata stage have landed in ITS shared memory: tell the leader,
    // whose MMAs read them.  Same unit / stage sequence as the leader's issue loop.
    const uint32_t rem_pfull = mapa_rank(bar_pfull, 0);
    int stage = 0, aslot = 0, r_count = 0;
    uint32_t phase = 0, aphase = 0;
    UnitParams nxt = unit_params<PAIR>(p, ublk, crank);
    for (int u = ublk; u < p.units; u += ugrid) {
      const int kp = nxt.kp;
      nxt = unit_params<PAIR>(p, u + ugrid, crank);
      if (kp == 0) continue;
      for (int s0 = 0; s0 < kp / BK; s0 += KS / BK) {
        mbar_wait(bar_full + 8 * stage, phase);
        if (lane == 0) TRACE(3, r_count);
        if (DBG != 8) mbar_wait(bar_afull + 8 * aslot, aphase);
        if (lane == 0) TRACE(4, r_count);
        ++r_count;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (elect_one()) mbar_arrive_remote(rem_pfull + 8 * stage);
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (++aslot == AST) { aslot = 0; aphase ^= 1; }
      }
    }
  } else if (warp == MMA_WARP) {
    // ============================================================ MMA issuer
    // The whole warp runs the loop (warp-uniform control flow keeps every descriptor in uniform
    // registers); one elected lane issues the tcgen05 instructions.  A single-lane loop forced
    // R2UR conversions of every operand per MMA and measured 2.6x slower MMA issue
    // (scripts/mma_bench.cu vs mma_bench_v1.cu).
    const uint32_t idesc = make_idesc(PAIR ? 256 : M64 ? 64 : 128, NTOK);
    // descriptors at stage 0; the start-address field (16 B units, bits 0-13) is advanced by
    // adding byte offsets >> 4
    const uint64_t a_desc0 = smem_desc(sA, 128, 256, 0);
    const uint64_t b_desc0 = smem_desc(sB, B_STAGE / NCHUNK, 1024, 2);
    const uint64_t e_desc0 = smem_desc(sE, 0, 128, 0);
    const uint32_t a_step = (uint32_t)(V * KS) >> 4, a_half = (uint32_t)(32 * V) >> 4;
    int stage = 0, aslot = 0, m_count = 0;
    uint32_t phase = 0, aphase = 0, eslot = 0, acc_uses = 0;
    UnitParams nxt = unit_params<PAIR>(p, ublk, crank);
    for (int u = ublk; u < p.units; u += ugrid) {
      const int kp = nxt.kp;
      nxt = unit_params<PAIR>(p, u + ugrid, crank);
      if (kp == 0) continue;
      const uint32_t acc = NACC == 2 ? (acc_uses & 1) : 0;
      mbar_wait(bar_acc_empty + 8 * acc, phase_acc_empty_parity(acc_uses / NACC));
      if (lane == 0) TRACE(9, acc_uses);
      ++acc_uses;
      tc_fence_after();
      const uint32_t dtm = tmem + acc * BNT;
      const int nst = kp / BK;
      // one iteration per X stage (SUB = 1 or 2 A stages): all waits first, then one elected
      // block issues the metadata copy, 2 * SUB MMAs and the commits (the issue loop, not the
      // tensor pipe, was the MMA warp's limiter: ncu source view)
      constexpr int SUB = KS / BK;
      for (int s0 = 0; s0 < nst; s0 += SUB) {
        const bool two = SUB == 2 && s0 + 1 < nst;
        mbar_wait(bar_full + 8 * stage, phase);
        if (lane == 0) TRACE(0, m_count);
        if (DBG != 8) mbar_wait(bar_afull + 8 * aslot, aphase);  // experiment 8: A loads off the critical path
        if (lane == 0) TRACE(1, m_count);
        if (PAIR) mbar_wait(bar_pfull + 8 * stage, phase);  // the peer's stage too (relayed)
        if (lane == 0) TRACE(2, m_count);
        ++m_count;
        tc_fence_after();
        if (elect_one()) {
          if ((s0 & 1) == 0) {  // metadata of the 128-K block starting at this step
            eslot = (eslot + 1) & (E_SLOTS - 1);
            tmem_cp_128x128b<PAIR>(tmem + E_COL + eslot * 4, e_desc0 + (uint64_t)((aslot * E_STAGE) >> 4));
          }
          const uint32_t ecol = tmem + E_COL + eslot * 4 + (s0 & 1) * 2;
          const uint64_t ad = a_desc0 + (uint64_t)(aslot * a_step);
          const uint64_t bd = b_desc0 + (uint64_t)((stage * B_STAGE) >> 4);
          if (DBG != 1 && DBG != 4 && DBG != 5) {
            mma_sp<PAIR>(dtm, ad, bd, idesc, ecol, s0 ? 1u : 0u);                      // id2 = 0
            mma_sp<PAIR>(dtm, ad + a_half, bd + (4096 >> 4), idesc | 1u, ecol, 1u);   // id2 = 1
            if (two) {
              mma_sp<PAIR>(dtm, ad + 2 * a_half, bd + (8192 >> 4), idesc, ecol + 2, 1u);
              mma_sp<PAIR>(dtm, ad + 3 * a_half, bd + (12288 >> 4), idesc | 1u, ecol + 2, 1u);
            }
          }
          tc_commit_x<PAIR>(bar_aempty + 8 * aslot);
          tc_commit_x<PAIR>(bar_empty + 8 * stage);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
        if (++aslot == AST) { aslot = 0; aphase ^= 1; }
      }
      if (elect_one()) tc_commit_x<PAIR>(bar_acc_full + 8 * acc);
      __syncwarp();
#ifdef HINM_TRACE
      if (lane == 0 && blockIdx.x < 160 && acc_uses < 71) g_utrace[blockIdx.x][acc_uses] = globaltimer();
      if (lane == 0 && blockIdx.x < 160 && acc_uses < 71) g_trace[9][blockIdx.x * 4 + (acc_uses & 3)] = clock64();
#endif
    }
  } else if (warp < EPI_WARPS) {
    // ============================================================ epilogue (warps 0-7)
    if (REBALANCE) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(EPI_REGS));
    // Warp w drains TMEM lane quadrant q = w & 3, column half h = w >> 2, with 32-column
    // tcgen05.ld's issued in pairs, and releases the accumulator to the MMA issuer right after
    // its last load, before that chunk's bf16 conversion and stores.  The drain is the
    // critical path between consecutive units (the next unit's MMAs wait for it): with small K
    // it dominated the kernel (scripts/spmm_shape.py, HINM_GATHER=dbg_noepi), hence 8 warps.
    //   M=64 : row 16q + (lane & 15); chunk c = columns 32c + (BNT/2)(lane >= 16) + [0, 32),
    //          c in [h NCH, (h+1) NCH)  (16x32bx2: lanes 0-15 of the quadrant hold the 16 rows)
    //   M=128: row 32q + lane;        chunk c = columns 32c + [0, 32), c in [h NCH, (h+1) NCH)
    // With two accumulators (BNT = 128) the drain of one overlaps the MMAs into the other.
    const int q = warp & 3, h = warp >> 2;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // Y may still be read by the previous kernel
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (q < n_quads) {
      uint32_t ucount = 0;
      const int r = M64 ? q * 16 + (lane & 15) : q * 32 + lane;
      const int c_own = M64 && lane >= 16 ? NTOK / 2 : 0;
      constexpr int NCH = M64 ? NTOK / 128 : NTOK / 64;  // 32-column chunks per warp
      const uint32_t t_row = tmem + ((uint32_t)(q * 32) << 16) + h * NCH * 32;
      // release of an accumulator: local, or (CTA pair, rank 1) to the leader's barrier
      const uint32_t acc_empty_dst = PAIR && crank ? mapa_rank(bar_acc_empty, 0) : bar_acc_empty;
      auto release = [&](uint32_t acc) {
        if (PAIR && crank) mbar_arrive_remote(acc_empty_dst + 8 * acc);
        else mbar_arrive(bar_acc_empty + 8 * acc);
      };
      // output row of this lane for a unit; -1: a padding row of a union-group pseudo pack
      auto out_row = [&](const UnitParams& u) -> int64_t {
        const int64_t prow = (int64_t)u.t * V + r;
        if (prow >= p.rows) return -1;
        return p.out_order == HINM_ORDER_ORIGINAL ? (int64_t)__ldg(p.sigma_o + prow) : prow;
      };
      // 32 accumulator columns (fp32 bits) -> bf16 -> 4 x 16-byte stores of one row segment
#if defined(HINM_Y_POLICY) && HINM_Y_POLICY == 1  // experiments: Y stores evict_normal / evict_last
      uint64_t pol_y;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_y));
#elif defined(HINM_Y_POLICY) && HINM_Y_POLICY == 2
      const uint64_t pol_y = l2_policy_evict_last();
#else
      const uint64_t pol_y = l2_policy_evict_first();
#endif
      auto store32 = [&](uint16_t* yrow, int col, const uint32_t (&v)[32]) {
        if (p.y_align32 && col + 32 <= p.B) {  // 2 x 32-byte stores: one full sector each
#pragma unroll
          for (int j = 0; j < 4; j += 2) {
            uint4 a, b;
            a.x = pack_bf16x2(v[j * 8 + 0], v[j * 8 + 1]);
            a.y = pack_bf16x2(v[j * 8 + 2], v[j * 8 + 3]);
            a.z = pack_bf16x2(v[j * 8 + 4], v[j * 8 + 5]);
            a.w = pack_bf16x2(v[j * 8 + 6], v[j * 8 + 7]);
            b.x = pack_bf16x2(v[j * 8 + 8], v[j * 8 + 9]);
            b.y = pack_bf16x2(v[j * 8 + 10], v[j * 8 + 11]);
            b.z = pack_bf16x2(v[j * 8 + 12], v[j * 8 + 13]);
            b.w = pack_bf16x2(v[j * 8 + 14], v[j * 8 + 15]);
            st_global_v8_hint(yrow + col + j * 8, a, b, pol_y);
          }
          return;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (col + j * 8 < p.B) {
            uint4 o;
            o.x = pack_bf16x2(v[j * 8 + 0], v[j * 8 + 1]);
            o.y = pack_bf16x2(v[j * 8 + 2], v[j * 8 + 3]);
            o.z = pack_bf16x2(v[j * 8 + 4], v[j * 8 + 5]);
            o.w = pack_bf16x2(v[j * 8 + 6], v[j * 8 + 7]);
            st_global_v4_hint(yrow + col + j * 8, o, pol_y);
          }
        }
      };
      UnitParams nxt = unit_params<PAIR>(p, ublk, crank);
      int64_t nxt_row = ublk < p.units ? out_row(nxt) : 0;
      for (int u = ublk; u < p.units; u += ugrid) {
        const UnitParams cur = nxt;
        const int64_t orow = nxt_row;
        nxt = unit_params<PAIR>(p, u + ugrid, crank);
        if (u + ugrid < p.units) nxt_row = out_row(nxt);
        const bool live = orow >= 0;
        // 14 (experiment): the same stores folded into a 64-row window of Y (L2-resident: the LSU / L2
        // traffic of the stores without their DRAM writes)
        uint16_t* yrow = p.Y + (live ? (DBG == 14 ? orow % 64 : orow) : 0) * p.ldy;
        const int col_base = cur.nb * NTOK + c_own + h * NCH * 32;
        if (cur.kp == 0) {  // empty tile: zero rows (spmm.py:89-90)
          for (int c = 0; c < NCH * 4; ++c)
            if (live && col_base + c * 8 < p.B)
              *reinterpret_cast<uint4*>(yrow + col_base + c * 8) = make_uint4(0, 0, 0, 0);
          continue;
        }
        const uint32_t acc = NACC == 2 ? (ucount & 1) : 0;
#ifdef HINM_EPI_SLEEP
        {  // experiment: idle epilogue warps back off instead of spinning on the accumulator barrier
          uint32_t ok = 0;
          while (true) {
            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(bar_acc_full + 8 * acc), "r"((ucount / NACC) & 1) : "memory");
            if (ok) break;
            __nanosleep(HINM_EPI_SLEEP);
          }
        }
#else
        mbar_wait(bar_acc_full + 8 * acc, (ucount / NACC) & 1);
#endif
        ++ucount;
        tc_fence_after();
        const uint32_t t_acc = t_row + acc * BNT;
        if (DBG == 3) {  // experiment: release at once, no drain / stores
          __syncwarp();
          if (lane == 0) release(acc);
          continue;
        }
        if (DBG == 13) {  // experiment: release at once, then the drain and the stores (stores off the critical path)
          __syncwarp();
          if (lane == 0) release(acc);
        }
        uint32_t v0[32], v1[32];
        if (NCH == 1) {  // one chunk per warp (M=64, BNT=128)
          tmem_ld_16x32bx2_x32<true, BNT / 2>(t_acc, v0);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release(acc);
          if (live) store32(yrow, col_base, v0);
          continue;
        }
        // chunks are loaded in pairs (two tcgen05.ld in flight, one wait); the accumulator is
        // released after the last pair's wait
#pragma unroll 1
        for (int c = 0; c < NCH; c += 2) {
          if (M64) {
            tmem_ld_16x32bx2_x32<false, NTOK / 2>(t_acc + c * 32, v0);
            tmem_ld_16x32bx2_x32<false, NTOK / 2>(t_acc + c * 32 + 32, v1);
          } else {
            tmem_ld_32x32b_x32<false>(t_acc + c * 32, v0);
            tmem_ld_32x32b_x32<false>(t_acc + c * 32 + 32, v1);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 2 == NCH && DBG != 13) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release(acc);
          }
          if (live && DBG != 12) {  // 12 (experiment): the drain without the stores
            store32(yrow, col_base + c * 32, v0);
            store32(yrow, col_base + c * 32 + 32, v1);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the peer's remote arrivals and TMEM reads are done
  if (warp == MMA_WARP) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace sm100
}  // namespace hinm

// ------------------------------------------------------------------------------ host side
namespace {

thread_local int g_last_launches = 0;
thread_local int g_last_image = 0;  // 0: per-tile image, 1: union-group image (CTA pair)

// Per-device SM count and per-(kernel, device) shared-memory opt-in, cached: the launch path is
// on the critical path of short SpMMs (host time per call, scripts/host_overhead.py).
constexpr int MAX_DEVICES = 64;
int g_sms[MAX_DEVICES] = {};

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

int sm_count(int dev) {
  if (dev < 0 || dev >= MAX_DEVICES) return 148;
  if (g_sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_sms[dev] = n > 0 ? n : 148;
  }
  return g_sms[dev];
}

cudaError_t ensure_smem(const void* fn, int /*dev*/, int bytes) { return hinm::smem_optin(fn, bytes); }

}  // namespace

extern "C" int hinm_last_launch_count(void) { return g_last_launches; }
extern "C" int hinm_last_image(void) { return g_last_image; }

#ifdef HINM_TRACE
// experiments: copy the pair-0 event trace (11 x 1024 clock64 values) to host memory
extern "C" int hinm_exp_trace(unsigned long long* host) {
  HINM_CUDA_TRY(cudaDeviceSynchronize());
  HINM_CUDA_TRY(cudaMemcpyFromSymbol(host, hinm::sm100::g_trace, sizeof(unsigned long long) * 11 * 1024));
  return HINM_OK;
}
extern "C" int hinm_exp_utrace(unsigned long long* host) {
  HINM_CUDA_TRY(cudaDeviceSynchronize());
  HINM_CUDA_TRY(cudaMemcpyFromSymbol(host, hinm::sm100::g_utrace, sizeof(unsigned long long) * 160 * 72));
  HINM_CUDA_TRY(cudaMemset(nullptr, 0, 0));
  return HINM_OK;
}
#endif

namespace {

// The union-group pseudo pack on the CTA-pair kernel (hinm_group_build; spmm_sm100.cu PAIR).
int spmm_pair(const hinm_pack_t* g, const uint16_t* X, int64_t ldx, int B, uint16_t* Y, int64_t ldy,
              int out_order, int y_align32, cudaStream_t st) {
  using namespace hinm::sm100;
  Params prm;
  prm.tile_kofs = g->tile_kofs;
  prm.tile_eofs = g->tile_eofs;
  prm.gidx = g->gidx;
  prm.a_vals = g->a_vals;
  prm.a_meta = g->a_meta;
  prm.sigma_o = g->sigma_o;
  prm.Y = Y;
  prm.ldy = ldy;
  prm.B = B;
  prm.T = g->T;
  prm.V = 128;
  prm.out_order = out_order;
  prm.rows = g->rows;
  prm.tdiv = g->T / 2;
  prm.y_align32 = y_align32;
  prm.units = ((B + 255) / 256) * prm.tdiv;
  prm.xpitch = (uint32_t)(ldx * 2);
  prm.xblk = 256 * 2;
  const int dev = current_device();
  const int pairs = std::min(prm.units, sm_count(dev) / 2);
  // HINM_PAIR_KS = 64 | 128 (K-rows per X stage), HINM_PAIR_GW = 8 | 16 (gather warps)
  static const int pks = [] { const char* e = getenv("HINM_PAIR_KS"); return e && !strcmp(e, "64") ? 64 : 128; }();
  static const int pgw = [] { const char* e = getenv("HINM_PAIR_GW"); return e && !strcmp(e, "16") ? 16 : 8; }();
  const int KS = pks, GW = pgw;
  auto kern = KS == 64 ? (GW == 16 ? k_hinm_spmm<64, 16, 0, false, 128, true> : k_hinm_spmm<64, 8, 0, false, 128, true>)
                       : (GW == 16 ? k_hinm_spmm<128, 16, 0, false, 128, true> : k_hinm_spmm<128, 8, 0, false, 128, true>);
#ifdef HINM_EXPERIMENTS
  // timing-only: HINM_PAIR_DBG = 1 (no MMAs) | 2 (no gather) | 3 (no epilogue); results are garbage
  if (const char* e = getenv("HINM_PAIR_DBG")) {
    if (e[0] == '1') kern = k_hinm_spmm<128, 8, 1, false, 128, true>;
    if (e[0] == '2') kern = k_hinm_spmm<128, 8, 2, false, 128, true>;
    if (e[0] == '3') kern = k_hinm_spmm<128, 8, 3, false, 128, true>;
    if (e[0] == '4') kern = k_hinm_spmm<128, 8, 4, false, 128, true>;
    if (e[0] == '8') kern = k_hinm_spmm<128, 8, 8, false, 128, true>;
    if (e[0] == '9') kern = k_hinm_spmm<128, 8, 9, false, 128, true>;
    if (!strcmp(e, "10")) kern = k_hinm_spmm<128, 8, 10, false, 128, true>;
    if (!strcmp(e, "11")) kern = k_hinm_spmm<128, 8, 11, false, 128, true>;
    if (!strcmp(e, "12")) kern = k_hinm_spmm<128, 8, 12, false, 128, true>;
    if (!strcmp(e, "13")) kern = k_hinm_spmm<128, 8, 13, false, 128, true>;
    if (!strcmp(e, "14")) kern = k_hinm_spmm<128, 8, 14, false, 128, true>;
  }
#endif
  const SmemLayout L = smem_layout(128, KS, false, 128, true);
  HINM_CUDA_TRY(ensure_smem((const void*)kern, dev, (int)L.total));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(32 * kernel_warps(GW, true));
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // short launches overlap their prologue with the previous kernel's tail (programmatic dependent
  // launch), as on the per-tile path
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = prm.units <= 8 * pairs ? 2 : 1;
  HINM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, X, ldx, prm));
  HINM_LAUNCH_CHECK();
  g_last_launches = 1;
  g_last_image = 1;
  return HINM_OK;
}

// Per-call choice between a pack's per-tile image and its union-group image.  Modelled time =
// ramp + waves x max(K-steps x cycles per 32-K step + unit overhead, unit floor), fitted on B200
// (profiles/r02_pair.txt: scripts/pair_sweep.py, bench.py --config cfg2 / cfg4 / cfg5):
//   per-tile (148 SMs):     270 cycles per step + 2300 per unit, ramp 3000
//   union-group (74 pairs): 226 cycles per 32-K_u step + 3300 per unit, >= 5000 per unit, ramp 8000
//                           (5000 for launches short enough for PDL);
//                           >= 12000 per unit for <= 128-slot groups over > 256k tokens (the
//                           pair's 128-row x 256-token stores per CTA at a > 0.5 MB row pitch: the
//                           ResNet im2col 256x64 layer at 802816 tokens runs 2x slower than per-tile)
// HINM_GROUPS = 0 | 1 forces.
bool choose_group(const hinm_pack_t* pk, int B, int sms) {
  const hinm_pack_t* g = pk->group;
  if (!g || !g->pair || !g->a_vals || !g->tile_kofs || g->T < 2 || pk->T < 1) return false;
  static const int force = [] {
    const char* e = getenv("HINM_GROUPS");
    if (!e) return -1;
    if (!strcmp(e, "0")) return 0;
    if (!strcmp(e, "1")) return 1;
    fprintf(stderr, "[hinm] invalid HINM_GROUPS=%s (0 | 1)\n", e);
    return -2;
  }();
  if (force == 0 || force == -2) return false;
  if (force == 1) return true;
  const double nb = (double)((B + 255) / 256);
  auto steps = [](double k) { return std::ceil(k / 64.0) * 2.0; };  // kp = round_up(k, 64) in 32-K steps
  const double st_t = steps((double)pk->total_keep / pk->T), st_g = steps((double)g->total_keep / g->T);
  const double waves_t = std::ceil(pk->T * nb / sms), waves_g = std::ceil(g->T / 2 * nb / (sms / 2));
  // constants fitted to minimise the time lost to wrong picks over 84 measured (shape, tokens)
  // cases (scripts/fit_image_model.py on profiles/r02_image_choice_data.jsonl: 38.9 -> 16.9 us)
  const double floor_g = st_g <= 4.0 && B > 262144 ? 11000.0 : 5000.0;
  const double cost_t = 2000.0 + waves_t * (st_t * 270.0 + 2400.0);
  // short pair launches overlap their prologue with the previous kernel (PDL): a smaller ramp
  const double ramp_g = g->T / 2 * nb <= 8.0 * (sms / 2) ? 5000.0 : 8000.0;
  const double cost_g = ramp_g + waves_g * std::max(st_g * 205.0 + 1900.0, floor_g);
  return cost_g < cost_t;
}

}  // namespace

extern "C" int hinm_spmm_bf16(const hinm_pack_t* pk, const uint16_t* X, int64_t ldx, int B,
                              uint16_t* Y, int64_t ldy, int out_order, void* stream) {
  using namespace hinm::sm100;
  g_last_launches = 0;
  g_last_image = 0;
  if (!pk || !X || !Y) return HINM_ERR_VALUE;
  if (pk->N != 2 || pk->M != 4) return HINM_ERR_UNSUPPORTED;
  if (pk->V != 32 && pk->V != 64 && pk->V != 128) return HINM_ERR_UNSUPPORTED;
  if (!pk->gidx || !pk->a_vals || !pk->a_meta || !pk->tile_kofs) return HINM_ERR_VALUE;
  if (B < 0 || (B % 8) || (ldx % 8) || (ldy % 8) || ldx < B || ldy < B) return HINM_ERR_VALUE;
  if (((uintptr_t)X & 15) || ((uintptr_t)Y & 15)) return HINM_ERR_VALUE;
  if (ldx * 2 >= (int64_t)1 << 32) return HINM_ERR_UNSUPPORTED;  // 32-bit row pitch
  if (B == 0 || pk->m == 0) return HINM_OK;
  if (pk->pair) {  // a union-group pseudo pack given directly: the CTA-pair kernel
    if (pk->V != 128 || pk->T % 2 || !pk->tile_eofs || pk->rows < 1 || pk->rows > pk->m) return HINM_ERR_VALUE;
    const int a32 = (ldy % 16) == 0 && ((uintptr_t)Y & 31) == 0;
    return spmm_pair(pk, X, ldx, B, Y, ldy, out_order, a32, (cudaStream_t)stream);
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
  prm.out_order = out_order;
  prm.rows = pk->m;
  prm.tdiv = pk->T;
  // Tuning knobs (environment; every value is validated, an unknown one is an error rather than a
  // silent default).  Defaults are the B200 measurements (scripts/spmm_grid.sh): 8 gather warps (16
  // are no faster: the fill rate under a running MMA is the cap); V <= 64 -> 128-row X stages;
  // V = 128 -> 64-row X stages (its 8 KB A stages need the deeper A ring that the smaller X ring
  // leaves room for).  Unit width BNT: 256 tokens.  BNT = 128 (two accumulators: the drain of one
  // unit overlaps the next unit's MMAs, twice the units) is slower whenever the 256-token units
  // fill the machine, small-K shapes included (3072x768 @ 4096 tokens 0.024 -> 0.028 ms, 256x64 @
  // 802816 0.10 -> 0.12 ms): 256-byte row segments gather less efficiently and the A image is
  // re-read twice as often.  It is used only when the units would otherwise leave SMs idle.
  //   HINM_BN = 128 | 256, HINM_KS = 64 | 128, HINM_GW = 8 | 16, HINM_PDL = 0 | 1, HINM_Y_V8 = 0 | 1,
  //   HINM_GATHER = m128 (the M=128 instruction for V <= 64).
  // Timing-only variants (results are garbage: see the DBG note above the kernel) exist only in the
  // experiments build (-DHINM_EXPERIMENTS, scripts/ only): HINM_GATHER = dbg_nomma | dbg_nogather |
  // dbg_noepi | dbg_gather_x_only | dbg_gather_sparse | dbg_pad_quarter | dbg_half_a, HINM_XBLK = 1.
  struct Knobs {
    int v8, ks, gw, bn, pdl, variant, xblk;
    bool ok;
  };
  static const Knobs kn = [] {
    Knobs k{1, 0, 0, 0, -1, 0, 0, true};
    auto num = [&k](const char* name, int* dst, std::initializer_list<int> allowed) {
      const char* e = getenv(name);
      if (!e) return;
      char* endp = nullptr;
      const long v = strtol(e, &endp, 10);
      bool good = endp && *endp == 0 && endp != e;
      if (good) {
        good = false;
        for (int a : allowed) good |= v == a;
      }
      if (!good) {
        fprintf(stderr, "[hinm] invalid %s=%s\n", name, e);
        k.ok = false;
        return;
      }
      *dst = (int)v;
    };
    num("HINM_Y_V8", &k.v8, {0, 1});
    num("HINM_KS", &k.ks, {64, 128});
    num("HINM_GW", &k.gw, {8, 16});
    num("HINM_BN", &k.bn, {128, 256});
    num("HINM_PDL", &k.pdl, {0, 1});
    if (const char* e = getenv("HINM_GATHER")) {
      static const char* names[] = {"m128", "dbg_nomma", "dbg_nogather", "dbg_noepi", "dbg_gather_x_only",
                                    "dbg_gather_sparse", "dbg_pad_quarter", "dbg_half_a"};
      int v = -1;
      for (int i = 0; i < 8; ++i)
        if (!strcmp(e, names[i])) v = i + 1;
#ifndef HINM_EXPERIMENTS
      if (v > 1) v = -1;  // timing-only variants are not part of the product library
#endif
      if (v < 0) {
        fprintf(stderr, "[hinm] invalid HINM_GATHER=%s\n", e);
        k.ok = false;
      } else {
        k.variant = v;
      }
    }
#ifdef HINM_EXPERIMENTS
    num("HINM_XBLK", &k.xblk, {0, 1});
#endif
    return k;
  }();
  if (!kn.ok) return HINM_ERR_VALUE;
  prm.y_align32 = kn.v8 && (ldy % 16) == 0 && ((uintptr_t)Y & 31) == 0;
  const int variant = kn.variant;
  const int dev = current_device();
  const int sms = sm_count(dev);
  const bool has_group = pk->group && pk->group->pair && pk->group->a_vals;
  if (variant == 0 && !kn.xblk && pk->image != 1 && has_group && (pk->image == 2 || choose_group(pk, B, sms)))
    return spmm_pair(pk->group, X, ldx, B, Y, ldy, out_order, prm.y_align32, (cudaStream_t)stream);
  // 128-token units only when 256-token units would leave more than half the SMs idle (e.g. the
  // down projection at 256 tokens per GPU under 8-way token sharding: 64 units -> 128 units,
  // 0.030 -> 0.024 ms); with more units the 256-token kernel wins
  const int64_t units256 = (int64_t)((B + 255) / 256) * pk->T;
  int bnt = units256 * 2 <= sms ? 128 : 256;
  if (kn.bn) bnt = kn.bn;
  if (variant >= 2 || kn.xblk) bnt = 256;
  prm.units = ((B + bnt - 1) / bnt) * pk->T;
  prm.xpitch = (uint32_t)(ldx * 2);
  prm.xblk = (int64_t)bnt * 2;
  if (kn.xblk) {  // experiment: X stored token-block-major, [B/256][n][256]
    prm.xpitch = 512;
    prm.xblk = (int64_t)pk->n * 512;
  }
  const int grid = std::min(prm.units, sms);
  cudaStream_t st = (cudaStream_t)stream;
  const bool m64 = pk->V <= 64 && variant != 1;
  // Short kernels are launched with programmatic stream serialization (PDL): back-to-back SpMMs
  // (layer chains, CUDA graphs) overlap this kernel's prologue with the previous kernel's tail,
  // ~1-1.7 us per launch on the BERT / cfg1 shapes (scripts/small_shapes.py).  Long kernels (more
  // than 8 units per SM) gain nothing measurable and keep plain launches (HINM_PDL = 0 | 1 forces).
  const bool pdl = kn.pdl == 1 || (kn.pdl == -1 && prm.units <= 8 * sms);
  auto launch = [&](auto kern, int ks, int gw, int bn) -> int {
    const SmemLayout L = smem_layout(pk->V, ks, m64, bn);
    HINM_CUDA_TRY(ensure_smem((const void*)kern, dev, (int)L.total));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32 * kernel_warps(gw, false));
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    HINM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, X, ldx, prm));
    return HINM_OK;
  };
  const int ks = kn.ks ? kn.ks : (pk->V <= 64 ? 128 : 64);
  const int gw = kn.gw ? kn.gw : 8;
  int rc;
#ifdef HINM_EXPERIMENTS
  if (variant == 2) {
    rc = gw == 16 ? launch(k_hinm_spmm<128, 16, 1, true>, 128, 16, 256) : launch(k_hinm_spmm<128, 8, 1, true>, 128, 8, 256);
  } else if (variant == 3) {
    rc = launch(k_hinm_spmm<128, 8, 2, true>, 128, 8, 256);
  } else if (variant == 4) {
    rc = launch(k_hinm_spmm<128, 8, 3, true>, 128, 8, 256);
  } else if (variant == 5) {
    rc = launch(k_hinm_spmm<128, 8, 4, true>, 128, 8, 256);
  } else if (variant == 6) {
    rc = launch(k_hinm_spmm<128, 8, 5, true>, 128, 8, 256);
  } else if (variant == 7) {
    rc = m64 ? launch(k_hinm_spmm<128, 8, 6, true>, 128, 8, 256) : launch(k_hinm_spmm<64, 8, 6, false>, 64, 8, 256);
  } else if (variant == 8) {
    rc = launch(k_hinm_spmm<128, 8, 7, true>, 128, 8, 256);
  } else
#endif
  if (bnt == 128) {
    rc = ks == 128 ? (m64 ? launch(k_hinm_spmm<128, 8, 0, true, 128>, 128, 8, 128)
                          : launch(k_hinm_spmm<128, 8, 0, false, 128>, 128, 8, 128))
                   : (m64 ? launch(k_hinm_spmm<64, 8, 0, true, 128>, 64, 8, 128)
                          : launch(k_hinm_spmm<64, 8, 0, false, 128>, 64, 8, 128));
  } else if (ks == 128) {
    rc = gw == 8 ? (m64 ? launch(k_hinm_spmm<128, 8, 0, true>, 128, 8, 256) : launch(k_hinm_spmm<128, 8, 0, false>, 128, 8, 256))
                 : (m64 ? launch(k_hinm_spmm<128, 16, 0, true>, 128, 16, 256) : launch(k_hinm_spmm<128, 16, 0, false>, 128, 16, 256));
  } else {
    rc = gw == 8 ? (m64 ? launch(k_hinm_spmm<64, 8, 0, true>, 64, 8, 256) : launch(k_hinm_spmm<64, 8, 0, false>, 64, 8, 256))
                 : (m64 ? launch(k_hinm_spmm<64, 16, 0, true>, 64, 16, 256) : launch(k_hinm_spmm<64, 16, 0, false>, 64, 16, 256));
  }
  if (rc) return rc;
  HINM_LAUNCH_CHECK();
  g_last_launches = 1;
  return HINM_OK;
}
