// Union-group operand image for the CTA-pair HiNM SpMM (2:4, V in {32, 64}).
//
// The reference computes every V-row tile against its own gathered K-rows (spmm.py:88-98): the
// bytes staged per flop are 1/V, and at V = 64 the tcgen05 SpMM is bound by that L2 -> SMEM fill
// (profiles/r02_spmm_ceiling.txt).  Here G = 256 / V consecutive tiles (256 rows in sigma_o order)
// share ONE gather list: the union of their kept columns, arranged into 4-slot chunks such that
// every row of the 256 has at most two nonzeros per chunk.  That is again a 2:4 matrix (256 rows x
// K_u), computed by a CTA pair (tcgen05.mma.sp.cta_group::2, M = 256: each CTA 128 rows and half of
// the tokens of B, B shared over the pair).  The product is unchanged: every kept value of the
// reference view is placed once, at the slot of its column, and every other A entry is zero.
//
// Pipeline (hinm_group_plan + hinm_group_build):
//   k_inv       inv[t][c] = position of column c in tile t's vector order (-1: pruned vector)
//   k_masks     per group and column: the 256-bit set of rows that keep a nonzero there
//               (one warp per 32-row slab, one ballot per 2:4 slot -- no atomics)
//   k_greedy    first-fit of the union columns (ascending) into open chunks: a column joins the
//               oldest open chunk in which no row already has two nonzeros (one CTA per group)
//   k_view      the pseudo reference view of the two 128-row halves (V = 128 tiles of K_u
//               vectors): nm_index / kept_values per (row, chunk), then hinm_pack_build writes the
//               tcgen05 operand image exactly as for a V = 128 pack
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace hinm {
namespace grp {

constexpr int GR = 256;       // rows per group (CTA pair x 128 TMEM lanes)
constexpr int MW = GR / 32;   // 32-bit mask words per column
constexpr int GT = 256;       // threads of the greedy CTA
constexpr int EMAX = 1024;    // open-list entries (live open chunks measured <= 786 at n = 11008)
static_assert(EMAX == 4 * 256, "the first-fit scan gives each of the 256 threads 4 contiguous entries");

struct Ws {
  size_t inv, mask, cols, nch, err, total;
};

inline Ws ws_layout(int T, int n, int U) {
  Ws L;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  L.inv = 0;
  L.mask = L.inv + al((size_t)T * n * 2);
  L.cols = L.mask + al((size_t)U * n * MW * 4);
  L.nch = L.cols + al((size_t)U * n * 4 * 4);
  L.err = L.nch + al((size_t)(U + 1) * 4);
  L.total = L.err + 256;
  return L;
}

__global__ void k_inv(const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ vec_idx, int n,
                      int16_t* __restrict__ inv) {
  const int t = blockIdx.y;
  const int b = tile_ptr[t], k = tile_ptr[t + 1] - b;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
    inv[(int64_t)t * n + vec_idx[b + i]] = (int16_t)i;
}

// mask[(u * n + c) * MW + w], bit l: row 32 w + l of group u keeps a nonzero at column c.
// One warp per (tile, 32-row slab) x stride of 2:4 groups; lane = row.  Every (u, c, w) word is
// written by exactly one warp (a column appears once in a tile's vector order).
__global__ void k_masks(const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ vec_idx,
                        const uint8_t* __restrict__ nm_pos, int n, int V, uint32_t* __restrict__ mask) {
  const int t = blockIdx.y;
  const int G = GR / V, slabs = V / 32;
  const int u = t / G, j = t % G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int slab = warp % slabs, gstep = (wpb / slabs) * gridDim.x;
  const int w = j * slabs + slab, r = slab * 32 + lane;
  const int b = tile_ptr[t], k = tile_ptr[t + 1] - b, Gt = k / 4;
  const uint8_t* rowp = nm_pos + (int64_t)V * (b / 4) * 2 + (int64_t)r * Gt * 2;
  uint32_t* mu = mask + (int64_t)u * n * MW + w;
  for (int g = blockIdx.x * (wpb / slabs) + warp / slabs; g < Gt; g += gstep) {
    const uint32_t p0 = rowp[2 * g], p1 = rowp[2 * g + 1];
    const int col = lane < 4 ? __ldg(vec_idx + b + 4 * g + lane) : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t bits = __ballot_sync(0xffffffffu, p0 == (uint32_t)q || p1 == (uint32_t)q);
      if (lane == q) mu[(int64_t)col * MW] = bits;
    }
  }
}

// First-fit chunking of one group's union columns (one CTA per group).  Open chunks form a list
// in creation order; a column c with row set m fits entry e iff twos[e] & m == 0 (rows with >= 2
// nonzeros in the chunk) and the chunk has a free slot; it joins the lowest fitting entry, else a
// new chunk is appended.  The list state lives in registers: thread tid owns entries
// 4 tid .. 4 tid + 3 (ones / twos masks of all 256 rows, fill count, chunk id), so a column costs
// one broadcast of its mask, 64 register ANDs per thread, a warp min and one barrier (the owner
// updates its entry).  Full chunks stay in the list until it reaches EMAX entries, then a stable
// compaction through shared memory drops them; if the open chunks alone fill the list the oldest
// is closed (deterministic).  Output: chunk_cols[u][4 * chunk + slot] (column, -1 = empty slot),
// nchunks[u].
__global__ void __launch_bounds__(GT, 1) k_greedy(const uint32_t* __restrict__ mask, int n, int cap_chunks,
                                                  int32_t* __restrict__ chunk_cols, int32_t* __restrict__ nchunks) {
  constexpr int PER = EMAX / GT;
  extern __shared__ __align__(16) uint32_t gsm[];
  uint32_t* st_ones = gsm;                                   // compaction staging [EMAX][MW]
  uint32_t* st_twos = st_ones + EMAX * MW;
  int32_t* st_cid = reinterpret_cast<int32_t*>(st_twos + EMAX * MW);
  int32_t* st_cnt = st_cid + EMAX;
  __shared__ uint32_t bm[GT][MW + 1];
  __shared__ int bcol[GT];
  __shared__ int s_wsum[GT / 32], s_wmin[2][GT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = blockIdx.x;
  const uint32_t* mu = mask + (int64_t)u * n * MW;
  int32_t* cc = chunk_cols + (int64_t)u * cap_chunks * 4;
  uint32_t on[PER][MW], tw[PER][MW];
  int cn[PER], id[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    cn[q] = 4;
    id[q] = 0;
#pragma unroll
    for (int w = 0; w < MW; ++w) on[q][w] = tw[q][w] = 0u;
  }
  int L = 0, nchunk = 0, it = 0;  // list length and chunk count: identical in every thread
  for (int c0 = 0; c0 < n; c0 += GT) {
    // ---- batch of GT columns: keep the ones some row of the group uses (the union), in order
    const int c = c0 + tid;
    uint32_t m[MW];
    bool nz = false;
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      m[w] = c < n ? mu[(int64_t)c * MW + w] : 0u;
      nz |= m[w] != 0u;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, nb = 0;
    for (int w = 0; w < GT / 32; ++w) {
      off += w < warp ? s_wsum[w] : 0;
      nb += s_wsum[w];
    }
    if (nz) {
      const int pos = off + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
      for (int w = 0; w < MW; ++w) bm[pos][w] = m[w];
      bcol[pos] = c;
    }
    __syncthreads();
    for (int i = 0; i < nb; ++i, ++it) {
      uint32_t mm[MW];
#pragma unroll
      for (int w = 0; w < MW; ++w) mm[w] = bm[i][w];
      int mine = INT_MAX;
#pragma unroll
      for (int q = PER - 1; q >= 0; --q) {  // the thread's lowest fitting entry
        uint32_t conf = 0u;
#pragma unroll
        for (int w = 0; w < MW; ++w) conf |= tw[q][w] & mm[w];
        if (tid * PER + q < L && cn[q] < 4 && conf == 0u) mine = tid * PER + q;
      }
      mine = __reduce_min_sync(0xffffffffu, mine);
      // double-buffered warp minima: the buffer written at column it + 2 is behind column it + 1's barrier
      if (lane == 0) s_wmin[it & 1][warp] = mine;
      __syncthreads();
      int bj = INT_MAX;
#pragma unroll
      for (int w = 0; w < GT / 32; ++w) bj = min(bj, s_wmin[it & 1][w]);
      const int tgt = bj != INT_MAX ? bj : L;  // the entry that takes the column
      if (tid == tgt / PER) {
        // the owner updates entry qs with selects over its four entries (a branch on qs would let
        // the compiler index the register arrays dynamically, i.e. move them to local memory)
        const int qs = tgt % PER;
        const bool grow = bj != INT_MAX;
        int idq = 0, cnq = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          idq = q == qs ? id[q] : idq;
          cnq = q == qs ? cn[q] : cnq;
        }
        if (grow) cc[(int64_t)idq * 4 + cnq] = bcol[i];
        else *reinterpret_cast<int4*>(cc + (int64_t)nchunk * 4) = make_int4(bcol[i], -1, -1, -1);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const bool hit = q == qs;
#pragma unroll
          for (int w = 0; w < MW; ++w) {
            const uint32_t t2 = grow ? (tw[q][w] | (on[q][w] & mm[w])) : 0u;
            const uint32_t o2 = grow ? (on[q][w] | mm[w]) : mm[w];
            tw[q][w] = hit ? t2 : tw[q][w];
            on[q][w] = hit ? o2 : on[q][w];
          }
          cn[q] = hit ? (grow ? cn[q] + 1 : 1) : cn[q];
          id[q] = hit && !grow ? nchunk : id[q];
        }
      }
      if (bj == INT_MAX) {
        ++L;
        ++nchunk;
      }
      while (L == EMAX) {
        // ---- stable compaction of the open entries through shared memory; if the open chunks
        // alone fill the list, the oldest is closed and the loop compacts again
        int open = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) open += cn[q] < 4;
        int incl = open;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        int base = incl - open, tot = 0;
        for (int w = 0; w < GT / 32; ++w) {
          base += w < warp ? s_wsum[w] : 0;
          tot += s_wsum[w];
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (cn[q] < 4) {
#pragma unroll
            for (int w = 0; w < MW; ++w) {
              st_ones[base * MW + w] = on[q][w];
              st_twos[base * MW + w] = tw[q][w];
            }
            st_cid[base] = id[q];
            st_cnt[base] = cn[q];
            ++base;
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          const int e = tid * PER + q;
          if (e < tot) {
#pragma unroll
            for (int w = 0; w < MW; ++w) {
              on[q][w] = st_ones[e * MW + w];
              tw[q][w] = st_twos[e * MW + w];
            }
            id[q] = st_cid[e];
            cn[q] = (tot == EMAX && e == 0) ? 4 : st_cnt[e];
          } else {
            cn[q] = 4;
          }
        }
        L = tot;
        __syncthreads();  // staging and s_wsum are reused by the next compaction / batch
      }
    }
    __syncthreads();  // bm / bcol are refilled by the next batch
  }
  if (tid == 0) nchunks[u] = nchunk;
}

#ifdef HINM_EXPERIMENTS
// First-fit chunking of one group's union columns (one CTA per group).  Open chunks live in a
// list in creation order (SoA: ones / twos = rows with >= 1 / >= 2 nonzeros in the chunk); a column
// c with row set m fits chunk e iff twos[e] & m == 0.  Each thread scans its entries e = tid +
// GT*i in increasing order and stops at its first fit; the block minimum is the first fit.  Full
// chunks stay in the list (skipped) until the list reaches EMAX, then a stable compaction drops
// them; if the live open chunks alone fill the list the oldest open one is closed (deterministic).
// Output: chunk_cols[u][4 * chunk + slot] (column, -1 = empty slot), nchunks[u].
__global__ void __launch_bounds__(GT, 1) k_greedy_smem(const uint32_t* __restrict__ mask, int n, int cap_chunks,
                                                  int32_t* __restrict__ chunk_cols, int32_t* __restrict__ nchunks) {
  extern __shared__ __align__(16) uint32_t gsm[];
  uint32_t* ones = gsm;                                    // [MW][EMAX]
  uint32_t* twos = ones + MW * EMAX;                       // [MW][EMAX]
  uint32_t* ones2 = twos + MW * EMAX;                      // compaction target
  uint32_t* twos2 = ones2 + MW * EMAX;
  int32_t* cid = reinterpret_cast<int32_t*>(twos2 + MW * EMAX);  // [EMAX] chunk id
  int32_t* cid2 = cid + EMAX;
  int32_t* cnt = cid2 + EMAX;                              // [EMAX] columns in the chunk
  int32_t* cnt2 = cnt + EMAX;
  __shared__ uint32_t bm[GT][MW + 1];
  __shared__ int bcol[GT];
  __shared__ int s_nb, s_nlist, s_nchunk, s_best[2], s_wsum[GT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = blockIdx.x;
  const uint32_t* mu = mask + (int64_t)u * n * MW;
  int32_t* cc = chunk_cols + (int64_t)u * cap_chunks * 4;
  if (tid == 0) {
    s_nlist = 0;
    s_nchunk = 0;
    s_best[0] = s_best[1] = INT_MAX;
  }
  __syncthreads();
  int it = 0;
  for (int c0 = 0; c0 < n; c0 += GT) {
    // ---- batch of GT columns: keep the ones some row of the group uses (the union), in order
    const int c = c0 + tid;
    uint32_t m[MW];
    bool nz = false;
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      m[w] = c < n ? mu[(int64_t)c * MW + w] : 0u;
      nz |= m[w] != 0u;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) s_wsum[warp] = __popc(bal);
    __syncthreads();
    int off = 0, nb = 0;
    for (int w = 0; w < GT / 32; ++w) {
      off += w < warp ? s_wsum[w] : 0;
      nb += s_wsum[w];
    }
    if (nz) {
      const int pos = off + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
      for (int w = 0; w < MW; ++w) bm[pos][w] = m[w];
      bcol[pos] = c;
    }
    __syncthreads();
    for (int i = 0; i < nb; ++i, ++it) {
      uint32_t mm[MW];
#pragma unroll
      for (int w = 0; w < MW; ++w) mm[w] = bm[i][w];
      // each thread checks its 4 contiguous entries with 16-byte loads (EMAX = 4 * GT): the lowest
      // fitting entry of the lowest thread is the first fit
      const int L = s_nlist;
      int mine = INT_MAX;
      const int e0 = tid * 4;
      if (e0 < L) {
        const int4 c4 = *reinterpret_cast<const int4*>(cnt + e0);
        uint4 conf = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int w = 0; w < MW; ++w) {
          const uint4 t4 = *reinterpret_cast<const uint4*>(twos + w * EMAX + e0);
          conf.x |= t4.x & mm[w];
          conf.y |= t4.y & mm[w];
          conf.z |= t4.z & mm[w];
          conf.w |= t4.w & mm[w];
        }
        if (c4.x < 4 && conf.x == 0u) mine = e0;
        else if (e0 + 1 < L && c4.y < 4 && conf.y == 0u) mine = e0 + 1;
        else if (e0 + 2 < L && c4.z < 4 && conf.z == 0u) mine = e0 + 2;
        else if (e0 + 3 < L && c4.w < 4 && conf.w == 0u) mine = e0 + 3;
      }
      mine = __reduce_min_sync(0xffffffffu, mine);
      if (lane == 0 && mine != INT_MAX) atomicMin(&s_best[it & 1], mine);
      __syncthreads();
      const int bj = s_best[it & 1];
      if (bj != INT_MAX) {
        if (tid < MW) {
          const uint32_t on = ones[tid * EMAX + bj];
          twos[tid * EMAX + bj] |= on & mm[tid];
          ones[tid * EMAX + bj] = on | mm[tid];
        }
        if (tid == 0) {
          const int s = cnt[bj];
          cc[(int64_t)cid[bj] * 4 + s] = bcol[i];
          cnt[bj] = s + 1;
        }
      } else {
        if (tid < MW) {
          ones[tid * EMAX + L] = mm[tid];
          twos[tid * EMAX + L] = 0u;
        }
        if (tid == 0) {
          const int id = s_nchunk;
          cid[L] = id;
          cnt[L] = 1;
          cc[(int64_t)id * 4] = bcol[i];
          cc[(int64_t)id * 4 + 1] = -1;
          cc[(int64_t)id * 4 + 2] = -1;
          cc[(int64_t)id * 4 + 3] = -1;
          s_nchunk = id + 1;
          s_nlist = L + 1;
        }
      }
      if (tid == 0) s_best[(it + 1) & 1] = INT_MAX;
      __syncthreads();
      while (s_nlist == EMAX) {
        // ---- stable compaction of the open entries (contiguous blocks of EMAX / GT per thread);
        // if the open chunks alone fill the list, the oldest is closed and the loop compacts again
        constexpr int PER = EMAX / GT;
        int open = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) open += cnt[tid * PER + q] < 4;
        int incl = open;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        int base = incl - open, tot = 0;
        for (int w = 0; w < GT / 32; ++w) {
          base += w < warp ? s_wsum[w] : 0;
          tot += s_wsum[w];
        }
        for (int q = 0; q < PER; ++q) {
          const int e = tid * PER + q;
          if (cnt[e] < 4) {
#pragma unroll
            for (int w = 0; w < MW; ++w) {
              ones2[w * EMAX + base] = ones[w * EMAX + e];
              twos2[w * EMAX + base] = twos[w * EMAX + e];
            }
            cid2[base] = cid[e];
            cnt2[base] = cnt[e];
            ++base;
          }
        }
        __syncthreads();
        for (int e = tid; e < tot; e += GT) {
#pragma unroll
          for (int w = 0; w < MW; ++w) {
            ones[w * EMAX + e] = ones2[w * EMAX + e];
            twos[w * EMAX + e] = twos2[w * EMAX + e];
          }
          cid[e] = cid2[e];
          cnt[e] = (tot == EMAX && e == 0) ? 4 : cnt2[e];
        }
        if (tid == 0) s_nlist = tot;
        __syncthreads();
      }
    }
    __syncthreads();
  }
  if (tid == 0) nchunks[u] = s_nchunk;
}

#endif

// Pseudo-tile offsets: pseudo tile 2u + h has 4 * nchunks[u] vectors.
__global__ void k_gptr(const int32_t* __restrict__ nchunks, int U, int32_t* __restrict__ gptr) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int acc = 0;
    for (int u = 0; u < U; ++u) {
      gptr[2 * u] = acc;
      acc += 4 * nchunks[u];
      gptr[2 * u + 1] = acc;
      acc += 4 * nchunks[u];
    }
    gptr[2 * U] = acc;
  }
}

// Pseudo reference view (V = 128 tiles): thread per (pseudo tile, row, chunk).  The chunk's
// nonzeros of the row are looked up through inv / nm_pos / kept; at most two by construction
// (err otherwise).  Positions ascend; a lone nonzero at slot s sits at (s, 3) or (2, 3), an empty
// (row, chunk) at (0, 1), with zero values.  vec_idx of an empty slot = the chunk's first column
// (gathered, multiplied by zeros).
__global__ void k_view(const int32_t* __restrict__ tile_ptr, const uint8_t* __restrict__ nm_pos,
                       const uint16_t* __restrict__ kept, const int16_t* __restrict__ inv, int n, int V, int T,
                       const int32_t* __restrict__ chunk_cols, int cap_chunks, const int32_t* __restrict__ gptr,
                       uint8_t* __restrict__ nm2, uint16_t* __restrict__ kept2, int32_t* __restrict__ vec2,
                       int* __restrict__ err) {
  const int tp = blockIdx.y, u = tp >> 1, h = tp & 1;
  const int b2 = gptr[tp], C = (gptr[tp + 1] - b2) / 4;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)C * 128) return;
  const int r2 = (int)(idx / C), g = (int)(idx % C);
  const int32_t* cc = chunk_cols + (int64_t)u * cap_chunks * 4 + (int64_t)g * 4;
  const int4 cols = *reinterpret_cast<const int4*>(cc);
  const int cs[4] = {cols.x, cols.y, cols.z, cols.w};
  if (r2 == 0) {
#pragma unroll
    for (int s = 0; s < 4; ++s) vec2[b2 + 4 * g + s] = cs[s] >= 0 ? cs[s] : cs[0];
  }
  const int R = h * 128 + r2, G = GR / V;
  const int t = u * G + R / V, rl = R % V;
  int np = 0, pos[2] = {0, 1};
  uint16_t val[2] = {0, 0};
  if (t < T) {
    const int b = tile_ptr[t], Gt = (tile_ptr[t + 1] - b) / 4;
    const int64_t rbase = (int64_t)V * (b / 4) * 2 + (int64_t)rl * Gt * 2;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (cs[s] < 0) continue;
      const int p = inv[(int64_t)t * n + cs[s]];
      if (p < 0) continue;
      const int q = p & 3;
      const int64_t o = rbase + 2 * (p >> 2);
      const int a0 = nm_pos[o], a1 = nm_pos[o + 1];
      int which = q == a0 ? 0 : q == a1 ? 1 : -1;
      if (which < 0) continue;
      if (np == 2) {
        atomicExch(err, 1);
        return;
      }
      pos[np] = s;
      val[np] = kept[o + which];
      ++np;
    }
  }
  if (np == 1) {
    if (pos[0] == 3) {
      pos[0] = 2;
      pos[1] = 3;
      val[1] = val[0];
      val[0] = 0;
    } else {
      pos[1] = 3;
      val[1] = 0;
    }
  }
  const int64_t o2 = (int64_t)128 * (b2 / 4) * 2 + (int64_t)r2 * C * 2 + 2 * g;
  nm2[o2] = (uint8_t)pos[0];
  nm2[o2 + 1] = (uint8_t)pos[1];
  kept2[o2] = val[0];
  kept2[o2 + 1] = val[1];
}

}  // namespace grp
}  // namespace hinm

using namespace hinm;

static int group_check(const hinm_pack_t* p) {
  if (!p || !p->tile_ptr || !p->vec_idx || !p->nm_pos || !p->kept_bf16) return HINM_ERR_VALUE;
  if (p->N != 2 || p->M != 4 || (p->V != 32 && p->V != 64)) return HINM_ERR_UNSUPPORTED;
  if (p->n > 32767 || p->n < 1 || p->m < 1) return HINM_ERR_UNSUPPORTED;
  return HINM_OK;
}

extern "C" int hinm_group_workspace(const hinm_pack_t* p, size_t* bytes) {
  const int st = group_check(p);
  if (st) return st;
  const int U = (int)ceil_div(p->m, grp::GR);
  if (bytes) *bytes = grp::ws_layout(p->T, p->n, U).total;
  return HINM_OK;
}

extern "C" int hinm_group_plan(const hinm_pack_t* p, void* ws, size_t ws_bytes, int32_t* nchunks_host, void* stream_) {
  using namespace hinm::grp;
  cudaStream_t stream = (cudaStream_t)stream_;
  int st = group_check(p);
  if (st) return st;
  const int T = p->T, n = p->n, V = p->V, U = (int)ceil_div(p->m, GR);
  const Ws L = ws_layout(T, n, U);
  if (!ws || ws_bytes < L.total || !nchunks_host) return HINM_ERR_WORKSPACE;
  char* w = (char*)ws;
  int16_t* inv = (int16_t*)(w + L.inv);
  uint32_t* mask = (uint32_t*)(w + L.mask);
  int32_t* cols = (int32_t*)(w + L.cols);
  int32_t* nch = (int32_t*)(w + L.nch);
  HINM_CUDA_TRY(cudaMemsetAsync(inv, 0xFF, (size_t)T * n * 2, stream));
  HINM_CUDA_TRY(cudaMemsetAsync(mask, 0, (size_t)U * n * MW * 4, stream));
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 16));
  k_inv<<<dim3(gx, T), 256, 0, stream>>>(p->tile_ptr, p->vec_idx, n, inv);
  HINM_LAUNCH_CHECK();
  // masks: 8 warps per CTA, (8 / slabs) 2:4 groups in flight per CTA, grid.x strides the groups
  const int mgx = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n / 4, 8 / (V / 32)), 64));
  k_masks<<<dim3(mgx, T), 256, 0, stream>>>(p->tile_ptr, p->vec_idx, p->nm_pos, n, V, mask);
  HINM_LAUNCH_CHECK();
  const size_t gsmem = (size_t)2 * MW * EMAX * 4 + (size_t)2 * EMAX * 4;  // compaction staging
  auto kg = k_greedy;
  size_t ksmem = gsmem;
#ifdef HINM_EXPERIMENTS
  if (getenv("HINM_GREEDY_SMEM")) {  // the shared-memory list (A / B of identical chunking)
    kg = k_greedy_smem;
    ksmem = (size_t)4 * MW * EMAX * 4 + (size_t)4 * EMAX * 4;
  }
#endif
  HINM_CUDA_TRY(smem_optin((const void*)kg, (int)ksmem));
  kg<<<U, GT, ksmem, stream>>>(mask, n, n, cols, nch);
  HINM_LAUNCH_CHECK();
  HINM_CUDA_TRY(cudaMemcpyAsync(nchunks_host, nch, (size_t)U * 4, cudaMemcpyDeviceToHost, stream));
  HINM_CUDA_TRY(cudaStreamSynchronize(stream));
  return HINM_OK;
}

extern "C" int hinm_group_build(const hinm_pack_t* p, void* ws, size_t ws_bytes, hinm_pack_t* g, void* stream_) {
  using namespace hinm::grp;
  cudaStream_t stream = (cudaStream_t)stream_;
  int st = group_check(p);
  if (st) return st;
  const int T = p->T, n = p->n, V = p->V, U = (int)ceil_div(p->m, GR);
  const Ws L = ws_layout(T, n, U);
  if (!ws || ws_bytes < L.total) return HINM_ERR_WORKSPACE;
  if (!g || g->V != 128 || g->N != 2 || g->M != 4 || g->T != 2 * U || g->m != 2 * U * 128 || g->n != n)
    return HINM_ERR_VALUE;
  if (!g->tile_ptr || !g->vec_idx || !g->nm_pos || !g->kept_bf16) return HINM_ERR_VALUE;
  char* w = (char*)ws;
  const int16_t* inv = (const int16_t*)(w + L.inv);
  const int32_t* cols = (const int32_t*)(w + L.cols);
  const int32_t* nch = (const int32_t*)(w + L.nch);
  int* err = (int*)(w + L.err);
  HINM_CUDA_TRY(cudaMemsetAsync(err, 0, 4, stream));
  k_gptr<<<1, 32, 0, stream>>>(nch, U, g->tile_ptr);
  HINM_LAUNCH_CHECK();
  if (g->total_keep > 0) {
    // a group has at most n chunks (each holds >= 1 union column)
    const int vx = (int)ceil_div((int64_t)n * 128, 256);
    k_view<<<dim3(vx, 2 * U), 256, 0, stream>>>(p->tile_ptr, p->nm_pos, p->kept_bf16, inv, n, V, T, cols, n,
                                                g->tile_ptr, g->nm_pos, g->kept_bf16, g->vec_idx, err);
    HINM_LAUNCH_CHECK();
  }
  int herr = 0;
  HINM_CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, stream));
  HINM_CUDA_TRY(cudaStreamSynchronize(stream));
  if (herr) return HINM_ERR_INVARIANT;
  g->pair = 1;
  g->rows = p->m;
  return g->a_vals ? hinm_pack_build(g, stream_) : HINM_OK;
}
