// hinm_unpack_to_reference: a device pack back to the reference's HiNMEncoding arrays in HOST
// memory (pruning.py:261-281 TileEncoding / HiNMEncoding).
//
// Two sources:
//   HINM_UNPACK_REFERENCE_VIEW  copies the pack's reference view (vec_idx, nm_pos, kept_bf16)
//   HINM_UNPACK_OPERAND_IMAGE   DECODES the tcgen05 operand image the SpMM actually consumes
//                               (gidx, a_vals in UMMA K-major core-matrix order, a_meta in the
//                               tcgen05 2:4 E layout) -- the parity path for "2:4 metadata
//                               bit-exact": every nibble, value and gather index the MMA reads is
//                               mapped back to nm_index / kept_values / vector_index, and the padding
//                               (zero values, positions {0,1}, repeated last gather index) is checked.
// Layout of the image (written by compress.cu k_select_pack / k_pack_*):
//   kp_t = round_up(k_t, 64), tile_kofs = prefix of kp_t, tile_eofs = prefix of ceil(kp_t / 128)
//   a_vals : tile t at kofs_t / 2 * V; MMA step s (32 logical K = 16 compressed values) at s * 16 * V;
//            element (row r, compressed column c < 16) at (r/8)*128 + (c/8)*64 + (r%8)*8 + c%8
//   a_meta : tile t block e (128 logical K) at (eofs_t + e) * V * 4 words; lane L = m0 + 8*k1 + 16*m2
//            holds rows m = m0 + 8*m1 + 16*m2, K-half k1; word w = MMA step w of the block; bits
//            16*m1 + 4*c = nibble p0 | p1 << 2 of group 32*e + 8*w + 4*k1 + c
//   gidx   : tile t at kofs_t, k_t real indices then the last real index repeated
// Synchronous (device -> host copies on `stream`).
#include <vector>

#include "common.cuh"

namespace {

template <class T>
int d2h(std::vector<T>& dst, const T* src, int64_t n, cudaStream_t st) {
  dst.resize((size_t)(n > 0 ? n : 0));
  if (n > 0) HINM_CUDA_TRY(cudaMemcpyAsync(dst.data(), src, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, st));
  return HINM_OK;
}

}  // namespace

extern "C" int hinm_unpack_to_reference(const hinm_pack_t* p, int source, int32_t* tile_ptr_h,
                                        int32_t* vec_idx_h, uint8_t* nm_pos_h, uint16_t* kept_h,
                                        int32_t* sigma_o_h, void* stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!p || !tile_ptr_h || !vec_idx_h || !nm_pos_h || !kept_h || !sigma_o_h) return HINM_ERR_VALUE;
  if (source != HINM_UNPACK_REFERENCE_VIEW && source != HINM_UNPACK_OPERAND_IMAGE) return HINM_ERR_VALUE;
  const int T = p->T, V = p->V, N = p->N, M = p->M;
  const int64_t K = p->total_keep, L = (int64_t)V * (K / M) * N;
  HINM_CUDA_TRY(cudaMemcpyAsync(tile_ptr_h, p->tile_ptr, (size_t)(T + 1) * 4, cudaMemcpyDeviceToHost, st));
  HINM_CUDA_TRY(cudaMemcpyAsync(sigma_o_h, p->sigma_o, (size_t)p->m * 4, cudaMemcpyDeviceToHost, st));
  if (source == HINM_UNPACK_REFERENCE_VIEW) {
    if (K > 0) {
      HINM_CUDA_TRY(cudaMemcpyAsync(vec_idx_h, p->vec_idx, (size_t)K * 4, cudaMemcpyDeviceToHost, st));
      HINM_CUDA_TRY(cudaMemcpyAsync(nm_pos_h, p->nm_pos, (size_t)L, cudaMemcpyDeviceToHost, st));
      HINM_CUDA_TRY(cudaMemcpyAsync(kept_h, p->kept_bf16, (size_t)L * 2, cudaMemcpyDeviceToHost, st));
    }
    HINM_CUDA_TRY(cudaStreamSynchronize(st));
    return tile_ptr_h[T] == K ? HINM_OK : HINM_ERR_INVARIANT;
  }
  // ---- decode the operand image
  if (N != 2 || M != 4 || (V != 32 && V != 64 && V != 128)) return HINM_ERR_UNSUPPORTED;
  if (!p->tile_kofs || !p->tile_eofs || !p->gidx || !p->a_vals || !p->a_meta) return HINM_ERR_VALUE;
  std::vector<int32_t> kofs, eofs;
  if (d2h(kofs, p->tile_kofs, T + 1, st) || d2h(eofs, p->tile_eofs, T + 1, st)) return HINM_ERR_CUDA;
  HINM_CUDA_TRY(cudaStreamSynchronize(st));
  std::vector<int32_t> gidx;
  std::vector<uint16_t> av;
  std::vector<uint32_t> am;
  if (d2h(gidx, p->gidx, kofs[T], st) || d2h(av, p->a_vals, (int64_t)kofs[T] / 2 * V, st) ||
      d2h(am, p->a_meta, (int64_t)eofs[T] * V * 4, st))
    return HINM_ERR_CUDA;
  HINM_CUDA_TRY(cudaStreamSynchronize(st));
  if (tile_ptr_h[T] != K) return HINM_ERR_INVARIANT;
  auto aval = [&](int t, int r, int c) -> uint16_t {  // compressed column c of row r in tile t
    const int s = c >> 4, cs = c & 15;
    return av[(size_t)kofs[t] / 2 * V + (size_t)s * 16 * V + (r >> 3) * 128 + (cs >> 3) * 64 + (r & 7) * 8 +
              (cs & 7)];
  };
  auto nibble = [&](int t, int r, int g) -> uint32_t {  // 2:4 metadata of row r, group g
    const int e = g >> 5, w = (g >> 3) & 3, k1 = (g >> 2) & 1, c = g & 3;
    const int m0 = r & 7, m1 = (r >> 3) & 1, m2 = r >> 4;
    const uint32_t word = am[((size_t)eofs[t] + e) * V * 4 + (size_t)(m0 + 8 * k1 + 16 * m2) * 4 + w];
    return (word >> (16 * m1 + 4 * c)) & 0xFu;
  };
  for (int t = 0; t < T; ++t) {
    const int b = tile_ptr_h[t], k = tile_ptr_h[t + 1] - b, G = k / 4;
    const int kp = kofs[t + 1] - kofs[t];
    if (k < 0 || k % 4 || kp != (int)hinm::round_up(k, 64) || eofs[t + 1] - eofs[t] != (int)hinm::ceil_div(kp, 128))
      return HINM_ERR_INVARIANT;
    for (int i = 0; i < kp; ++i) {
      const int32_t gi = gidx[(size_t)kofs[t] + i];
      if (gi < 0 || gi >= p->n) return HINM_ERR_INDEX;
      if (i < k) vec_idx_h[b + i] = gi;
      else if (gi != gidx[(size_t)kofs[t] + k - 1]) return HINM_ERR_INVARIANT;  // padding repeats
    }
    const size_t base = (size_t)V * (b / 4) * 2;
    const int nblk_groups = (eofs[t + 1] - eofs[t]) * 32;
    for (int r = 0; r < V; ++r) {
      for (int g = 0; g < nblk_groups; ++g) {
        const uint32_t nib = nibble(t, r, g);
        const uint32_t p0 = nib & 3u, p1 = nib >> 2;
        if (g >= G) {  // padding groups: positions {0, 1}, values zero (inside kp)
          if (nib != 0x4u) return HINM_ERR_INVARIANT;
          if (2 * g < kp / 2 && (aval(t, r, 2 * g) || aval(t, r, 2 * g + 1))) return HINM_ERR_INVARIANT;
          continue;
        }
        if (p0 >= p1) return HINM_ERR_INVARIANT;  // nm_index pairs are strictly ascending
        const size_t o = base + (size_t)r * G * 2 + (size_t)g * 2;
        nm_pos_h[o] = (uint8_t)p0;
        nm_pos_h[o + 1] = (uint8_t)p1;
        kept_h[o] = aval(t, r, 2 * g);
        kept_h[o + 1] = aval(t, r, 2 * g + 1);
      }
    }
  }
  return HINM_OK;
}
