// Cross-check SpMM on CUDA cores, computed from the REFERENCE VIEW of a pack (vec_idx, nm_pos,
// kept values) exactly like hinm_spmm (spmm.py:88-98): out[tV+r] = sum_{g,s} val * X[vec[gM+pos]].
// fp32 accumulation, fp32 output.  Used by the tests to separate compressor bugs from tcgen05
// operand-image / kernel bugs; it is not the product SpMM.
#include "common.cuh"

namespace hinm {

__global__ void k_spmm_simt(const int32_t* __restrict__ tile_ptr, const int32_t* __restrict__ vec,
                            const uint8_t* __restrict__ nm_pos, const uint16_t* __restrict__ kept,
                            const int32_t* __restrict__ sigma_o, const uint16_t* __restrict__ X,
                            int64_t ldx, int B, int V, int N, int M, float* __restrict__ Y,
                            int64_t ldy, int out_order) {
  const int t = blockIdx.y;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.z;
  if (b >= B) return;
  const int k = tile_ptr[t + 1] - tile_ptr[t];
  const int G = k / M;
  const int32_t* vi = vec + tile_ptr[t];
  const int64_t base = (int64_t)V * (tile_ptr[t] / M) * N + (int64_t)r * G * N;
  float acc = 0.f;
  for (int g = 0; g < G; ++g)
    for (int s = 0; s < N; ++s) {
      const int p = nm_pos[base + g * N + s];
      acc = fmaf(bf16_to_f32(kept[base + g * N + s]), bf16_to_f32(X[(int64_t)vi[g * M + p] * ldx + b]),
                 acc);
    }
  const int64_t prow = (int64_t)t * V + r;
  const int64_t orow = out_order == HINM_ORDER_ORIGINAL ? sigma_o[prow] : prow;
  Y[orow * ldy + b] = acc;
}

}  // namespace hinm

extern "C" int hinm_spmm_simt_f32(const hinm_pack_t* p, const uint16_t* X, int64_t ldx, int B,
                                  float* Y, int64_t ldy, int out_order, void* stream) {
  if (!p || !X || !Y || B < 0) return HINM_ERR_VALUE;
  if (B == 0 || p->m == 0) return HINM_OK;
  dim3 grid((unsigned)hinm::ceil_div(B, 128), p->T, p->V);
  hinm::k_spmm_simt<<<grid, 128, 0, (cudaStream_t)stream>>>(
      p->tile_ptr, p->vec_idx, p->nm_pos, p->kept_bf16, p->sigma_o, X, ldx, B, p->V, p->N, p->M, Y,
      ldy, out_order);
  HINM_LAUNCH_CHECK();
  return HINM_OK;
}
