// Squared distances of the gyro search's balanced k-means on the GPU (
// reference _kmeans_pp_init / _balanced_assign, permutation.py:102-145):
//
//   out[p][c] = ((points[p] - centroids[c]) ** 2).sum()      (numpy, last axis contiguous)
//
// numpy reduces the contiguous last axis with its pairwise summation, so each entry is summed in
// exactly that order (np_pairwise_sum): the distances -- and every k-means decision taken from
// them on the host -- are bit-identical to the reference.  At LLaMA scale (P*k = 5504 sampled
// channels x 172 centroids x 4096 features per round) the reference's broadcast materialises a
// 31 GB temporary; here one thread per (point, centroid) streams both rows.
#include "common.cuh"

namespace hinm {
namespace {

__global__ void k_sq_dists(const double* __restrict__ pts, int P, const double* __restrict__ cents, int C,
                           int F, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)P * C) return;
  const int64_t p = i / C, c = i % C;
  const double* a = pts + p * F;
  const double* b = cents + c * F;
  auto get = [&](int64_t f) {
    const double d = __dsub_rn(a[f], b[f]);
    return __dmul_rn(d, d);  // rounded before the add: no FMA contraction (numpy squares, then sums)
  };
  out[i] = np_pairwise_sum_iter(get, 0, F);
}

}  // namespace
}  // namespace hinm

extern "C" int hinm_sq_dists(const double* points, int P, const double* centroids, int C, int F, double* out,
                             void* stream) {
  if (!points || !centroids || !out || P < 0 || C < 0 || F < 1) return HINM_ERR_VALUE;
  if (F > (128 << 15)) return HINM_ERR_UNSUPPORTED;  // depth of the summation-tree walk
  const int64_t n = (int64_t)P * C;
  if (n == 0) return HINM_OK;
  hinm::k_sq_dists<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(points, P, centroids, C, F,
                                                                                   out);
  HINM_LAUNCH_CHECK();
  return HINM_OK;
}
