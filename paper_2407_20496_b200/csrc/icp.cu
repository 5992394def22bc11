// Tile-wise input channel permutation (ICP) cost matrix on the GPU (permutation.py:414-421).
//
// One ICP iteration draws one vector per group; costs[i][j] is the saliency the N:M stage loses
// when sample j completes group i's remainder:
//   costs[i][j] = (base_i + colsum_j) - kept_ij,
//   base_i  = vals[:, rem_i].sum()                 (a (V, M-1) F-ordered fancy-index copy)
//   colsum_j = vals[:, s_j].sum()                  (a strided column)
//   kept_ij = np.sort(union, 1)[:, -N:].sum()      (an F-ordered (V, N) view)
// Every sum follows numpy's pairwise summation over the operand in memory order (column-major
// for the F-ordered copies), so the matrix is bit-identical to the reference's Python double
// loop, which is O(G^2 V) numpy calls per iteration (422 s for one cfg1 tile iteration).
#include "common.cuh"

namespace hinm {
namespace {

constexpr int MAXM = 16;

__global__ void k_icp_costs(const double* __restrict__ vals, int V, int k,
                            const int32_t* __restrict__ rem, const int32_t* __restrict__ samp,
                            int G, int M, int N, double* __restrict__ costs) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)G * G) return;
  const int i = (int)(idx / G), j = (int)(idx % G);
  const int32_t* ri = rem + (int64_t)i * (M - 1);
  const int sj = samp[j];
  auto base_get = [&](int64_t p) { return vals[(p % V) * k + ri[p / V]]; };
  auto col_get = [&](int64_t r) { return vals[r * k + sj]; };
  // the (M - N + q)-th smallest of row r of the union (rem_i columns, then s_j)
  auto kept_get = [&](int64_t p) {
    const int q = (int)(p / V);
    const int64_t r = p % V;
    double a[MAXM];
    for (int c = 0; c < M - 1; ++c) a[c] = vals[r * k + ri[c]];
    a[M - 1] = vals[r * k + sj];
    for (int x = 1; x < M; ++x) {  // insertion sort (values only; ties are irrelevant)
      const double t = a[x];
      int y = x - 1;
      while (y >= 0 && a[y] > t) {
        a[y + 1] = a[y];
        --y;
      }
      a[y + 1] = t;
    }
    return a[M - N + q];
  };
  const double base = np_pairwise_sum(base_get, 0, (int64_t)(M - 1) * V);
  const double col = np_pairwise_sum(col_get, 0, (int64_t)V);
  const double kept = np_pairwise_sum(kept_get, 0, (int64_t)N * V);
  costs[idx] = (base + col) - kept;
}

}  // namespace
}  // namespace hinm

extern "C" int hinm_icp_costs(const double* vals, int V, int k, const int32_t* rem,
                              const int32_t* samp, int G, int M, int N, double* costs,
                              void* stream) {
  if (!vals || !rem || !samp || !costs || V < 1 || G < 0 || M < 2 || M > hinm::MAXM || N < 1 ||
      N > M)
    return HINM_ERR_VALUE;
  if (G == 0) return HINM_OK;
  const int64_t total = (int64_t)G * G;
  hinm::k_icp_costs<<<(unsigned)hinm::ceil_div(total, 128), 128, 0, (cudaStream_t)stream>>>(
      vals, V, k, rem, samp, G, M, N, costs);
  HINM_LAUNCH_CHECK();
  return HINM_OK;
}
