// Output-channel permutation (OCP) cost matrix of the gyro-permutation search on the GPU
// (reference _ocp_cost_matrix, permutation.py:295-327):
//
//   C[i][j] = total - retained(i, j),   retained(i, j) = sum of the k_groups largest of
//             { rem_gains[i'][q] : i' != i }  U  gains(rem_cols[i] + clu_cols[j])
//
// where gains(col) are the sums of consecutive M-chunks of col sorted descending (ties to the lower
// column, _tile_order_and_gains :83-96).  The reference evaluates this with one lexsort and one
// np.partition over all P*G gains per (i, j) -- P^2 of each per OCP iteration, hours at LLaMA scale.
// Here:
//   k_ocp_prep     rem gains of every partition: the compressor's tile sort + chunk sums (compress.cu)
//   (cub)          all P*G rem gains sorted descending once (stable: ties by (row, q)), prefix sums
//   k_ocp_pairs    one CTA per (i, j): the union column scores are formed while loading, sorted
//                  descending in registers / shared memory (keys only: only the values matter),
//                  chunk-summed in numpy's order, prefix-summed; then one thread merges the two
//                  descending lists by binary search: t = #union gains inside the top k_groups,
//                  retained = top(k_groups - t) of the others (from the global prefix sums minus
//                  row i's own prefix) + the top t union gains.
// The retained sum is mathematically the reference's (the same multiset); its floating-point
// association differs from np.partition(...).sum() by a few ulps, which the assignment's 1e-9 tie
// tolerance (hungarian, permutation.py:199-235) absorbs -- tests/test_gpu_gyro.py replays the
// reference's gyro runs bit-for-bit through this path.
#include <cub/cub.cuh>

#include "common.cuh"

namespace hinm {
namespace {

__device__ __forceinline__ uint64_t okey(double d) {
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return b ^ ((b >> 63) ? ~0ull : (1ull << 63));
}
__device__ __forceinline__ double oval(uint64_t k) {
  return __longlong_as_double((long long)(k ^ ((k >> 63) ? (1ull << 63) : ~0ull)));
}

// chunk sum of M descending values in numpy's order (pairwise_sum: sequential below 8 terms)
template <class Get>
__device__ __forceinline__ double chunk_sum(const Get& get, int M) {
  return np_pairwise_sum(get, 0, M) + 0.0;
}

// rows x n scores -> rows x G gains (descending chunk sums); one CTA per row.
template <int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_row_gains(const double* __restrict__ a, const double* __restrict__ b,
                                                  int n, int M, int pairs_b, double* __restrict__ gains) {
  typedef cub::BlockRadixSort<uint64_t, NT, ITEMS> BRS;
  extern __shared__ __align__(16) uint8_t rg_smem[];  // sort temp storage, then the sorted values
  typename BRS::TempStorage& sort_tmp = *reinterpret_cast<typename BRS::TempStorage*>(rg_smem);
  double* vals = reinterpret_cast<double*>(rg_smem);
  const int row = blockIdx.x;
  // pairs_b = 0: row of a; else row = i * pairs_b + j of a[i] + b[j]
  const double* ra = a + (int64_t)(pairs_b ? row / pairs_b : row) * n;
  const double* rb = pairs_b ? b + (int64_t)(row % pairs_b) * n : nullptr;
  uint64_t keys[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = threadIdx.x * ITEMS + i;
    keys[i] = j < n ? okey((rb ? ra[j] + rb[j] : ra[j]) + 0.0) : 0ull;  // padding sorts last
  }
  BRS(sort_tmp).SortDescending(keys);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) vals[threadIdx.x * ITEMS + i] = oval(keys[i]);
  __syncthreads();
  const int G = n / M;
  for (int q = threadIdx.x; q < G; q += NT) {
    auto get = [&](int64_t k) { return vals[q * M + k]; };
    gains[(int64_t)row * G + q] = chunk_sum(get, M);
  }
}

// bytes of the union {sort temp storage, NT * ITEMS sorted doubles}, 16-byte aligned
template <int NT, int ITEMS>
__host__ __device__ constexpr size_t sort_bytes() {
  return ((sizeof(typename cub::BlockRadixSort<uint64_t, NT, ITEMS>::TempStorage) > (size_t)NT * ITEMS * 8
               ? sizeof(typename cub::BlockRadixSort<uint64_t, NT, ITEMS>::TempStorage)
               : (size_t)NT * ITEMS * 8) + 15) & ~size_t(15);
}

// #{q : g[q] > v} (strict) or >= v, for a non-increasing row g of length G
__device__ __forceinline__ int count_above(const double* g, int G, double v, bool inclusive) {
  int lo = 0, hi = G;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (inclusive ? g[mid] >= v : g[mid] > v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct Others {
  const double* sval;    // all P*G rem gains, descending, ties by (row, q)
  const int32_t* sflat;  // their flat index row * G + q
  const double* spref;   // spref[x] = sum of sval[0..x)
  const double* rg;      // P x G rem gains (rows non-increasing)
  const double* rpref;   // P x (G+1) row prefix sums
  int P, G;
  // row-i entries among the first x entries of the sorted list
  __device__ int cnt(int i, int64_t x) const {
    if (x <= 0) return 0;
    const double v = sval[x - 1];
    const int f = sflat[x - 1], r = f / G;
    const double* g = rg + (int64_t)i * G;
    if (r == i) return f - r * G + 1;
    return count_above(g, G, v, i < r);
  }
  // smallest x with x - cnt(i, x) >= m  (the first m entries of "all but row i" end at x)
  __device__ int64_t span(int i, int64_t m) const {
    const int64_t PG = (int64_t)P * G;
    int64_t lo = m, hi = m + G < PG ? m + G : PG;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (mid - cnt(i, mid) >= m) hi = mid; else lo = mid + 1;
    }
    return lo;
  }
  // sum of the m largest rem gains outside row i
  __device__ double top(int i, int64_t m) const {
    if (m <= 0) return 0.0;
    const int64_t x = span(i, m);
    return spref[x] - rpref[(int64_t)i * (G + 1) + cnt(i, x)];
  }
  // the m-th largest (1-based) rem gain outside row i
  __device__ double nth(int i, int64_t m) const { return sval[span(i, m) - 1]; }
};

template <int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_ocp_pairs(const double* __restrict__ rem_cols,
                                                  const double* __restrict__ clu_cols, int n, int M,
                                                  int64_t k_groups, double total, Others o,
                                                  double* __restrict__ C) {
  typedef cub::BlockRadixSort<uint64_t, NT, ITEMS> BRS;
  typedef cub::BlockScan<double, NT> BS;
  __shared__ typename BS::TempStorage scan_tmp;
  // dynamic: [sort temp storage | sorted values] then the G + 1 prefix sums of the union gains
  extern __shared__ __align__(16) uint8_t op_smem[];
  typename BRS::TempStorage& sort_tmp = *reinterpret_cast<typename BRS::TempStorage*>(op_smem);
  double* vals = reinterpret_cast<double*>(op_smem);
  double* upref = reinterpret_cast<double*>(op_smem + sort_bytes<NT, ITEMS>());
  const int P = o.P, G = o.G;
  const int i = blockIdx.x / P, j = blockIdx.x % P;
  const double* ra = rem_cols + (int64_t)i * n;
  const double* rb = clu_cols + (int64_t)j * n;
  uint64_t keys[ITEMS];
#pragma unroll
  for (int e = 0; e < ITEMS; ++e) {
    const int c = threadIdx.x * ITEMS + e;
    keys[e] = c < n ? okey((ra[c] + rb[c]) + 0.0) : 0ull;
  }
  BRS(sort_tmp).SortDescending(keys);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < ITEMS; ++e) vals[threadIdx.x * ITEMS + e] = oval(keys[e]);
  __syncthreads();
  // union gains -> inclusive prefix sums (chunks per thread in order, then a block scan)
  constexpr int PER = ITEMS;  // chunks per thread <= ITEMS (M >= 1)
  const int per = (G + NT - 1) / NT;
  double local = 0.0;
  double g_loc[PER];
  for (int u = 0; u < per; ++u) {
    const int q = threadIdx.x * per + u;
    double g = 0.0;
    if (q < G) {
      auto get = [&](int64_t k) { return vals[q * M + k]; };
      g = chunk_sum(get, M);
    }
    g_loc[u] = g;
    local += g;
  }
  double excl;
  BS(scan_tmp).ExclusiveSum(local, excl);
  double run = excl;
  for (int u = 0; u < per; ++u) {
    const int q = threadIdx.x * per + u;
    if (q < G) {
      run += g_loc[u];
      upref[q + 1] = run;
    }
  }
  if (threadIdx.x == 0) upref[0] = 0.0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  // merge: t = #union gains among the k_groups largest of (others U union)
  const int64_t others = (int64_t)(P - 1) * G;
  double retained;
  if (k_groups <= 0) {
    retained = 0.0;
  } else if (k_groups >= others + G) {
    retained = o.top(i, others) + upref[G];
  } else {
    int64_t tlo = k_groups - others > 0 ? k_groups - others : 0;
    int64_t thi = k_groups < G ? k_groups : G;
    // largest t in [tlo, thi] with (t == tlo) or union[t-1] >= others_nth(k_groups - t + 1)
    while (tlo < thi) {
      const int64_t t = (tlo + thi + 1) >> 1;
      const double u = upref[t] - upref[t - 1];  // union gain t-1 (descending)
      const int64_t m = k_groups - t + 1;        // the other list's m-th largest competes for the slot
      const bool take = m > others || u >= o.nth(i, m);
      if (take) tlo = t; else thi = t - 1;
    }
    retained = o.top(i, k_groups - tlo) + upref[tlo];
  }
  C[(int64_t)i * P + j] = total - retained;
}

__global__ void k_row_prefix(const double* __restrict__ g, int P, int G, double* __restrict__ pref) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  double s = 0.0;
  pref[(int64_t)i * (G + 1)] = 0.0;
  for (int q = 0; q < G; ++q) {
    s += g[(int64_t)i * G + q];
    pref[(int64_t)i * (G + 1) + q + 1] = s;
  }
}

__global__ void k_iota(int32_t* __restrict__ v, int64_t count) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < count) v[x] = (int32_t)x;
}

__global__ void k_keys_of(const double* __restrict__ v, uint64_t* __restrict__ k, int64_t count) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < count) k[x] = okey(v[x] + 0.0);
}

__global__ void k_vals_of(const uint64_t* __restrict__ k, double* __restrict__ v, int64_t count) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < count) v[x] = oval(k[x]);
}

struct OcpWs {
  size_t rg, rpref, keys_in, keys_out, flat_in, flat_out, sval, spref, cub, scan, total;
};

int ocp_ws(int P, int n, int M, OcpWs* L) {
  const int64_t G = n / M, PG = (int64_t)P * G;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~size_t(255); return o; };
  L->rg = take(8 * PG);
  L->rpref = take(8 * (int64_t)P * (G + 1));
  L->keys_in = take(8 * PG);
  L->keys_out = take(8 * PG);
  L->flat_in = take(4 * PG);
  L->flat_out = take(4 * PG);
  L->sval = take(8 * PG);
  L->spref = take(8 * (PG + 1));
  size_t a = 0, b = 0;
  if (cub::DeviceRadixSort::SortPairsDescending(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                                (const int32_t*)nullptr, (int32_t*)nullptr, PG) != cudaSuccess)
    return HINM_ERR_CUDA;
  if (cub::DeviceScan::InclusiveSum(nullptr, b, (const double*)nullptr, (double*)nullptr, PG) != cudaSuccess)
    return HINM_ERR_CUDA;
  L->cub = take(a);
  L->scan = take(b);
  L->total = off;
  return HINM_OK;
}

}  // namespace
}  // namespace hinm

using namespace hinm;

extern "C" int hinm_ocp_workspace(int P, int n, int M, size_t* bytes) {
  if (P < 1 || n < 1 || M < 1 || !bytes) return HINM_ERR_VALUE;
  OcpWs L;
  const int st = ocp_ws(P, n, M, &L);
  if (st) return st;
  *bytes = L.total;
  return HINM_OK;
}

extern "C" int hinm_ocp_costs(const double* rem_cols, const double* clu_cols, int P, int n, int M,
                              int64_t k_groups, double total, double* C, void* workspace,
                              size_t workspace_bytes, void* stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!rem_cols || !clu_cols || !C || P < 1 || n < 1 || M < 1) return HINM_ERR_VALUE;
  if (n > 16384) return HINM_ERR_UNSUPPORTED;  // 1024 threads x 16 keys per CTA
  const int G = n / M;
  if (G < 1 || M > 32) return HINM_ERR_UNSUPPORTED;
  OcpWs L;
  int rc = ocp_ws(P, n, M, &L);
  if (rc) return rc;
  if (!workspace || workspace_bytes < L.total) return HINM_ERR_WORKSPACE;
  char* ws = (char*)workspace;
  double* rg = (double*)(ws + L.rg);
  double* rpref = (double*)(ws + L.rpref);
  uint64_t* kin = (uint64_t*)(ws + L.keys_in);
  uint64_t* kout = (uint64_t*)(ws + L.keys_out);
  int32_t* fin = (int32_t*)(ws + L.flat_in);
  int32_t* fout = (int32_t*)(ws + L.flat_out);
  double* sval = (double*)(ws + L.sval);
  double* spref = (double*)(ws + L.spref);
  const int64_t PG = (int64_t)P * G;
  // 1. rem gains of every partition, and their row prefix sums
  auto row_gains = [&](auto nt, auto items) -> int {
    constexpr int NT = decltype(nt)::value, IT = decltype(items)::value;
    const size_t dyn = sort_bytes<NT, IT>();
    if (dyn > 48 * 1024)
      HINM_CUDA_TRY(smem_optin((const void*)k_row_gains<NT, IT>, (int)dyn));
    k_row_gains<NT, IT><<<P, NT, dyn, st>>>(rem_cols, nullptr, n, M, 0, rg);
    HINM_LAUNCH_CHECK();
    return HINM_OK;
  };
  using N256 = std::integral_constant<int, 256>;
  using N1024 = std::integral_constant<int, 1024>;
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  using I16 = std::integral_constant<int, 16>;
  rc = n <= 1024 ? row_gains(N256{}, I4{}) : n <= 2048 ? row_gains(N256{}, I8{})
     : n <= 4096 ? row_gains(N256{}, I16{}) : n <= 8192 ? row_gains(N1024{}, I8{}) : row_gains(N1024{}, I16{});
  if (rc) return rc;
  k_row_prefix<<<(P + 127) / 128, 128, 0, st>>>(rg, P, G, rpref);
  // 2. all rem gains sorted descending; radix sort is stable, so ties keep (row, q) order
  const unsigned gb = (unsigned)((PG + 255) / 256);
  k_keys_of<<<gb, 256, 0, st>>>(rg, kin, PG);
  k_iota<<<gb, 256, 0, st>>>(fin, PG);
  HINM_LAUNCH_CHECK();
  size_t cb = L.scan - L.cub;
  HINM_CUDA_TRY(cub::DeviceRadixSort::SortPairsDescending(ws + L.cub, cb, kin, kout, fin, fout, PG, 0, 64, st));
  k_vals_of<<<gb, 256, 0, st>>>(kout, sval, PG);
  HINM_LAUNCH_CHECK();
  HINM_CUDA_TRY(cudaMemsetAsync(spref, 0, 8, st));
  size_t sb = L.total - L.scan;
  HINM_CUDA_TRY(cub::DeviceScan::InclusiveSum(ws + L.scan, sb, sval, spref + 1, PG, st));
  // 3. one CTA per (i, j)
  Others o{sval, fout, spref, rg, rpref, P, G};
  auto pairs = [&](auto nt, auto items) -> int {
    constexpr int NT = decltype(nt)::value, IT = decltype(items)::value;
    const size_t dyn = sort_bytes<NT, IT>() + (size_t)(G + 1) * 8;
    if (dyn > 48 * 1024)
      HINM_CUDA_TRY(smem_optin((const void*)k_ocp_pairs<NT, IT>, (int)dyn));
    k_ocp_pairs<NT, IT><<<(unsigned)((int64_t)P * P), NT, dyn, st>>>(rem_cols, clu_cols, n, M, k_groups,
                                                                      total, o, C);
    HINM_LAUNCH_CHECK();
    return HINM_OK;
  };
  return n <= 1024 ? pairs(N256{}, I4{}) : n <= 2048 ? pairs(N256{}, I8{})
       : n <= 4096 ? pairs(N256{}, I16{}) : n <= 8192 ? pairs(N1024{}, I8{}) : pairs(N1024{}, I16{});
}
