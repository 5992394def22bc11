// Shared helpers for the HiNM B200 library (host + device).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>
#include <vector>

#include "hinm_b200.h"

#define HINM_CUDA_TRY(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      fprintf(stderr, "[hinm] CUDA error %s at %s:%d: %s\n", cudaGetErrorName(_e),   \
              __FILE__, __LINE__, cudaGetErrorString(_e));                           \
      return HINM_ERR_CUDA;                                                          \
    }                                                                                \
  } while (0)

#define HINM_LAUNCH_CHECK() HINM_CUDA_TRY(cudaGetLastError())

namespace hinm {

// Dynamic shared-memory opt-in above 48 KB, cached per (kernel, device, bytes): the attribute call
// costs host time on every launch otherwise (short kernels / per-call launch paths).
inline cudaError_t smem_optin(const void* fn, int bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  struct Entry {
    const void* fn;
    int dev, bytes;
  };
  static std::mutex mu;
  static std::vector<Entry> done;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : done)
      if (e.fn == fn && e.dev == dev && e.bytes >= bytes) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    done.push_back({fn, dev, bytes});
  }
  return e;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

__device__ __forceinline__ double bf16_abs_f64(uint16_t bits) {
  uint32_t u = uint32_t(bits & 0x7FFFu) << 16;
  return (double)__uint_as_float(u);
}

__device__ __forceinline__ float bf16_to_f32(uint16_t bits) {
  return __uint_as_float(uint32_t(bits) << 16);
}

// Saliency of element (row, col): external fp64 scores when given, else |W| from bf16.
struct ScoreSource {
  const uint16_t* W;
  int64_t ldw;
  const double* S;
  int64_t lds;
  __device__ __forceinline__ double operator()(int64_t row, int64_t col) const {
    return S ? S[row * lds + col] : bf16_abs_f64(W[row * ldw + col]);
  }
};

// numpy's pairwise summation order (pairwise_sum_DOUBLE) over n values get(i).
template <class Get>
__device__ double np_pairwise_sum(const Get& get, int64_t lo, int64_t n) {
  if (n < 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = acc + get(lo + i);
    return acc;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
    int64_t i = 8;
    const int64_t stop = n - (n % 8);
    for (; i < stop; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = r[j] + get(lo + i + j);
    }
    double acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) acc = acc + get(lo + i);
    return acc;
  }
  int64_t half = n / 2;
  half -= half % 8;
  return np_pairwise_sum(get, lo, half) + np_pairwise_sum(get, lo + half, n - half);
}

// numpy's pairwise block for n <= 128 (no recursion): 8 accumulators, then the remainder.
template <class Get>
__device__ __forceinline__ double np_pairwise_leaf(const Get& get, int64_t lo, int64_t n) {
  if (n < 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = acc + get(lo + i);
    return acc;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
  int64_t i = 8;
  const int64_t stop = n - (n % 8);
  for (; i < stop; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = r[j] + get(lo + i + j);
  }
  double acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) acc = acc + get(lo + i);
  return acc;
}

// The same summation tree without recursion, for long operands (every recursion level costs a
// device-stack frame; the default 1 KB stack overflows around n ~ 10^4): an explicit post-order
// walk with a small frame stack (16 levels: n up to 128 * 2^15).
template <class Get>
__device__ double np_pairwise_sum_iter(const Get& get, int64_t lo, int64_t n) {
  constexpr int DEPTH = 16;
  int32_t f_lo[DEPTH], f_n[DEPTH];
  double f_left[DEPTH];
  uint8_t f_stage[DEPTH];
  int sp = 0;
  f_lo[0] = (int32_t)lo;
  f_n[0] = (int32_t)n;
  f_stage[0] = 0;
  double ret = 0.0;
  while (true) {
    const int32_t cn = f_n[sp];
    int32_t half = cn / 2;
    half -= half % 8;
    if (cn <= 128) {
      ret = np_pairwise_leaf(get, f_lo[sp], cn);
    } else if (f_stage[sp] == 0) {
      f_stage[sp] = 1;
      f_lo[sp + 1] = f_lo[sp];
      f_n[sp + 1] = half;
      f_stage[sp + 1] = 0;
      ++sp;
      continue;
    } else if (f_stage[sp] == 1) {  // left done (in ret): descend right
      f_left[sp] = ret;
      f_stage[sp] = 2;
      f_lo[sp + 1] = f_lo[sp] + half;
      f_n[sp + 1] = cn - half;
      f_stage[sp + 1] = 0;
      ++sp;
      continue;
    } else {
      ret = f_left[sp] + ret;  // both children done
    }
    if (sp == 0) return ret;
    --sp;
  }
}

// Device error word: lowest (tile, rank) wins, mirroring the reference's per-tile check order.
__device__ __forceinline__ void report_error(int* err, int tile, int rank_code) {
  atomicMin(err, tile * 16 + rank_code);
}

}  // namespace hinm
