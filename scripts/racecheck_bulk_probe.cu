// Probe (experiment): does compute-sanitizer racecheck model the completion of cp.async.bulk
// (mbarrier complete_tx) -> mbarrier.try_wait -> ld.shared ordering?  One bulk copy into shared
// memory, every thread waits on the barrier, then reads.  A correct program; if racecheck reports
// hazards here, its reports on the same pattern in k_select_pack2 are tool artefacts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/bin/racecheck_bulk_probe scripts/racecheck_bulk_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void k(const int* src, int* out) {
  __shared__ __align__(128) int buf[1024];
  __shared__ __align__(8) uint64_t bar, empty;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t e = (uint32_t)__cvta_generic_to_shared(&empty);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(e), "r"(blockDim.x / 32));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf)), "l"(src), "r"(4096), "r"(b) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b), "r"(0) : "memory");
  int v = buf[(threadIdx.x * 7) & 1023];
  // round 2 (WAR): every warp releases the buffer on an "empty" barrier (one arrive per warp), the
  // producer waits for all of them, then refills it with a second bulk copy
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(e) : "memory");
  if (threadIdx.x == 0) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(e), "r"(0) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf)), "l"(src + 1024), "r"(4096), "r"(b) : "memory");
  }
  done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b), "r"(1) : "memory");
  out[threadIdx.x] = v + buf[(threadIdx.x * 5) & 1023];
}
int main() {
  int *src, *out;
  cudaMalloc(&src, 8192); cudaMalloc(&out, 4096);
  cudaMemset(src, 1, 8192);
  k<<<4, 256>>>(src, out);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
