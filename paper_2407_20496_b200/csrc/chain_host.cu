// Host-buffer execution of a chain of HiNM SpMMs (the end-to-end path of the bench metric).
//
// The reference's user-facing call is `hinm_spmm(enc, X)` on host arrays (spmm.py:75-99),
// optionally followed by restore_row_order (pruning.py:356) and, for multi-layer use, a chain
// of such products (spmm.py:206-244, cli.py:234-249).  Here the whole chain runs per token
// chunk out of pinned host memory: chunk i's host->device copy, chunk i-1's SpMMs and chunk
// i-2's device->host copy run concurrently on three streams (two internal copy streams plus the
// caller's compute stream), so the end-to-end time approaches max(H2D, compute, D2H) instead of
// their sum.  Three chunk slots of device scratch live in the caller's workspace.
#include <stdlib.h>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace {

#ifndef HINM_CHAIN_SLOTS
#define HINM_CHAIN_SLOTS 3
#endif
constexpr int NSLOT = HINM_CHAIN_SLOTS;

struct CopyStreams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t h2d_done[NSLOT], comp_done[NSLOT], d2h_done[NSLOT];
};

// One set of copy streams / events per (host thread, device): calls are reentrant across
// threads, and a thread's calls are ordered by the host anyway.
int copy_streams(CopyStreams** out) {
  thread_local std::unordered_map<int, CopyStreams> cache;
  int dev = 0;
  HINM_CUDA_TRY(cudaGetDevice(&dev));
  auto it = cache.find(dev);
  if (it == cache.end()) {
    CopyStreams cs;
    HINM_CUDA_TRY(cudaStreamCreateWithFlags(&cs.h2d, cudaStreamNonBlocking));
    HINM_CUDA_TRY(cudaStreamCreateWithFlags(&cs.d2h, cudaStreamNonBlocking));
    for (int s = 0; s < NSLOT; ++s) {
      HINM_CUDA_TRY(cudaEventCreateWithFlags(&cs.h2d_done[s], cudaEventDisableTiming));
      HINM_CUDA_TRY(cudaEventCreateWithFlags(&cs.comp_done[s], cudaEventDisableTiming));
      HINM_CUDA_TRY(cudaEventCreateWithFlags(&cs.d2h_done[s], cudaEventDisableTiming));
    }
    it = cache.emplace(dev, cs).first;
  }
  *out = &it->second;
  return HINM_OK;
}

int64_t slot_elems(const int64_t* buf_rows, int nbuf, int chunk) {
  int64_t rows = 0;
  for (int b = 0; b < nbuf; ++b) rows += buf_rows[b];
  return rows * chunk;
}

}  // namespace

extern "C" int hinm_chain_workspace(const int64_t* buf_rows, int nbuf, int chunk_tokens,
                                    size_t* bytes) {
  if (!buf_rows || !bytes || nbuf < 1 || chunk_tokens < 8 || chunk_tokens % 8) return HINM_ERR_VALUE;
  for (int b = 0; b < nbuf; ++b)
    if (buf_rows[b] < 1) return HINM_ERR_VALUE;
  *bytes = (size_t)NSLOT * slot_elems(buf_rows, nbuf, chunk_tokens) * sizeof(uint16_t);
  return HINM_OK;
}

extern "C" int hinm_chain_run_host(const hinm_chain_step_t* steps, int nsteps, const int64_t* buf_rows,
                                   int nbuf, int out_buf, const uint16_t* X_host, int64_t ldx, int B,
                                   uint16_t* Y_host, int64_t ldy, int chunk_tokens, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (!steps || nsteps < 1 || !buf_rows || nbuf < 2 || out_buf < 1 || out_buf >= nbuf) return HINM_ERR_VALUE;
  if (!X_host || !Y_host || B < 0 || B % 8 || ldx < B || ldy < B) return HINM_ERR_VALUE;
  size_t need = 0;
  int rc = hinm_chain_workspace(buf_rows, nbuf, chunk_tokens, &need);
  if (rc) return rc;
  if (!workspace || workspace_bytes < need) return HINM_ERR_WORKSPACE;
  for (int i = 0; i < nsteps; ++i) {
    const hinm_chain_step_t& s = steps[i];
    if (!s.pack || s.src < 0 || s.src >= nbuf || s.dst < 1 || s.dst >= nbuf || s.src == s.dst)
      return HINM_ERR_VALUE;
    if (s.pack->n != buf_rows[s.src] || s.pack->m != buf_rows[s.dst]) return HINM_ERR_SHAPE_MISMATCH;
  }
  if (B == 0) return HINM_OK;
  CopyStreams* cs = nullptr;
  if ((rc = copy_streams(&cs))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint16_t* ws = (uint16_t*)workspace;
  const int64_t per_slot = slot_elems(buf_rows, nbuf, chunk_tokens);
  auto buf = [&](int slot, int b) {
    int64_t off = (int64_t)slot * per_slot;
    for (int j = 0; j < b; ++j) off += buf_rows[j] * chunk_tokens;
    return ws + off;
  };
  // the chunk slots are free with respect to earlier work on the caller's stream
  HINM_CUDA_TRY(cudaEventRecord(cs->comp_done[0], st));
  HINM_CUDA_TRY(cudaStreamWaitEvent(cs->h2d, cs->comp_done[0], 0));
  HINM_CUDA_TRY(cudaStreamWaitEvent(cs->d2h, cs->comp_done[0], 0));
  // Chunk schedule: the pipeline fills with a quarter chunk and drains with a quarter chunk
  // (the first H2D and the last D2H are not overlapped with anything), full chunks in between.
  std::vector<int> starts, widths;
  {
    const int ramp = std::max(8, (chunk_tokens / 4) / 8 * 8);
    int c0 = 0;
    if (B > 2 * chunk_tokens) {
      starts.push_back(0);
      widths.push_back(ramp);
      c0 = ramp;
    }
    while (c0 < B) {
      int w = std::min(chunk_tokens, B - c0);
      const int left = B - c0 - w;
      if (left > 0 && left < ramp) w = B - c0 - ramp;  // keep a quarter chunk for the drain
      starts.push_back(c0);
      widths.push_back(w);
      c0 += w;
    }
    // split the final full chunk so the drain is a quarter chunk
    if (widths.size() >= 3 && widths.back() > ramp) {
      const int wl = widths.back();
      const int s0 = starts.back();
      widths.back() = wl - ramp;
      starts.push_back(s0 + wl - ramp);
      widths.push_back(ramp);
    }
  }
  const int nchunks = (int)starts.size();
  for (int c = 0; c < nchunks; ++c) {
    const int slot = c % NSLOT;
    const int c0 = starts[c];
    const int w = widths[c];
    // H2D of the chain input once the slot's previous compute has consumed it
    if (c >= NSLOT) HINM_CUDA_TRY(cudaStreamWaitEvent(cs->h2d, cs->comp_done[slot], 0));
    HINM_CUDA_TRY(cudaMemcpy2DAsync(buf(slot, 0), (size_t)chunk_tokens * 2, X_host + c0, (size_t)ldx * 2,
                                    (size_t)w * 2, (size_t)buf_rows[0], cudaMemcpyHostToDevice, cs->h2d));
    HINM_CUDA_TRY(cudaEventRecord(cs->h2d_done[slot], cs->h2d));
    // compute: after the input arrived and the slot's previous result was copied out
    HINM_CUDA_TRY(cudaStreamWaitEvent(st, cs->h2d_done[slot], 0));
    if (c >= NSLOT) HINM_CUDA_TRY(cudaStreamWaitEvent(st, cs->d2h_done[slot], 0));
#ifdef HINM_EXPERIMENTS
    static const bool no_compute = getenv("HINM_CHAIN_NOCOMPUTE") != nullptr;  // copy pipeline alone
#else
    constexpr bool no_compute = false;
#endif
    for (int i = 0; i < nsteps && !no_compute; ++i) {
      const hinm_chain_step_t& s = steps[i];
      rc = hinm_spmm_bf16(s.pack, buf(slot, s.src), chunk_tokens, w, buf(slot, s.dst), chunk_tokens,
                          s.out_order, st);
      if (rc) return rc;
    }
    HINM_CUDA_TRY(cudaEventRecord(cs->comp_done[slot], st));
    // D2H of the chain output
    HINM_CUDA_TRY(cudaStreamWaitEvent(cs->d2h, cs->comp_done[slot], 0));
    HINM_CUDA_TRY(cudaMemcpy2DAsync(Y_host + c0, (size_t)ldy * 2, buf(slot, out_buf), (size_t)chunk_tokens * 2,
                                    (size_t)w * 2, (size_t)buf_rows[out_buf], cudaMemcpyDeviceToHost, cs->d2h));
    HINM_CUDA_TRY(cudaEventRecord(cs->d2h_done[slot], cs->d2h));
  }
  // the call completes on the caller's stream once the last result is on the host
  HINM_CUDA_TRY(cudaEventRecord(cs->d2h_done[0], cs->d2h));
  HINM_CUDA_TRY(cudaStreamWaitEvent(st, cs->d2h_done[0], 0));
  return HINM_OK;
}
