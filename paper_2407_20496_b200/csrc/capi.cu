// Small C-ABI utilities: version and status strings (include/hinm_b200.h).
#include "common.cuh"

extern "C" const char* hinm_version(void) { return "hinm_b200 0.1.0 (sm_100a)"; }

namespace {
__global__ void k_stream_fence() {}
}  // namespace

// A plain (non-PDL) launch after every weight writer: an SpMM launched next with programmatic
// dependent launch may start streaming its weights during the previous kernel's tail (before
// griddepcontrol.wait), and that previous kernel is then never the one that wrote them.
extern "C" int hinm_stream_fence(void* stream) {
  k_stream_fence<<<1, 32, 0, (cudaStream_t)stream>>>();
  HINM_LAUNCH_CHECK();
  return HINM_OK;
}

extern "C" const char* hinm_status_string(int s) {
  switch (s) {
    case HINM_OK: return "ok";
    case HINM_ERR_SHAPE_MISMATCH: return "shape mismatch";
    case HINM_ERR_INDEX: return "index out of range";
    case HINM_ERR_INVARIANT: return "invariant violation";
    case HINM_ERR_GROUPING: return "survivor count not a multiple of the group size";
    case HINM_ERR_BUDGET: return "keep budget not expressible in whole groups";
    case HINM_ERR_DIMENSION: return "shape incompatible with the block sizes";
    case HINM_ERR_VALUE: return "invalid argument";
    case HINM_ERR_CUDA: return "CUDA error";
    case HINM_ERR_WORKSPACE: return "workspace or capacity too small";
    case HINM_ERR_UNSUPPORTED: return "configuration not supported by the kernel";
    default: return "unknown status";
  }
}
