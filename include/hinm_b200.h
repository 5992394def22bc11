/*
 * hinm_b200.h -- C ABI of the B200-native HiNM hot path (libhinm_b200.so).
 *
 * The reference (arXiv 2407.20496, package `hinm`) is pure Python; its hot path
 * sits behind these functions:
 *
 *   hinm_vector_prune   <- hinm.vector_prune(saliency, cfg, sigma_o)       pruning.py:150-164
 *                          (tile_column_scores :68, _tile_order_and_gains :83,
 *                           allocate_vector_budget :99, survivors_per_tile :167)
 *   hinm_nm_select      <- hinm.nm_prune(saliency, vector_mask, cfg, sigma) pruning.py:182-213
 *                          hinm.encode(weights, masks, sigma, cfg)          pruning.py:284-324
 *                          (validate_masks :226-254 in mask mode)
 *   hinm_pack_build     <- (no reference analogue) HiNMEncoding -> tcgen05 operand image
 *   hinm_compress_bf16  <- `hinm encode --permutation` call chain           cli.py:185-194
 *   hinm_spmm_bf16      <- hinm.hinm_spmm(enc, X)                           spmm.py:75-99
 *                          + restore_row_order (out_order=ORIGINAL)        pruning.py:356-360
 *   hinm_spmm_simt_f32  <- same product on CUDA cores (cross-check kernel, not the product path)
 *   hinm_unpack_to_reference <- HiNMEncoding / TileEncoding arrays (pruning.py:261-281) from a pack,
 *                          decoding the tcgen05 operand image (parity of the bytes the MMA reads)
 *
 * Conventions
 *   - All array arguments are DEVICE pointers owned by the caller; the library never
 *     allocates or frees caller memory.  bf16 values are passed as uint16_t bit patterns.
 *   - All work is ordered on `stream` (a cudaStream_t passed as void*).  Functions that
 *     perform input validation on the device (documented "synchronizing") synchronize the
 *     stream once at the end to return the validation status; the others are async.
 *   - Return value: hinm_status_t.  Codes map 1:1 onto the reference's exception classes
 *     (errors.py:8-49) in the Python wrapper.
 *   - Layouts: W is m x n row-major with leading dimension ldw (elements).  X is n x B
 *     channel-major (rows = input channels, tokens contiguous, leading dim ldx).  Y is m x B.
 */
#ifndef HINM_B200_H
#define HINM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HINM_OK = 0,
  HINM_ERR_SHAPE_MISMATCH = 1, /* ShapeMismatch      */
  HINM_ERR_INDEX = 2,          /* IndexError         */
  HINM_ERR_INVARIANT = 3,      /* InvariantViolation */
  HINM_ERR_GROUPING = 4,       /* GroupingError      */
  HINM_ERR_BUDGET = 5,         /* BudgetError        */
  HINM_ERR_DIMENSION = 6,      /* DimensionError     */
  HINM_ERR_VALUE = 7,          /* ValueError (bad argument / unsupported config) */
  HINM_ERR_CUDA = 8,           /* CUDA runtime / launch failure */
  HINM_ERR_WORKSPACE = 9,      /* workspace too small */
  HINM_ERR_UNSUPPORTED = 10    /* config outside what a kernel implements */
} hinm_status_t;

/* Output row order of the SpMM epilogue (north-star subsystem 3). */
enum { HINM_ORDER_SIGMA = 0, HINM_ORDER_ORIGINAL = 1 };

/* Selection source for hinm_nm_select. */
enum { HINM_SELECT_SCORES = 0, HINM_SELECT_MASK = 1 };

/* Source of hinm_unpack_to_reference. */
enum { HINM_UNPACK_REFERENCE_VIEW = 0, HINM_UNPACK_OPERAND_IMAGE = 1 };

/*
 * Device pack of one HiNM-encoded matrix.
 *
 * Reference view (any V, N:M) -- identical content to hinm.HiNMEncoding:
 *   tile_ptr[T+1]          prefix sums of k_t (survivors per tile)
 *   vec_idx[K]             vector_index of every tile, concatenated (sigma_i gather order)
 *   nm_pos / kept_bf16     tile t occupies V * (k_t/M*N) entries starting at V*tile_ptr[t]/M*N,
 *                          row-major (V rows x G_t*N): nm_index / kept_values
 *   sigma_o[m]
 * SpMM operand image (2:4, V in {32,64,128}; NULL pointers when not built):
 *   tile_kofs[T+1]         prefix of kp_t = round_up(k_t, 64)
 *   tile_eofs[T+1]         prefix of ceil(kp_t / 128)  (metadata blocks)
 *   gidx[kpad_cap]         padded gather index (pad = last real index of the tile)
 *   a_vals                 compressed A (V x kp_t/2 per tile) in UMMA K-major core-matrix order
 *   a_meta                 tcgen05 2:4 metadata, V lanes x 16 B per 128-K block
 */
typedef struct hinm_pack_s {
  int32_t m, n, V, N, M, T;
  int64_t total_keep;
  int32_t* tile_ptr;
  int32_t* vec_idx;
  uint8_t* nm_pos;
  uint16_t* kept_bf16;
  int32_t* sigma_o;
  int64_t kpad_cap;
  int64_t meta_words_cap;
  int32_t* tile_kofs;
  int32_t* tile_eofs;
  int32_t* gidx;
  uint16_t* a_vals;
  uint32_t* a_meta;
  /* Union-group image (hinm_group_plan / hinm_group_build; NULL / 0 when not built):
   *   group   a pseudo pack of 128-row tiles used by hinm_spmm_bf16 instead of this pack's image
   *           when it is the faster of the two for the call's token count
   * and, in that pseudo pack:
   *   pair    1: tiles 2u, 2u+1 are the two halves of 256-row group u (the CTA-pair kernel)
   *   rows    output rows (the original m; pseudo rows >= rows are zero padding) */
  struct hinm_pack_s* group;
  int32_t pair;
  int32_t rows;
  /* image choice of hinm_spmm_bf16 for this pack: 0 = the faster for the call, 1 = per-tile only,
   * 2 = union-group (when `group` is set) */
  int32_t image;
} hinm_pack_t;

const char* hinm_version(void);
const char* hinm_status_string(int status);

/* Bytes of device workspace needed by hinm_vector_prune / hinm_compress_bf16. */
int hinm_compress_workspace(int m, int n, int V, int M, size_t* bytes);

/* Capacities of the SpMM operand image: kpad_cap = K + 64*T, meta words, a_vals elements. */
int hinm_pack_capacity(int m, int n, int V, int64_t total_keep, int64_t* kpad_cap,
                       int64_t* meta_words, int64_t* a_vals_elems);

/*
 * Vector pruning (pruning.py:150-164): column scores of every tile in sigma_o row order
 * (fp64, numpy summation order), per-tile descending order (ties -> lower column), group
 * gains, and the global greedy budget (== the total_keep/M smallest keys (-gain, q, t)).
 * Scores come from `S` (fp64, lds) when non-NULL, else |Wd| (fp64 weights) when non-NULL,
 * else |W| (bf16, ldw).
 * Outputs: tile_ptr[T+1] (prefix of k_t), surv[total_keep] ascending survivors per tile
 * (= the default sigma_i), vector_mask[T*n] (uint8 0/1) when non-NULL.  Async.
 */
int hinm_vector_prune(const uint16_t* W, int64_t ldw, const double* Wd, int64_t ldwd,
                      const double* S, int64_t lds, const int32_t* sigma_o, int m, int n, int V, int M, int64_t total_keep,
                      int32_t* tile_ptr, int32_t* surv, uint8_t* vector_mask,
                      void* workspace, size_t workspace_bytes, void* stream);

/*
 * N:M selection inside the sigma_i groups of each tile (pruning.py:182-213) and the
 * reference-view encoding (pruning.py:284-324).  Synchronizing (validates on device):
 *   - sigma_i[t] must be a permutation of the tile's surviving columns (vector_mask row t)
 *     -> HINM_ERR_INVARIANT; k_t % M != 0 -> HINM_ERR_GROUPING (first failing tile wins,
 *     invariant checked before grouping, as in the reference);
 *   - mode HINM_SELECT_MASK (encode from masks): every (row, group) keeps exactly N and no
 *     element survives in a pruned vector -> HINM_ERR_INVARIANT (validate_masks :226-254).
 * Mode SCORES picks the top-N of S (or |W|) per group, ties to the lower position.
 * In mask mode `total_keep` >= 0 also checks sum(vector_mask) == total_keep (validate_masks :234).
 * Outputs (any may be NULL): element_mask[m*n] (uint8, original coords; must be zeroed by the
 * caller), nm_pos / kept_bf16 (from W) / kept_f64 (from Wd) in the reference-view layout above.
 */
int hinm_nm_select(int mode, const uint16_t* W, int64_t ldw, const double* Wd, int64_t ldwd,
                   const double* S, int64_t lds, const uint8_t* element_mask_in,
                   const int32_t* sigma_o, const uint8_t* vector_mask, const int32_t* sig_ptr,
                   const int32_t* sig_idx, int m, int n, int V, int N, int M, int64_t total_keep,
                   uint8_t* element_mask_out, uint8_t* nm_pos, uint16_t* kept_bf16,
                   double* kept_f64, void* stream);

/* Build the SpMM operand image of `pack` from its reference view (2:4, V in {32,64,128}). Async. */
int hinm_pack_build(hinm_pack_t* pack, void* stream);

/*
 * Fused compressor (north-star subsystem 1; the `hinm encode --permutation [--saliency]` chain,
 * cli.py:185-194): W bf16 + sigma_o (+ optional sigma_i CSR) -> complete pack (reference view +
 * operand image).  Scores are |W| when `saliency` is NULL, else the caller's fp64 scores
 * (m x n, leading dim lds; any real values -- load_saliency, pruning.py:42-54, feeding
 * vector_prune / nm_prune as in cli.py:189-190); the kept values always come from W.  `pack`
 * buffers are caller-allocated with the capacities above; sig_ptr/sig_idx NULL selects ascending
 * survivors.  Synchronizing only when a caller sigma_i is validated.
 * The compressor's kernels (here and in hinm_vector_prune) are one dependent chain launched with
 * programmatic stream serialization: each waits for its predecessor (griddepcontrol.wait) before
 * touching memory, so ordinary stream order holds for the caller -- a plain launch after the call
 * waits for all of it; a caller's own PDL-launched kernel must wait as usual before reading the
 * outputs.  The call ends with hinm_stream_fence (see below).
 */
int hinm_compress_bf16(const uint16_t* W, int64_t ldw, const double* saliency, int64_t lds,
                       const int32_t* sigma_o, const int32_t* sig_ptr, const int32_t* sig_idx,
                       hinm_pack_t* pack, uint8_t* vector_mask_scratch, void* workspace,
                       size_t workspace_bytes, void* stream);

/*
 * HiNM SpMM on tcgen05 (north-star subsystems 2+3): Y = W_hinm @ X, bf16 in, fp32 accumulate
 * in TMEM, bf16 out.  Rows of Y in sigma_o order (HINM_ORDER_SIGMA, == hinm_spmm) or original
 * channel order (HINM_ORDER_ORIGINAL, == restore_row_order(hinm_spmm)).  Requires the operand
 * image, B % 8 == 0, ldx % 8 == 0, ldy % 8 == 0, 16-byte aligned X/Y.  With a union-group image
 * attached (pack->group) the image pack->image selects runs (default: the faster one for B tokens;
 * the two images differ only in fp32 summation order); a union-group pseudo pack passed directly
 * always runs on the CTA-pair kernel.  Async.
 */
int hinm_spmm_bf16(const hinm_pack_t* pack, const uint16_t* X, int64_t ldx, int B,
                   uint16_t* Y, int64_t ldy, int out_order, void* stream);

/*
 * End-to-end execution from HOST buffers (the user-facing call of the reference, spmm.py:75-99,
 * for a chain of layers as in spmm.py:206-244 / cli.py:234-249): buffer 0 is the chain input X
 * (buf_rows[0] x B, host, leading dim ldx), every step computes buf[dst] = W(pack) @ buf[src],
 * and buffer out_buf is copied back to Y_host (buf_rows[out_buf] x B, leading dim ldy).  Tokens
 * are processed in chunks of chunk_tokens; H2D, SpMMs and D2H of consecutive chunks overlap on
 * two internal copy streams and `stream`.  Host buffers must be page-locked for the copies to
 * overlap.  Work completes on `stream` (async w.r.t. the host).  B % 8 == 0, chunk % 8 == 0.
 */
typedef struct {
  const hinm_pack_t* pack;
  int32_t src, dst;
  int32_t out_order;
} hinm_chain_step_t;

/* Device workspace of hinm_chain_run_host: 3 chunk slots x sum(buf_rows) x chunk bf16. */
int hinm_chain_workspace(const int64_t* buf_rows, int nbuf, int chunk_tokens, size_t* bytes);

int hinm_chain_run_host(const hinm_chain_step_t* steps, int nsteps, const int64_t* buf_rows,
                        int nbuf, int out_buf, const uint16_t* X_host, int64_t ldx, int B,
                        uint16_t* Y_host, int64_t ldy, int chunk_tokens, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Same product from the reference view on CUDA cores, fp32 out (test cross-check). Async. */
int hinm_spmm_simt_f32(const hinm_pack_t* pack, const uint16_t* X, int64_t ldx, int B,
                       float* Y, int64_t ldy, int out_order, void* stream);

/*
 * The reference view of `pack` in HOST memory, in the pack's flat layout (tile_ptr[T+1],
 * vec_idx[K], nm_pos / kept (bf16 bits) [V*K/M*N], sigma_o[m]): HINM_UNPACK_REFERENCE_VIEW copies the
 * reference-view arrays; HINM_UNPACK_OPERAND_IMAGE decodes the tcgen05 operand image instead (2:4,
 * V in {32,64,128}) and checks its padding (HINM_ERR_INVARIANT / HINM_ERR_INDEX on a malformed
 * image).  Synchronous.
 */
int hinm_unpack_to_reference(const hinm_pack_t* pack, int source, int32_t* tile_ptr, int32_t* vec_idx,
                             uint8_t* nm_pos, uint16_t* kept, int32_t* sigma_o, void* stream);

/*
 * Union-group operand image (2:4, V in {32, 64}; SURVEY §8(a) a10/a13 -- a B200 layout of the same
 * HiNMEncoding, no reference analogue).  G = 256 / V consecutive tiles (256 rows in sigma_o order)
 * share one gather list: the union of their kept vectors, cut into 4-slot chunks in which every row
 * has at most two nonzeros, i.e. a 2:4 matrix of 256 rows that one CTA pair computes with
 * tcgen05.mma.sp.cta_group::2 (half the gathered bytes per flop of the per-tile image at V = 64).
 *   hinm_group_workspace  device workspace bytes for plan + build
 *   hinm_group_plan       chunking (first fit of the union columns); writes the chunk count of
 *                         each of the U = ceil(m / 256) groups to nchunks_host.  Synchronizing.
 *   hinm_group_build      fills the caller-allocated pseudo pack `g` (V = 128, T = 2U, m = 256U,
 *                         n = pack n, total_keep = 8 * sum(nchunks), sigma_o = the pack's, operand
 *                         image capacities from hinm_pack_capacity) -- its reference view is the
 *                         union layout (nm_index / kept_values per row and chunk), its operand image
 *                         is built as for V = 128; sets g->pair = 1, g->rows = m.  Synchronizing
 *                         (HINM_ERR_INVARIANT if a chunk would hold three nonzeros of one row).
 * Link the result with pack->group = g; hinm_spmm_bf16 then picks the faster image per call.
 */
int hinm_group_workspace(const hinm_pack_t* pack, size_t* bytes);
int hinm_group_plan(const hinm_pack_t* pack, void* workspace, size_t workspace_bytes, int32_t* nchunks_host,
                    void* stream);
int hinm_group_build(const hinm_pack_t* pack, void* workspace, size_t workspace_bytes, hinm_pack_t* g,
                     void* stream);

/*
 * Weights and programmatic dependent launch: short hinm_spmm_bf16 launches use PDL, and their weight
 * streams (operand image, gather indices, tile offsets) start during the previous kernel's tail --
 * only the activation reads and the Y stores wait for it (griddepcontrol.wait).  The immediately
 * preceding kernel on the stream must therefore not be one that writes the pack's arrays: every
 * function here that writes them (hinm_compress_bf16, hinm_pack_build, hinm_group_build) ends with
 * hinm_stream_fence, a plain one-CTA launch; a caller that writes pack arrays itself (copies,
 * broadcasts) calls it before the next SpMM.  Async.
 */
int hinm_stream_fence(void* stream);

/* Number of kernel launches issued by the most recent hinm_spmm_bf16 call on this thread. */
int hinm_last_launch_count(void);
/* Image the most recent hinm_spmm_bf16 call on this thread ran: 0 per-tile, 1 union-group. */
int hinm_last_image(void);

/*
 * Gyro-permutation search kernels (the search driver is
 * paper_2407_20496_b200/permutation.py).
 *
 * hinm_icp_costs  <- the ICP cost double loop of icp_tile                  permutation.py:414-421
 *   vals: DEVICE V x k fp64 (row-major, one tile's surviving columns), rem: G x (M-1) and
 *   samp: G column ids into vals (DEVICE int32), costs: DEVICE G x G fp64.  Bit-identical to
 *   the reference (numpy pairwise sums in memory order).  Async.
 * hinm_lex_assignment <- hungarian (lexicographically smallest optimal matching) permutation.py:199-235
 *   C: HOST n x n fp64, assignment: HOST int64[n].  O(n^3) host code (the reference's O(n^2)
 *   linear_sum_assignment calls become one matching + one Dijkstra per row).  Synchronous.
 */
int hinm_icp_costs(const double* vals, int V, int k, const int32_t* rem, const int32_t* samp,
                   int G, int M, int N, double* costs, void* stream);

/*
 * hinm_ocp_costs  <- _ocp_cost_matrix (the global output-channel assignment costs)  permutation.py:295-327
 *   rem_cols / clu_cols: DEVICE P x n fp64 column scores of the partition remainders / sampled
 *   clusters (tile_column_scores order); C: DEVICE P x P fp64,
 *   C[i][j] = total - (sum of the k_groups largest of {gains of every remainder but i} U
 *   gains(rem_cols[i] + clu_cols[j])).  One CTA per (i, j); the reference's per-pair lexsort +
 *   np.partition become a keys-only block sort + a two-list merge over global prefix sums (the
 *   retained sum differs from np.partition(...).sum() only in floating-point association).
 *   n <= 16384.  Workspace from hinm_ocp_workspace.  Async.
 */
int hinm_ocp_workspace(int P, int n, int M, size_t* bytes);

/*
 * hinm_sq_dists   <- the balanced k-means distances of the OCP sampling  permutation.py:102-145
 *   out[p][c] = ((points[p] - centroids[c]) ** 2).sum() in numpy's pairwise summation order
 *   (bit-identical).  points: DEVICE P x F, centroids: DEVICE C x F, out: DEVICE P x C fp64.  Async.
 */
int hinm_sq_dists(const double* points, int P, const double* centroids, int C, int F, double* out,
                  void* stream);
int hinm_ocp_costs(const double* rem_cols, const double* clu_cols, int P, int n, int M, int64_t k_groups,
                   double total, double* C, void* workspace, size_t workspace_bytes, void* stream);
int hinm_lex_assignment(const double* C, int n, int64_t* assignment);

#ifdef __cplusplus
}
#endif
#endif /* HINM_B200_H */
