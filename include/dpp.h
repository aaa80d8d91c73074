/*
 * dpp.h -- C ABI of the B200-native factorization-based DPP sampler.
 *
 * Implements the method of arXiv 1905.00165 ("High-performance sampling of
 * generic Determinantal Point Processes"): an exact sample of DPP(K) from its
 * marginal kernel K by a randomly modified, unpivoted, right-looking
 * factorization (Theorem "Factorization-based DPP sampling", PAPER.md:389-423;
 * Listing 1), blocked as in Listing 3/4.
 * At pivot j the item is kept with probability Re A(j,j) (u_j <= Re A(j,j));
 * otherwise A(j,j) -= 1; then the usual Schur-complement update.  The result is
 * the kept set (mask), its log-likelihood sum_j ln|final pivot_j|
 * (PAPER.md:395-396), and, in place, the factor of K - 1_{Y^c}
 * (Listing 1 caption).
 *
 * Conventions (every entry point):
 *  - Matrices are column-major with leading dimension ld >= max(1, n).
 *    Complex matrices are interleaved (re, im) pairs of doubles (dpp_complex_t).
 *  - Unless the name ends in _host, ALL pointers (K, mask, loglik, info, work,
 *    opts->forced) are DEVICE pointers and the call is stream-ordered and
 *    asynchronous: results are valid once `stream` has been synchronised.
 *    `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - The caller owns every buffer.  The library never allocates device memory
 *    on the sampling path: it uses `work` (>= dpp_workspace_bytes(...) bytes,
 *    256-byte aligned).
 *  - Uniforms: u_j = Philox4x32-10 with key (lo32 seed, hi32 seed) and counter
 *    (lo32 j, hi32 j, lo32 b, hi32 b), x = (r.y << 32) | r.x,
 *    u = (2 (x >> 12) + 1) 2^-53 -- j is the GLOBAL pivot index, b the sample
 *    index.  Results are therefore independent of nb, lookahead, chunking and
 *    GPU count (reading R2).
 *  - Hermitian entry points read and write the LOWER triangle only (strict
 *    lower = L with implicit unit diagonal, diagonal = real D); the strict
 *    upper triangle is never touched; Im of a diagonal entry is treated as 0.
 *    The LU entry point overwrites all of K (strict lower = L, diag+upper = U).
 *  - Return codes: 0 = OK; negative = error (dpp_strerror).  Numerical
 *    anomalies are NOT errors: ties (|u_j - d_j| <= tie_tol), out-of-range
 *    pivots (d_j outside [-range_tol, 1+range_tol]) and non-real LU pivots are
 *    counted in dpp_info_t.  A zero pivot cannot occur: |final pivot| >=
 *    min(u, 1-u) >= 2^-53 for any real pivot value (reading R7).
 *    Asynchronous CUDA faults surface at the caller's synchronisation.
 *  - n = 0 is valid: loglik = 0, info zeroed (first_tie = -1), mask untouched.
 *  - Streams: with lookahead (default) a call runs on an internal pair of
 *    prioritised streams forked from and joined back into the caller's
 *    `stream`.  Each device has a pool of 4 pairs; a caller stream keeps the
 *    pair it was first given, new caller streams take the pairs round robin,
 *    so calls on up to 4 distinct caller streams run concurrently and calls
 *    on one caller stream stay in call order.  Beyond 4 caller streams a pair
 *    is shared (stream-ordered: still correct, less overlap).  Concurrent
 *    calls on different streams MUST use distinct workspaces and distinct
 *    mask / loglik / info buffers.
 *  - Thread safety: calls are reentrant; enqueueing on one stream pair is
 *    serialised by a per-pair mutex.  Stage profiling is per host thread.
 */
#ifndef DPP_B200_H_
#define DPP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPP_OK 0
#define DPP_EINVAL (-1)      /* bad size, ld, nb, batch or NULL required pointer */
#define DPP_EWORKSPACE (-2)  /* work == NULL or work_bytes too small or misaligned */
#define DPP_ECUDA (-3)       /* CUDA launch / configuration error */
#define DPP_ENCCL (-4)       /* NCCL error (distributed entry points) */
#define DPP_EUNSUPPORTED (-5)/* device is not sm_100 */

typedef struct { double re, im; } dpp_complex_t;
typedef struct { float re, im; } dpp_complex64_t;
typedef struct CUstream_st* dpp_stream_t; /* == cudaStream_t */

/* Options; pass NULL (or a zero-initialised struct) for the defaults.  The library reads no
 * environment variables: every knob that changes a result's rounding or the schedule is here. */
#define DPP_FLAG_GENERIC_UPDATE 1u /* every update / panel GEMM on the cp.async fallback kernel
                                      (diagnostics: it is otherwise used only for operands that are
                                      not 16-byte aligned); same results up to rounding */
#define DPP_FLAG_FP32_SIMT 2u      /* dpp_sample_herm_s / dpp_sample_lu_c: the updates on the FP32 SIMT pipe (every
                                      product and sum an fp32 operation) instead of the default
                                      3xTF32 split on the tcgen05 tensor cores (each product to
                                      ~2^-21 relative, fp32 accumulation) */
#define DPP_FLAG_NO_SPLIT_CHAIN 4u /* schedule only (results bit-identical): keep the ungrouped
                                      steps' panel and lookahead updates whole on the chain stream
                                      instead of splitting off the next diagonal tile (see DESIGN §6,
                                      "Split chain"); for measurements and tests */
typedef struct {
  int32_t nb;            /* block size: 32, 64, 128 or 256 (0 = default: 128 real, 64 complex).
                            Blocks wider than the kind's tile (128 real, 64 complex) are factored
                            as nb / tile sub-blocks whose trailing updates are applied as one
                            K = nb pass (lookahead on) -- the blocked algorithm of Listing 3/4 with
                            a blocked diagonal-block factorization (Prop. 5) */
  int32_t lookahead;     /* 0 = single stream, 1 = depth-1 lookahead on two streams (default) */
  double tie_tol;        /* default 1e-9 */
  double range_tol;      /* default 1e-8 */
  const uint8_t* forced; /* DEVICE, nullable: forced decisions (replay / likelihood of a
                            given set, SPEC log_likelihood_of); batch x n bytes, row b at
                            forced + b*n; decision j is forced[j] != 0 */
  int64_t batch_chunk;   /* batched: samples factored concurrently (0 = whole batch) */
  int32_t group;         /* G: the trailing updates of G consecutive block steps are applied as
                            one K = G nb pass (lookahead on).  0 = default (3), 1 = off, <= 8 */
  uint32_t flags;        /* DPP_FLAG_* */
  int64_t group_min_rows;/* grouping only while more than this many trailing rows remain;
                            0 = the library's defaults (6144 real nb = 128, 8192 LU, 0 otherwise
                            and for batches >= 8), < 0 = at every size */
} dpp_opts_t;

/* Per-sample diagnostics (DEVICE memory unless the call is _host). */
typedef struct {
  int32_t n_kept;             /* |Y| */
  int32_t n_ties;             /* pivots with |u_j - Re p_j| <= tie_tol */
  int32_t first_tie;          /* first such pivot, -1 if none */
  int32_t n_out_of_range;     /* pivots with Re p_j outside [-range_tol, 1 + range_tol] */
  double min_abs_pivot;       /* min_j |final pivot_j| (+inf if n = 0) */
  double max_abs_imag_pivot;  /* LU only: max_j |Im p_j| before the decision */
} dpp_info_t;

/* Operation codes for dpp_workspace_bytes. */
#define DPP_OP_HERM_D 0
#define DPP_OP_HERM_Z 1
#define DPP_OP_LU_Z 2
#define DPP_OP_HERM_S 3     /* single precision: real symmetric (float) */
#define DPP_OP_LU_C 4       /* single precision: complex non-Hermitian (complex64) */
#define DPP_OP_BATCHED 0x10 /* OR-ed: batched entry point (K copied into work) */
#define DPP_OP_HOST 0x20    /* OR-ed: _host entry point (implies a K copy in work) */

/* Bytes of device workspace needed by the call (op, batch, n, opts). */
size_t dpp_workspace_bytes(int op, int64_t batch, int64_t n, const dpp_opts_t* opts);

/* ---- single sample (sample index b = 0), K overwritten in place ----------
 * n:      order of K (>= 0)
 * K:      DEVICE, n x n column-major, ld >= max(1, n); OVERWRITTEN by the factor
 * seed:   Philox key
 * mask:   DEVICE uint8[n]; 1 = item kept
 * loglik: DEVICE double[1]; sum_j ln|final pivot_j| in pivot order
 * info:   DEVICE dpp_info_t[1] or NULL
 * Cites: Listing 1 blocked per Listing 3/4;
 * Hermitian specialisation PAPER.md:396-398, 626-628. */
int dpp_sample_herm_d(int64_t n, double* K, int64_t ld, uint64_t seed, uint8_t* mask,
                      double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                      size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_z(int64_t n, dpp_complex_t* K, int64_t ld, uint64_t seed, uint8_t* mask,
                      double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                      size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_z(int64_t n, dpp_complex_t* K, int64_t ld, uint64_t seed, uint8_t* mask,
                    double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                    size_t work_bytes, dpp_stream_t stream);

/* ---- single precision (the paper's single-precision
 * runs) ------------------------------------------------
 * Same arguments, layout and semantics as dpp_sample_herm_d / dpp_sample_lu_z
 * with float / complex64 matrices, factored in fp32: the diagonal tiles on the
 * FP32 SIMT pipe, the update GEMMs of unbatched calls on the tcgen05 tensor
 * cores as a 3xTF32 split (complex64: through the real embedding) unless
 * opts->flags has DPP_FLAG_FP32_SIMT (sm_100a has no exact-fp32 tensor-core
 * MMA; batched calls always use the SIMT kernel).  Reading R19: the decision compares the
 * fp64 uniform with the fp32 pivot promoted to fp64; loglik is accumulated in
 * fp64 from the fp32 pivots.  K must be 4- (herm_s) / 8-byte (lu_c) aligned. */
int dpp_sample_herm_s(int64_t n, float* K, int64_t ld, uint64_t seed, uint8_t* mask,
                      double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                      size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_c(int64_t n, dpp_complex64_t* K, int64_t ld, uint64_t seed, uint8_t* mask,
                    double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                    size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_s_batched(int64_t batch, int64_t n, const float* K, int64_t ld,
                              int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                              double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                              void* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_c_batched(int64_t batch, int64_t n, const dpp_complex64_t* K, int64_t ld,
                            int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                            double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                            void* work, size_t work_bytes, dpp_stream_t stream);

/* ---- elementary (projection) DPP sampler -----------------------------------
 * Listing 2, Theorem "Factorization-based elementary DPP
 * sampling": for K an orthogonal projection of rank k, k
 * steps of a left-looking, diagonally pivoted Cholesky factorization whose
 * pivot j is drawn from the current diagonal with probability d_t / (k - j);
 * O(n k^2) instead of O(n^3).  Reading R20: candidates are the unchosen items
 * in original index order; t_j is the first whose running sum of d exceeds
 * u_j * sum(d) (u_j: the Philox uniform of pivot j, sample b, R2).
 * batch independent samples b = b0 .. b0+batch-1 of ONE kernel K (DEVICE,
 * n x n column-major, ld >= n, read-only, real symmetric; only the diagonal
 * and the columns of the drawn items are read).
 * order:  DEVICE int64[batch x k]: items in pivot order (row s at order + s*k)
 * loglik: DEVICE double[batch]: sum_j ln d_{t_j} = ln det(K_Y)
 * ties:   DEVICE int32[batch x 2] (n_ties, first_tie) or NULL: draws whose
 *         target lay within 1e-12 * sum(d) of a candidate boundary
 * work:   DEVICE, >= dpp_elementary_workspace_bytes(batch, n, k) (holds the
 *         n x k factor of every sample).  k * 8 bytes <= 200 KB.
 * Stream-ordered; 2k kernel launches. */
size_t dpp_elementary_workspace_bytes(int64_t batch, int64_t n, int64_t k);
int dpp_elementary_herm_d(int64_t batch, int64_t n, int64_t k, const double* K, int64_t ld,
                          uint64_t seed, uint64_t b0, int64_t* order, double* loglik,
                          int32_t* ties, void* work, size_t work_bytes, dpp_stream_t stream);

/* ---- L-ensemble -> marginal kernel: K = I - (L + I)^{-1} --------------------
 * PAPER.md:1494-1498 ("converting a Hermitian L-ensemble kernel into a
 * marginal kernel via K = I - (L + I)^{-1} ... the equivalent of 3 samples
 * worth of time").  Hermitian PSD L (DEVICE, n x n column-major, ld >= n; real
 * fp64 (_d) or complex128 (_z, 16-byte aligned); 16-byte aligned columns take
 * the fast kernels); the LOWER triangle of L is read and OVERWRITTEN by the
 * lower triangle of K (the strict upper triangle is not touched).
 * Method: LDL^T of L + I with the sampler's kernels (every decision forced to
 * "keep"), inverse of the unit-lower factor by block forward substitution on
 * DMMA GEMMs, then K = I - Y D^{-1} Y^T, Y = Lf^{-T} (3 x n^3/3 flops).
 * logdet: DEVICE double[1] or NULL: ln det(L + I) (the L-ensemble's
 * normaliser).  work: DEVICE, >= dpp_lensemble_workspace_bytes(n) (~8 n^2
 * bytes; op = DPP_OP_HERM_D or DPP_OP_HERM_Z, 0 otherwise).  Stream-ordered. */
size_t dpp_lensemble_workspace_bytes(int op, int64_t n);
int dpp_lensemble_to_marginal_d(int64_t n, double* A, int64_t ld, double* logdet, void* work,
                                size_t work_bytes, dpp_stream_t stream);
int dpp_lensemble_to_marginal_z(int64_t n, dpp_complex_t* A, int64_t ld, double* logdet, void* work,
                                size_t work_bytes, dpp_stream_t stream);

/* ---- greedy MAP inference (in place) ----------------------------------------
 * "By replacing the Bernoulli samples of algorithm [Listing 1]
 * with the maximum-likelihood result for each index inclusion, we arrive at an
 * analogous (approximate) maximum-likelihood inference algorithm."  Same
 * arguments, layout and factor as dpp_sample_* (no seed): item j is kept iff
 * Re p_j >= 1/2 (include at exactly 1/2; reading R18); a tie is
 * |Re p_j - 1/2| <= tie_tol.  loglik = sum_j ln|final pivot_j| is the
 * log-probability of the returned set.  Deterministic. */
int dpp_map_herm_d(int64_t n, double* K, int64_t ld, uint8_t* mask, double* loglik,
                   dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes,
                   dpp_stream_t stream);
int dpp_map_herm_z(int64_t n, dpp_complex_t* K, int64_t ld, uint8_t* mask, double* loglik,
                   dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes,
                   dpp_stream_t stream);
int dpp_map_lu_z(int64_t n, dpp_complex_t* K, int64_t ld, uint8_t* mask, double* loglik,
                 dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes,
                 dpp_stream_t stream);

/* ---- batched independent samples b = b0 .. b0+batch-1 ----------------------
 * K is READ-ONLY: strideK == 0 -> one kernel shared by every sample; else
 * sample s reads the kernel at K + s*strideK (elements).  Each sample is
 * factored in its own copy inside `work`.  mask: batch x n (row s at mask +
 * s*n); loglik: batch; info: batch or NULL. */
int dpp_sample_herm_d_batched(int64_t batch, int64_t n, const double* K, int64_t ld,
                              int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                              double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                              void* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_z_batched(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                              int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                              double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                              void* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_z_batched(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                            int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                            double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                            void* work, size_t work_bytes, dpp_stream_t stream);

/* ---- host-buffer entry points (end-to-end: H2D copy, sample, D2H copy) ----
 * Same as *_batched but K, mask, loglik and info are HOST pointers (pinned
 * memory gives the fastest copies).  `work` is DEVICE memory of at least
 * dpp_workspace_bytes(op | DPP_OP_HOST, batch, n, opts) bytes.  Synchronous:
 * results are valid on return. */
int dpp_sample_herm_d_host(int64_t batch, int64_t n, const double* K, int64_t ld,
                           int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                           double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_z_host(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                           int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                           double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_z_host(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                         int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                         double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                         size_t work_bytes, dpp_stream_t stream);

/* ---- asynchronous host-buffer entry points (pipelined serving) ------------
 * Same as *_host but stream-ordered: the H2D copy of K, the sample and the D2H
 * copies of mask / loglik / info are ENQUEUED on `stream` and the call returns
 * without waiting; results are valid once `stream` has completed.  Host buffers
 * must be pinned (page-locked) and stay valid until then; `work` must not be
 * reused by another call before then.  Two calls on two streams with two
 * workspaces overlap the second call's H2D copy with the first call's
 * factorization (each caller stream gets its own internal stream pair; see
 * "Streams" above). */
int dpp_sample_herm_d_host_async(int64_t batch, int64_t n, const double* K, int64_t ld,
                                 int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                                 double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                                 void* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_z_host_async(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                                 int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                                 double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                                 void* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_lu_z_host_async(int64_t batch, int64_t n, const dpp_complex_t* K, int64_t ld,
                               int64_t strideK, uint64_t seed, uint64_t b0, uint8_t* mask,
                               double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                               void* work, size_t work_bytes, dpp_stream_t stream);

/* ---- device Philox uniforms (the generator the sampler uses) ---------------
 * u[i] = u(seed, j0 + i, b) for i < count, written to DEVICE u.  Exposed so the
 * generator can be checked against curand and the oracle (reading R2). */
int dpp_philox_uniforms(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u,
                        dpp_stream_t stream);

/* ---- distributed 1D block-column-cyclic factorization (one sample) ---------
 * SURVEY §8(e) mode 2; Listing 3/4 with the block
 * columns dealt round-robin over the ranks.  Hermitian kernels only (real:
 * nb = 128, complex: nb = 64 -- opts->nb must be 0 or that value; opts->group
 * is not used).
 * Rank r of P owns block columns c = r, r+P, r+2P, ... (block width nb), stored
 * contiguously as an n x ncols_local column-major array K_local with leading
 * dimension ld_local >= n (ncols_local = dpp_bcc_local_cols(n, nb, P, r));
 * only rows >= the block's first column are read/written (lower triangle).
 * Per block step the owner factors its diagonal tile and panel and broadcasts
 * [partial loglik + counters | pivots D1 | decisions | panel L21 (live rows
 * only, pitch round_up(n - j1, 16))] (dpp_dist_message_bytes), root = owner;
 * every rank then updates its local trailing columns.  With opts->lookahead
 * != 0 (default) the owner of block k+1 updates that block column first and
 * factors it while every rank's trailing update of step k runs (two
 * prioritised streams per rank).  On return (stream-ordered) every rank holds
 * the full mask (n bytes) and loglik; K_local holds the local columns of the
 * factor.  Every rank must call with the same n, seed and opts.
 * Uniforms: global pivot j, sample index b = 0 -- the sample equals the
 * single-GPU sample of the same K and seed whatever P is.
 * Errors: DPP_EINVAL (bad sizes/nb/pointers, or a comm of the other kind),
 * DPP_EWORKSPACE, DPP_ECUDA, DPP_ENCCL (a failed collective; the comm must
 * then be destroyed).
 *
 * Transports (the same per-step code drives both):
 *  - dpp_comm_init: one process per GPU; comm wraps an ncclComm_t created from
 *    a 128-byte ncclUniqueId (all ranks pass the same id) on the CURRENT
 *    device and owns two streams and their events; broadcast = ncclBroadcast.
 *  - dpp_comm_init_local: nranks VIRTUAL ranks on the current device, driven
 *    by ONE call (dpp_sample_herm_{d,z}_dist_local) that takes every rank's
 *    K_local, mask, workspace (arrays of nranks device pointers) and writes
 *    loglik[r], info[r] (device arrays of nranks, info nullable) for each rank
 *    r.  The broadcast is a device-to-device copy per receiver, ordered by
 *    stream events (no kernel waits on another rank's kernel).  For testing
 *    the P > 1 schedule on one GPU and for sampling kernels whose columns are
 *    spread over several allocations; it gives the same results as P
 *    processes. */
typedef struct dpp_comm_s* dpp_comm_t;
int dpp_comm_init(const void* nccl_unique_id, int nranks, int rank, dpp_comm_t* comm);
int dpp_comm_init_local(int nranks, dpp_comm_t* comm);
int dpp_comm_destroy(dpp_comm_t comm);
int64_t dpp_bcc_local_cols(int64_t n, int32_t nb, int nranks, int rank);
/* op: DPP_OP_HERM_D or DPP_OP_HERM_Z; 0 if unsupported.  Per rank. */
size_t dpp_dist_workspace_bytes(int op, int64_t n, int nranks, const dpp_opts_t* opts);
/* Bytes broadcast at block step k (-1 if k is past the last block).  With
 * nranks = 1 nothing is copied: the header only. */
int64_t dpp_dist_message_bytes(int op, int64_t n, int nranks, int64_t k);
int dpp_sample_herm_d_dist(dpp_comm_t comm, int64_t n, double* K_local, int64_t ld_local,
                           uint64_t seed, uint8_t* mask, double* loglik, dpp_info_t* info,
                           const dpp_opts_t* opts, void* work, size_t work_bytes,
                           dpp_stream_t stream);
int dpp_sample_herm_z_dist(dpp_comm_t comm, int64_t n, dpp_complex_t* K_local, int64_t ld_local,
                           uint64_t seed, uint8_t* mask, double* loglik, dpp_info_t* info,
                           const dpp_opts_t* opts, void* work, size_t work_bytes,
                           dpp_stream_t stream);
int dpp_sample_herm_d_dist_local(dpp_comm_t comm, int64_t n, double* const* K_local,
                                 int64_t ld_local, uint64_t seed, uint8_t* const* mask,
                                 double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                                 void* const* work, size_t work_bytes, dpp_stream_t stream);
int dpp_sample_herm_z_dist_local(dpp_comm_t comm, int64_t n, dpp_complex_t* const* K_local,
                                 int64_t ld_local, uint64_t seed, uint8_t* const* mask,
                                 double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                                 void* const* work, size_t work_bytes, dpp_stream_t stream);

/* ---- stage profiling (diagnostics; used by bench.py for the roofline) ------
 * Between dpp_profile_begin() and dpp_profile_end() every stage launch made by
 * this thread's calls on the current device is bracketed by CUDA events ON THE
 * STREAM IT IS LAUNCHED ON.  dpp_profile_end() synchronises those events and
 * returns, per stage (0 = diag tile, 1 = panel, 2 = lookahead update (a),
 * 3 = trailing update (b), 4 = auxiliary kernels: kernel copies, panel scaling and
 * transposes), the number of launches, the summed event time and
 * the ALGORITHMIC flops (paper convention: real flops; a complex multiply-add
 * counts 8, i.e. 4x the real count).  Not reentrant across host threads. */
typedef struct {
  int64_t launches[5];
  double ms[5];        /* summed launch durations */
  double flops[5];
  double ms_union[5];  /* length of the union of the launch intervals (launches of one stage that
                          overlap -- calls in flight on several streams -- count once) */
  double top_flops[5]; /* the stage's launch with the most flops: its flops ... */
  double top_ms[5];    /* ... and its duration */
} dpp_profile_t;
int dpp_profile_begin(void);
/* The same, recording only the stages whose bit (1 << stage) is set in stage_mask
 * (the others launch without events).  DPP_EINVAL if stage_mask has no bit 0..4. */
int dpp_profile_begin_stages(unsigned stage_mask);
int dpp_profile_end(dpp_profile_t* out);
/* The same, plus the launch timeline: records[4 i .. 4 i + 3] = (stage, start ms, end ms, flops) of
 * the i-th bracketed launch in issue order (times relative to the first one issued), for
 * i < max_records; *count (nullable) = the number of launches recorded. */
int dpp_profile_end_records(dpp_profile_t* out, double* records, int64_t max_records, int64_t* count);

/* Diagnostics (the roofline probe of the dominant kernel): ONE launch of the real trailing-update
 * kernel, C -= W L^T on the lower triangle of an m x m region with K-deep operands (W, L: m x K
 * column-major, leading dimension ldo; C: ldc), alone and persistent on every SM, timed with CUDA
 * events on `stream` (synchronises it); *ms = its duration.  The operands are arbitrary data: this
 * measures the kernel, it samples nothing.  Listing 3 line 586. */
int dpp_probe_update_d(int64_t m, int32_t K, const double* W, const double* L, int64_t ldo, double* C,
                       int64_t ldc, float* ms, dpp_stream_t stream);

const char* dpp_strerror(int code);
const char* dpp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DPP_B200_H_ */
