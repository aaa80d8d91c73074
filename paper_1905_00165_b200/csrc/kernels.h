// kernels.h -- internal launch interface between the host driver and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdio>

namespace dpp {

// NVTX range (host side; a no-op unless a tool such as ncu --nvtx or nsys is attached): one per
// sampler call and one per block step, so a timeline or an ncu --nvtx-include filter can tell the
// steps' launches apart.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  template <class... T>
  NvtxRange(const char* fmt, T... args) {
    char b[96];
    snprintf(b, sizeof b, fmt, args...);
    nvtxRangePushA(b);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

enum Kind { HERM_D = 0, HERM_Z = 1, LU_Z = 2, HERM_S = 3, LU_C = 4 };  // _S/_C: single precision
inline bool kind_herm(Kind k) { return k == HERM_D || k == HERM_Z || k == HERM_S; }
inline bool kind_cplx(Kind k) { return k == HERM_Z || k == LU_Z || k == LU_C; }
inline size_t kind_esize(Kind k) { return k == HERM_S ? 4 : (k == HERM_D || k == LU_C) ? 8 : 16; }

// Stage 1: sequential sample-and-factor of the jb x jb diagonal tile at (j0, j0)
// (Listing 4 line "subsample, A_J1 = unblocked_dpp(A_J1)"), followed by the
// small dense operators stage 2 needs (inverses of the tile's triangular factors).
struct DiagArgs {
  void* A;              // element pointer of sample 0's matrix (origin (0,0))
  int64_t ld, strideA;  // leading dim, elements between consecutive samples
  int64_t n, j0;
  int64_t tcol;         // storage column of the tile's first column (= j0 except distributed)
  int jb;
  uint64_t seed, b0;
  uint8_t* mask;        // batch x n
  const uint8_t* forced;  // batch x n or null
  void* state;          // SampleState[batch]
  double* loglik;       // user loglik[batch] (written at the last tile) or null
  void* info;           // user dpp_info_t[batch] or null (written at the last tile)
  double tie_tol, range_tol;
  int batch;
  int map;              // greedy MAP (reading R18): u_j := 1/2, keep iff Re p >= 1/2
  // panel operators (written when need_ops): nb x nb column-major, ld = ldm, per sample strideM
  //   Hermitian: Bm(j,k) = delta_jk - conj(Linv(j,k)) / D(j)   (L21 = A21 - A21 (I - G),
  //              G = Linv^H D^-1, i.e. L21 = A21 L11^-H D1^-1), dvec = D1
  //   LU:        Bm(j,k) = delta_jk - Uinv(k,j)  (L21 = A21 U11^-1),
  //              Am(i,k) = -Linv(i,k) for i > k, else 0  (U12 = L11^-1 A12)
  int need_ops;
  void* Bm;
  void* Am;
  double* dvec;          // D1, stride ldm per sample
  int ldm;
  int64_t strideM;
};

// Stage 3 (and, through the same kernel, stage 2): C -= Aop * op(Bop)^T on a region of C.
//   Aop: element (i, k) at i + k*lda,  i < a_rows, k < K
//   Bop: bnmajor = 0: element (j, k) at j + k*ldb; bnmajor = 1: element (k, j) at k + j*ldb; j < b_rows
//   op(B)(j,k) = [conj] B(j,k) [* dscale[k]]
//   mask = 1: only elements on/below the global diagonal (row index >= column index) are written.
struct UpdateArgs {
  const void* Aop;
  int64_t lda, strideA;
  const void* Bop;
  int64_t ldb, strideB;
  void* C;              // C origin: element (i, j) at i + j*ldc
  int64_t ldc, strideC;
  int a_rows, b_rows;   // operand extents (rows of Aop, C-columns of Bop)
  int K;                // inner dimension jb
  int row0, col0;       // region origin inside C
  int rows, cols;       // region extent
  int tri;              // lower-triangular tile enumeration of a square region
  int tiles_m, tiles_n;
  int batch;
  int vec;              // 16-byte aligned operands
  int mask, conj, bnmajor;
  const double* dscale; // per-k scale of B (Hermitian trailing update: D1), stride dstride per sample
  int64_t dstride;
  int ktri;             // 1: A(i, k) = 0 for k < i (upper-triangular A): a tile starts its K loop at
                        //    its first row (fast kernel only; the others just multiply the zeros)
  int btri;             // 1: op(B)(j, k) = 0 for k > j (the stage-2 operators are triangular): a
                        //    warp's K loop stops at its last column (fast kernel only; the others
                        //    just multiply the zeros)
  int fp32_simt;        // single precision: the FP32 SIMT kernel instead of 3xTF32 tensor cores
  void* tcs;            // real single precision: scratch for the 3xTF32 packed operands (or null)
  int64_t tcs_bytes;
  int generic;          // 1: the cp.async fallback kernel even for aligned operands (DPP_FLAG_GENERIC_UPDATE)
  int grid_limit;       // > 0: persistent launch with at most this many CTAs (SMs left to the
                        //      lookahead stream); 0: short-lived CTAs (<= 4 tiles each)
  // 1D block-column-cyclic mode (bcc_P > 0, BN == nb): tile column tj is local block
  // q = bcc_q0 + tj whose global columns start at (bcc_r + q*bcc_P)*nb; C points at local storage
  // column 0, row j1 (A22 row 0); bcc_j1 = global index of A22 row 0.
  int bcc_P, bcc_r, bcc_nb, bcc_q0;
  int64_t bcc_j1;
  // optional second output W = C_new diag(wscale) over the region (the Hermitian panel's
  // pre-scaled copy W21 = L21 D1): element (i, j) at i + j*ldw, wscale[j] per column, strides per
  // sample strideWo / wsstride.  Written by the consumer warps of the warp-specialized panel
  // kernel (fused) or, for the other kernels, by a column-scaling pass after the update.
  void* wout;
  int64_t ldw, strideWo;
  const double* wscale;
  int64_t wsstride;
  // optional source of the C values READ (element (i, j) at i + j*ldcs, stride strideCs per sample;
  // results are still written to C): a region's first update reads the caller's kernel directly
  // instead of a workspace copy made beforehand (driver.cu, deferred copy).  Warp-specialized fast
  // kernel only: launch_update rejects it for the others.
  const void* csrc;
  int64_t ldcs, strideCs;
};

cudaError_t launch_diag(Kind kind, int nb, const DiagArgs& a, cudaStream_t s);
cudaError_t launch_update(Kind kind, UpdateArgs a, cudaStream_t s);
cudaError_t launch_update_simt(Kind kind, UpdateArgs a, cudaStream_t s);  // single precision
cudaError_t launch_update_tc32(UpdateArgs a, cudaStream_t s, bool cplx);  // single precision, 3xTF32 tcgen05
size_t tc32_scratch_bytes(int rows, int cols, int K, bool cplx);
// dst(j, k) = src(k, j) for k < rows, j < cols (elements of es = 8 or 16 bytes), `batch` matrices at
// the given strides: the LU row panel A12 / U12 (jb x m2, N-major as a GEMM operand) <-> its K-major
// transpose.
cudaError_t launch_transpose(size_t es, const void* src, int64_t lds, int64_t strideS, void* dst, int64_t ldd,
                             int64_t strideD, int rows, int cols, int batch, cudaStream_t s);
// W(i, k) = L(i, k) d[k] (i < rows, k < cols), any kind's element type, `batch` panels at the given strides
cudaError_t launch_scale_cols(Kind kind, const void* L, int64_t ldl, int64_t strideL, void* W, int64_t ldw,
                              int64_t strideW, const double* d, int64_t strideD, int rows, int cols, int batch,
                              cudaStream_t s);
// dst <- src for columns [c0, c1) (c1 < 0: n) of `batch` n x n column-major matrices of es-byte
// elements (lower: rows >= column only)
cudaError_t launch_copy_matrix(size_t es, const void* src, int64_t lds, int64_t strideS, void* dst, int64_t ldd,
                               int64_t strideD, int n, int batch, bool lower, cudaStream_t s, int c0 = 0,
                               int c1 = -1);
cudaError_t launch_uniforms(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u, cudaStream_t s);
cudaError_t launch_zero_state(void* state, double* loglik, void* info, int batch, cudaStream_t s);

// Split-chain step, real fp64, nb = 128 (next_tile.cu): the panel's first row tile P0
// (L21_0 = A21_0 - A21_0 Bm^T in place, W21_0 = L21_0 D1 into its slot) and the lookahead update of
// the next diagonal tile LT (lower triangle of C -= W21_0 L21_0^T), one CTA; bit-identical to the
// two update-kernel launches it replaces.  16-byte aligned A21, Bm, ld, ldm.
struct NextTileArgs {
  double* A21; int64_t ld;       // 128 x 128 block (rows j1.., block column j0), in place
  const double* Bm; int64_t ldm;  // the diag tile's panel operator (K-major)
  const double* d;                // D1 (128)
  double* W21; int64_t ldw;       // W21_0 destination (rows 0..127 of the panel slot)
  double* C;                      // the next diagonal tile (ld)
};
cudaError_t launch_next_tile(const NextTileArgs& a, cudaStream_t s);

}  // namespace dpp
