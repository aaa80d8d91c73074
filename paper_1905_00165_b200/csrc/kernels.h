// kernels.h -- internal launch interface between the host driver and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dpp {

enum Kind { HERM_D = 0, HERM_Z = 1, LU_Z = 2 };

// Stage 1: sequential sample-and-factor of the jb x jb diagonal tile at (j0, j0)
// (Listing 4 line "subsample, A_J1 = unblocked_dpp(A_J1)").
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
};

// Stage 2: panel.  Hermitian: W21 = A21 L11^{-H}, L21 = W21 D1^{-1} (rows j1..n).
// LU: L21 = A21 U11^{-1} and U12 = L11^{-1} A12 (Listing 3).
struct PanelArgs {
  void* A;
  int64_t ld, strideA;
 int64_t n, j0;
  int64_t tcol;         // storage column of the block column (= j0 except distributed)
  int jb;
  void* W;              // Hermitian: W21 workspace, element (r, k) at r + k*ldw (+ s*strideW)
  int64_t ldw, strideW;
  int batch;
};

// Stage 3: trailing update on a region of A22 (Listing 3).
// Hermitian: C -= L21 W21^H (lower triangle only).  LU: C -= L21 U12.
struct UpdateArgs {
  const void* Aop;      // L21 at A22-row 0: element (i, k) at i + k*lda
  int64_t lda, strideA;
  const void* Bop;      // Hermitian: W21 (j, k) at j + k*ldb;  LU: U12 (k, j) at k + j*ldb
  int64_t ldb, strideB;
  void* C;              // A22 origin: element (i, j) at i + j*ldc
  int64_t ldc, strideC;
  int m_total;          // rows of A22 (= cols); bounds for both operands
  int K;                // inner dimension jb
  int row0, col0;       // region origin inside A22
  int rows, cols;       // region extent
  int tri;              // lower-triangular tile enumeration of a square region
  int tiles_m, tiles_n;
  int batch;
  int vec;              // 16-byte aligned operands (real: 2 rows per cp.async)
  // 1D block-column-cyclic mode (bcc_P > 0, Hermitian real, BN == nb): tile column tj is local
  // block q = bcc_q0 + tj whose global columns start at (bcc_r + q*bcc_P)*nb; C points at
  // local storage column 0, row j1 (A22 row 0); bcc_j1 = global index of A22 row 0.
  int bcc_P, bcc_r, bcc_nb, bcc_q0;
  int64_t bcc_j1;
};

cudaError_t launch_diag(Kind kind, int nb, const DiagArgs& a, cudaStream_t s);
cudaError_t launch_panel(Kind kind, int nb, const PanelArgs& a, cudaStream_t s);
cudaError_t launch_update(Kind kind, UpdateArgs a, cudaStream_t s);
cudaError_t launch_uniforms(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u, cudaStream_t s);
cudaError_t launch_zero_state(void* state, double* loglik, void* info, int batch, cudaStream_t s);
size_t diag_smem_bytes(Kind kind, int nb);
int update_tile_m(Kind kind);
int update_tile_n(Kind kind);

}  // namespace dpp
