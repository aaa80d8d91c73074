// panel.cu -- Stage 2: the panel solves of the blocked factorization.
//
// Listing 3 lines 584-585 (derived at PAPER.md:592-607):
//   A_{J2,J1} := A_{J2,J1} triu(A_{J1})^{-1}          (L21 = A21 U11^{-1})
//   A_{J1,J2} := unit_tril(A_{J1})^{-1} A_{J1,J2}     (U12 = L11^{-1} A12)
// Hermitian specialisation (LDL^H): U11 = D1 L11^H, so
//   W21 = A21 L11^{-H}  (kept in workspace: the update's right operand, W21 = L21 D1)
//   L21 = W21 D1^{-1}   (written in place).
// The diagonal tile (L11, D1 / U11) is the output of stage 1, already in A.
//
// Design: one CTA per ROWS-row (or column) chunk; the chunk and the triangular factor are staged
// in shared memory and solved by right-looking column substitution (one barrier per pivot),
// then written back with coalesced stores.  HBM traffic = one read + one write of the panel
// (+ W21), i.e. SURVEY §8(a3): ~3 (n - j1) nb elements per step.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpp {

// X(r, k) at k*ROWS + r ; L11(l, k) at k*NB + l
template <typename T, int NB, int ROWS, int NT>
__global__ void __launch_bounds__(NT) panel_herm_kernel(const PanelArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* L = X + NB * ROWS;
  double* D = reinterpret_cast<double*>(L + NB * NB);
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t r0 = j1 + (int64_t)blockIdx.x * ROWS;
  const int nr = (int)(a.n - r0 < ROWS ? a.n - r0 : ROWS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A21 = A + r0 + a.tcol * a.ld;                   // (r, k) at r + k*ld
  const T* T11 = A + a.j0 + a.tcol * a.ld;           // factored diagonal tile
  T* W = reinterpret_cast<T*>(a.W) + (int64_t)s * a.strideW + (r0 - j1);
  const int tid = threadIdx.x;

  for (int idx = tid; idx < jb * ROWS; idx += NT) {
    const int k = idx / ROWS, r = idx % ROWS;
    X[k * ROWS + r] = r < nr ? A21[(int64_t)k * a.ld + r] : zero<T>();
  }
  for (int idx = tid; idx < jb * jb; idx += NT) {
    const int k = idx / jb, l = idx % jb;
    if (l > k) L[k * NB + l] = T11[(int64_t)k * a.ld + l];
    else if (l == k) D[k] = re(T11[(int64_t)k * a.ld + k]);
  }
  __syncthreads();

  // w solves w L11^H = a row by row:  for k: for l > k: X(:, l) -= X(:, k) conj(L(l, k))
  constexpr int G = NT / ROWS;  // column groups
  const int r = tid % ROWS, g = tid / ROWS;
  for (int k = 0; k < jb; ++k) {
    const T xk = X[k * ROWS + r];
    for (int l = k + 1 + g; l < jb; l += G) X[l * ROWS + r] = fms(X[l * ROWS + r], xk, cj(L[k * NB + l]));
    __syncthreads();
  }
  for (int idx = tid; idx < jb * ROWS; idx += NT) {
    const int k = idx / ROWS, rr = idx % ROWS;
    if (rr < nr) {
      const T w = X[k * ROWS + rr];
      W[(int64_t)k * a.ldw + rr] = w;
      A21[(int64_t)k * a.ld + rr] = divr(w, D[k]);  // L21 = W21 D1^{-1}
    }
  }
}

// LU, column panel: L21 = A21 U11^{-1}.  Right-looking: for k: X(:,k) /= U(k,k); for c > k:
// X(:,c) -= X(:,k) U(k,c).   U(k, c) at c*NB + k (column-major tile).
template <int NB, int ROWS, int NT>
__global__ void __launch_bounds__(NT) panel_lu_col_kernel(const PanelArgs a) {
  using T = double2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* X = reinterpret_cast<T*>(smem_raw);
  T* Ut = X + NB * ROWS;
  T* Rinv = Ut + NB * NB;
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t r0 = j1 + (int64_t)blockIdx.x * ROWS;
  const int nr = (int)(a.n - r0 < ROWS ? a.n - r0 : ROWS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A21 = A + r0 + a.j0 * a.ld;
  const T* T11 = A + a.j0 + a.j0 * a.ld;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < jb * ROWS; idx += NT) {
    const int k = idx / ROWS, r = idx % ROWS;
    X[k * ROWS + r] = r < nr ? A21[(int64_t)k * a.ld + r] : zero<T>();
  }
  for (int idx = tid; idx < jb * jb; idx += NT) {
    const int c = idx / jb, k = idx % jb;
    if (k <= c) Ut[c * NB + k] = T11[(int64_t)c * a.ld + k];
  }
  __syncthreads();
  for (int k = tid; k < jb; k += NT) Rinv[k] = recip(Ut[k * NB + k]);
  __syncthreads();
  constexpr int G = NT / ROWS;
  const int r = tid % ROWS, g = tid / ROWS;
  for (int k = 0; k < jb; ++k) {
    const T xk = mul(X[k * ROWS + r], Rinv[k]);  // final L(r, k)
    __syncthreads();
    if (g == 0) X[k * ROWS + r] = xk;
    for (int c = k + 1 + g; c < jb; c += G) X[c * ROWS + r] = fms(X[c * ROWS + r], xk, Ut[c * NB + k]);
    __syncthreads();
  }
  for (int idx = tid; idx < jb * ROWS; idx += NT) {
    const int k = idx / ROWS, rr = idx % ROWS;
    if (rr < nr) A21[(int64_t)k * a.ld + rr] = X[k * ROWS + rr];
  }
}

// LU, row panel: U12 = L11^{-1} A12, column by column (unit lower forward substitution).
// Y(i, c) at c*(NB+1) + i  (odd stride in 16-byte units -> conflict-free column-per-thread).
template <int NB, int COLS, int NT>
__global__ void __launch_bounds__(NT) panel_lu_row_kernel(const PanelArgs a) {
  using T = double2;
  constexpr int LDY = NB + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Y = reinterpret_cast<T*>(smem_raw);
  T* L = Y + LDY * COLS;  // L(i, k) at k*NB + i
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t c0 = j1 + (int64_t)blockIdx.x * COLS;
  const int nc = (int)(a.n - c0 < COLS ? a.n - c0 : COLS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A12 = A + a.j0 + c0 * a.ld;  // (i, c) at i + c*ld
  const T* T11 = A + a.j0 + a.j0 * a.ld;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < jb * COLS; idx += NT) {
    const int c = idx / jb, i = idx % jb;
    Y[c * LDY + i] = c < nc ? A12[(int64_t)c * a.ld + i] : zero<T>();
  }
  for (int idx = tid; idx < jb * jb; idx += NT) {
    const int k = idx / jb, i = idx % jb;
    if (i > k) L[k * NB + i] = T11[(int64_t)k * a.ld + i];
  }
  __syncthreads();
  constexpr int G = NT / COLS;
  const int c = tid % COLS, g = tid / COLS;
  for (int k = 0; k < jb; ++k) {
    const T yk = Y[c * LDY + k];
    for (int i = k + 1 + g; i < jb; i += G) Y[c * LDY + i] = fms(Y[c * LDY + i], L[k * NB + i], yk);
    __syncthreads();
  }
  for (int idx = tid; idx < jb * COLS; idx += NT) {
    const int cc = idx / jb, i = idx % jb;
    if (cc < nc) A12[(int64_t)cc * a.ld + i] = Y[cc * LDY + i];
  }
}

template <typename Fn>
static cudaError_t launch_with_smem(Fn fn, dim3 grid, int nt, size_t smem, cudaStream_t s, const PanelArgs& a) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, nt, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int NB>
static cudaError_t launch_herm_t(const PanelArgs& a, cudaStream_t s) {
  constexpr int ROWS = 64, NT = 256;
  const int64_t m2 = a.n - (a.j0 + a.jb);
  dim3 grid((unsigned)((m2 + ROWS - 1) / ROWS), a.batch);
  const size_t smem = (size_t)(NB * ROWS + NB * NB) * sizeof(T) + NB * sizeof(double);
  return launch_with_smem(panel_herm_kernel<T, NB, ROWS, NT>, grid, NT, smem, s, a);
}

template <int NB>
static cudaError_t launch_lu_t(const PanelArgs& a, cudaStream_t s) {
  constexpr int ROWS = 64, NT = 256;
  const int64_t m2 = a.n - (a.j0 + a.jb);
  dim3 grid((unsigned)((m2 + ROWS - 1) / ROWS), a.batch);
  size_t smem = (size_t)(NB * ROWS + NB * NB + NB) * 16;
  cudaError_t e = launch_with_smem(panel_lu_col_kernel<NB, ROWS, NT>, grid, NT, smem, s, a);
  if (e != cudaSuccess) return e;
  smem = (size_t)((NB + 1) * ROWS + NB * NB) * 16;
  return launch_with_smem(panel_lu_row_kernel<NB, ROWS, NT>, grid, NT, smem, s, a);
}

cudaError_t launch_panel(Kind kind, int nb, const PanelArgs& a, cudaStream_t s) {
  if (a.n - (a.j0 + a.jb) <= 0) return cudaSuccess;
  switch (kind) {
    case HERM_D:
      if (nb <= 32) return launch_herm_t<double, 32>(a, s);
      if (nb <= 64) return launch_herm_t<double, 64>(a, s);
      return launch_herm_t<double, 128>(a, s);
    case HERM_Z:
      if (nb <= 32) return launch_herm_t<double2, 32>(a, s);
      return launch_herm_t<double2, 64>(a, s);
    case LU_Z:
      if (nb <= 32) return launch_lu_t<32>(a, s);
      return launch_lu_t<64>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dpp
