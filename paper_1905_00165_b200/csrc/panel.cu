// panel.cu -- Stage 2: the panel solves of the blocked factorization.
//
// Listing 3 lines 584-585 (derived at PAPER.md:592-607):
//   A_{J2,J1} := A_{J2,J1} triu(A_{J1})^{-1}          (L21 = A21 U11^{-1})
//   A_{J1,J2} := unit_tril(A_{J1})^{-1} A_{J1,J2}     (U12 = L11^{-1} A12)
// Hermitian specialisation (LDL^H): U11 = D1 L11^H, so
//   W21 = A21 L11^{-H}  (kept in workspace: the update's right operand, W21 = L21 D1)
//   L21 = W21 D1^{-1}   (written in place; scaled by the reciprocal pivot, reading R17).
// The diagonal tile (L11, D1 / U11) is the output of stage 1, already in A.
//
// Design: each CTA owns a chunk of rows (columns for U12) held in REGISTERS, 2-D cyclic over a
// 16 x 16 thread grid; the triangular factor of the diagonal tile sits packed in shared memory;
// the substitution is right-looking with the current column (row) broadcast through a
// double-buffered shared array -> one __syncthreads per pivot.  HBM traffic = one read of the
// panel and one write of L21 (+ W21): SURVEY §8(a3) ~3 (n - j1) nb elements per step.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpp {

// strictly-lower (by columns) / strictly-upper (by rows) packed index of (l, k), l > k
__device__ __forceinline__ int packed(int NB, int k, int l) { return k * (2 * NB - k - 1) / 2 + (l - k - 1); }

// ---------------------------------------------------------------- Hermitian: W21, L21
template <typename T, int NB, int RA>
__global__ void __launch_bounds__(256, 2) panel_herm_kernel(const PanelArgs a) {
  constexpr int TR = 16, TC = 16, CB = NB / TC, ROWS = TR * RA;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Lp = reinterpret_cast<T*>(smem_raw);                 // packed strictly-lower L11
  T* colbuf = Lp + NB * (NB - 1) / 2;                      // [2][ROWS]
  double* rD = reinterpret_cast<double*>(colbuf + 2 * ROWS);  // 1 / D1
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t r0 = j1 + (int64_t)blockIdx.x * ROWS;
  const int nr = (int)(a.n - r0 < ROWS ? a.n - r0 : ROWS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A21 = A + r0 + a.tcol * a.ld;                         // (r, k) at r + k*ld
  const T* T11 = A + a.j0 + a.tcol * a.ld;                 // factored diagonal tile
  T* W = reinterpret_cast<T*>(a.W) + (int64_t)s * a.strideW + (r0 - j1);
  const int tid = threadIdx.x, tr = tid % TR, tc = tid / TR;

  for (int k = tid / 32; k < jb; k += 8)
    for (int l = k + 1 + (tid & 31); l < jb; l += 32) Lp[packed(NB, k, l)] = T11[(int64_t)k * a.ld + l];
  for (int k = tid; k < jb; k += 256) rD[k] = 1.0 / re(T11[(int64_t)k * a.ld + k]);
  T R[RA][CB];
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int r = tr + TR * ia, k = tc + TC * ib;
      R[ia][ib] = (r < nr && k < jb) ? A21[(int64_t)k * a.ld + r] : zero<T>();
    }
  if (tc == 0) {
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) colbuf[tr + TR * ia] = R[ia][0];
  }
  __syncthreads();
  // w solves w L11^H = a:  for k: for l > k: X(:, l) -= X(:, k) conj(L(l, k))
  for (int k = 0; k < jb; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    T xk[RA], Lk[CB];
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) xk[ia] = colbuf[cur * ROWS + tr + TR * ia];
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int l = tc + TC * ib;
      Lk[ib] = (l > k && l < jb) ? cj(Lp[packed(NB, k, l)]) : zero<T>();
    }
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      if (TC * ib + TC - 1 <= k) continue;
#pragma unroll
      for (int ia = 0; ia < RA; ++ia) R[ia][ib] = fms(R[ia][ib], xk[ia], Lk[ib]);
    }
    const int kn = k + 1;
    if (kn < jb) {
#pragma unroll
      for (int ib = 0; ib < CB; ++ib)
        if (tc + TC * ib == kn) {
#pragma unroll
          for (int ia = 0; ia < RA; ++ia) colbuf[nxt * ROWS + tr + TR * ia] = R[ia][ib];
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int r = tr + TR * ia, k = tc + TC * ib;
      if (r < nr && k < jb) {
        W[(int64_t)k * a.ldw + r] = R[ia][ib];
        A21[(int64_t)k * a.ld + r] = scal(R[ia][ib], rD[k]);  // L21 = W21 D1^{-1}
      }
    }
}

// ---------------------------------------------------------------- LU column panel: L21 = A21 U11^{-1}
template <int NB, int RA>
__global__ void __launch_bounds__(256, 2) panel_lu_col_kernel(const PanelArgs a) {
  using T = double2;
  constexpr int TR = 16, TC = 16, CB = NB / TC, ROWS = TR * RA;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Up = reinterpret_cast<T*>(smem_raw);   // packed strictly-upper U11 by rows
  T* colbuf = Up + NB * (NB - 1) / 2;       // [2][ROWS]
  T* rU = colbuf + 2 * ROWS;                // 1 / U(k,k)
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t r0 = j1 + (int64_t)blockIdx.x * ROWS;
  const int nr = (int)(a.n - r0 < ROWS ? a.n - r0 : ROWS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A21 = A + r0 + a.j0 * a.ld;
  const T* T11 = A + a.j0 + a.j0 * a.ld;
  const int tid = threadIdx.x, tr = tid % TR, tc = tid / TR;
  for (int c = tid / 32; c < jb; c += 8)
    for (int k = tid & 31; k < c; k += 32) Up[packed(NB, k, c)] = T11[(int64_t)c * a.ld + k];
  for (int k = tid; k < jb; k += 256) rU[k] = recip(T11[(int64_t)k * a.ld + k]);
  T R[RA][CB];
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int r = tr + TR * ia, k = tc + TC * ib;
      R[ia][ib] = (r < nr && k < jb) ? A21[(int64_t)k * a.ld + r] : zero<T>();
    }
  if (tc == 0) {
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) colbuf[tr + TR * ia] = R[ia][0];
  }
  __syncthreads();
  // l solves l U11 = a:  for k: l_k = x_k / U(k,k); for c > k: x_c -= l_k U(k, c)
  for (int k = 0; k < jb; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    const T rk = rU[k];
    T xk[RA], Uk[CB];
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) xk[ia] = mul(colbuf[cur * ROWS + tr + TR * ia], rk);
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int c = tc + TC * ib;
      Uk[ib] = (c > k && c < jb) ? Up[packed(NB, k, c)] : zero<T>();
    }
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      if (TC * ib + TC - 1 <= k) continue;
#pragma unroll
      for (int ia = 0; ia < RA; ++ia) R[ia][ib] = fms(R[ia][ib], xk[ia], Uk[ib]);
    }
    const int kn = k + 1;
    if (kn < jb) {
#pragma unroll
      for (int ib = 0; ib < CB; ++ib)
        if (tc + TC * ib == kn) {
#pragma unroll
          for (int ia = 0; ia < RA; ++ia) colbuf[nxt * ROWS + tr + TR * ia] = R[ia][ib];
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int r = tr + TR * ia, k = tc + TC * ib;
      if (r < nr && k < jb) A21[(int64_t)k * a.ld + r] = mul(R[ia][ib], rU[k]);
    }
}

// ---------------------------------------------------------------- LU row panel: U12 = L11^{-1} A12
template <int NB, int CB>
__global__ void __launch_bounds__(256, 2) panel_lu_row_kernel(const PanelArgs a) {
  using T = double2;
  constexpr int TR = 16, TC = 16, RA = NB / TR, COLS = TC * CB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Lp = reinterpret_cast<T*>(smem_raw);  // packed strictly-lower L11 by columns
  T* rowbuf = Lp + NB * (NB - 1) / 2;      // [2][COLS]
  const int s = blockIdx.y;
  const int jb = a.jb;
  const int64_t j1 = a.j0 + jb;
  const int64_t c0 = j1 + (int64_t)blockIdx.x * COLS;
  const int nc = (int)(a.n - c0 < COLS ? a.n - c0 : COLS);
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA;
  T* A12 = A + a.j0 + c0 * a.ld;  // (i, c) at i + c*ld
  const T* T11 = A + a.j0 + a.j0 * a.ld;
  const int tid = threadIdx.x, tr = tid % TR, tc = tid / TR;
  for (int k = tid / 32; k < jb; k += 8)
    for (int l = k + 1 + (tid & 31); l < jb; l += 32) Lp[packed(NB, k, l)] = T11[(int64_t)k * a.ld + l];
  T R[RA][CB];
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int i = tr + TR * ia, c = tc + TC * ib;
      R[ia][ib] = (i < jb && c < nc) ? A12[(int64_t)c * a.ld + i] : zero<T>();
    }
  if (tr == 0) {
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) rowbuf[tc + TC * ib] = R[0][ib];
  }
  __syncthreads();
  // u solves L11 u = a (unit lower):  for k: for i > k: x_i -= L(i, k) x_k
  for (int k = 0; k < jb; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    T xk[CB], Lk[RA];
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) xk[ib] = rowbuf[cur * COLS + tc + TC * ib];
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) {
      const int i = tr + TR * ia;
      Lk[ia] = (i > k && i < jb) ? Lp[packed(NB, k, i)] : zero<T>();
    }
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) {
      if (TR * ia + TR - 1 <= k) continue;
#pragma unroll
      for (int ib = 0; ib < CB; ++ib) R[ia][ib] = fms(R[ia][ib], Lk[ia], xk[ib]);
    }
    const int kn = k + 1;
    if (kn < jb) {
#pragma unroll
      for (int ia = 0; ia < RA; ++ia)
        if (tr + TR * ia == kn) {
#pragma unroll
          for (int ib = 0; ib < CB; ++ib) rowbuf[nxt * COLS + tc + TC * ib] = R[ia][ib];
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int i = tr + TR * ia, c = tc + TC * ib;
      if (i < jb && c < nc) A12[(int64_t)c * a.ld + i] = R[ia][ib];
    }
}

template <typename Fn>
static cudaError_t launch_with_smem(Fn fn, dim3 grid, size_t smem, cudaStream_t s, const PanelArgs& a) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, 256, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int NB, int RA>
static cudaError_t launch_herm_t(const PanelArgs& a, cudaStream_t s) {
  constexpr int ROWS = 16 * RA;
  const int64_t m2 = a.n - (a.j0 + a.jb);
  dim3 grid((unsigned)((m2 + ROWS - 1) / ROWS), a.batch);
  const size_t smem = (size_t)(NB * (NB - 1) / 2 + 2 * ROWS) * sizeof(T) + NB * sizeof(double);
  return launch_with_smem(panel_herm_kernel<T, NB, RA>, grid, smem, s, a);
}

template <int NB>
static cudaError_t launch_lu_t(const PanelArgs& a, cudaStream_t s) {
  constexpr int RA = 4, CB = 4;
  const int64_t m2 = a.n - (a.j0 + a.jb);
  dim3 grid((unsigned)((m2 + 16 * RA - 1) / (16 * RA)), a.batch);
  size_t smem = (size_t)(NB * (NB - 1) / 2 + 2 * 16 * RA + NB) * 16;
  cudaError_t e = launch_with_smem(panel_lu_col_kernel<NB, RA>, grid, smem, s, a);
  if (e != cudaSuccess) return e;
  dim3 grid2((unsigned)((m2 + 16 * CB - 1) / (16 * CB)), a.batch);
  smem = (size_t)(NB * (NB - 1) / 2 + 2 * 16 * CB) * 16;
  return launch_with_smem(panel_lu_row_kernel<NB, CB>, grid2, smem, s, a);
}

cudaError_t launch_panel(Kind kind, int nb, const PanelArgs& a, cudaStream_t s) {
  if (a.n - (a.j0 + a.jb) <= 0) return cudaSuccess;
  switch (kind) {
    case HERM_D:
      if (nb <= 32) return launch_herm_t<double, 32, 4>(a, s);
      if (nb <= 64) return launch_herm_t<double, 64, 4>(a, s);
      return launch_herm_t<double, 128, 4>(a, s);
    case HERM_Z:
      if (nb <= 32) return launch_herm_t<double2, 32, 4>(a, s);
      return launch_herm_t<double2, 64, 4>(a, s);
    case LU_Z:
      if (nb <= 32) return launch_lu_t<32>(a, s);
      return launch_lu_t<64>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dpp
