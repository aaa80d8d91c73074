// update_common.cuh -- pieces shared by the two stage-3 kernels (update.cu, update_ws.cu):
// tile enumeration, the DMMA.8x8x4 fragment loop over one shared-memory K-chunk, and the
// accumulator -> shared-memory C subtraction.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpp {

template <bool CPLX> struct Elem { using T = double; };
template <> struct Elem<true> { using T = double2; };

struct TileInfo {
  int grow0, gcol0, nrows, ncols, s;
  int64_t cshift;
  bool valid, diag;
};

// Tile t of the launch (t spans tiles_per_sample x batch).  Lower-triangular enumeration for a
// square Hermitian region, rectangular otherwise, block-column-cyclic column map in bcc mode.
template <int BM, int BN>
__device__ __forceinline__ TileInfo tile_info(const UpdateArgs& a, int t, int tiles_per_sample, bool mask) {
  TileInfo ti{};
  ti.s = t / tiles_per_sample;
  const int u = t % tiles_per_sample;
  int r, c;
  if (a.tri) {
    int q = (int)((sqrtf(8.0f * (float)u + 1.0f) - 1.0f) * 0.5f);  // fp32 guess, fixed up below
    while ((q + 1) * (q + 2) / 2 <= u) ++q;
    while (q * (q + 1) / 2 > u) --q;
    r = q;
    c = u - q * (q + 1) / 2;
  } else {
    r = u % a.tiles_m;
    c = u / a.tiles_m;
  }
  ti.grow0 = a.row0 + r * BM;
  const int row_end = a.row0 + a.rows;
  int col_end;
  if (a.bcc_P > 0) {
    const int64_t q = a.bcc_q0 + c;
    const int64_t gcs = (a.bcc_r + q * a.bcc_P) * (int64_t)a.bcc_nb;
    ti.gcol0 = (int)(gcs - a.bcc_j1);
    col_end = min(ti.gcol0 + a.bcc_nb, a.b_rows);
    ti.cshift = ti.gcol0 - q * a.bcc_nb;
  } else {
    ti.gcol0 = a.col0 + c * BN;
    col_end = a.col0 + a.cols;
    ti.cshift = 0;
  }
  ti.nrows = min(BM, row_end - ti.grow0);
  ti.ncols = min(BN, col_end - ti.gcol0);
  ti.valid = ti.nrows > 0 && ti.ncols > 0 && !(mask && ti.gcol0 > ti.grow0 + BM - 1);
  ti.diag = mask && (ti.gcol0 + ti.ncols - 1 > ti.grow0);
  return ti;
}

template <bool CPLX, int MI, int NI>
struct MmaAcc {
  double re[MI][NI][2];
  double im[CPLX ? MI : 1][CPLX ? NI : 1][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        re[i][j][0] = re[i][j][1] = 0.0;
        if (CPLX) im[CPLX ? i : 0][CPLX ? j : 0][0] = im[CPLX ? i : 0][CPLX ? j : 0][1] = 0.0;
      }
  }
  // Cs(r, c) -= acc for the elements this lane owns; MASK keeps the strict upper triangle intact
  template <bool MASK, int TM, int TN, int LDC>
  __device__ __forceinline__ void subtract_into(typename Elem<CPLX>::T* Cs, int wm, int wn, int lane,
                                                const TileInfo& ti) const {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int r = wm * TM + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < NI; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = wn * TN + j * 8 + 2 * (lane & 3) + e;
          if (r < ti.nrows && c < ti.ncols && (!MASK || ti.grow0 + r >= ti.gcol0 + c)) {
            auto* p = Cs + c * LDC + r;
            if constexpr (!CPLX) {
              *p = *p - re[i][j][e];
            } else {
              double2 v = *p;
              v.x -= re[i][j][e];
              v.y -= im[CPLX ? i : 0][CPLX ? j : 0][e];
              *p = v;
            }
          }
        }
      }
    }
  }
};

// One shared-memory K-chunk: acc += A_chunk * op(B_chunk)^T with DMMA.8x8x4.
//   A: [KC][LDA] (row k holds the BM rows), B: [KC][LDBK] (K-major) or [BN][LDBN] (N-major),
//   Ds: [KC] per-k scale of B (SCALE), CONJ: conjugate B (Hermitian complex).
//   tri (real only, warp-uniform): the warp tile sits on the diagonal of a masked Hermitian tile,
//   so the 8x8 fragments strictly above it (j > i) are never stored and their DMMAs are
//   predicated off (one predicate, no second copy of the loop; grouping them under one branch per
//   k-step keeps all A fragments live and spills).
// Fragments: a = A[m = lane>>2][k = lane&3], b = B[k = lane&3][n = lane>>2].
template <bool CPLX, bool BNMAJ, bool SCALE, bool CONJ, int KC, int MI, int NI, int LDA, int LDBK, int LDBN>
__device__ __forceinline__ void mma_chunk(MmaAcc<CPLX, MI, NI>& acc, const typename Elem<CPLX>::T* As,
                                          const typename Elem<CPLX>::T* Bs, const double* Ds, int m_off, int n_off,
                                          int lane, bool tri = false) {
  using T = typename Elem<CPLX>::T;
#pragma unroll
  for (int ks = 0; ks < KC / 4; ++ks) {
    const int kk = ks * 4 + (lane & 3);
    T af[MI], bf[NI];
#pragma unroll
    for (int i = 0; i < MI; ++i) af[i] = As[kk * LDA + m_off + i * 8 + (lane >> 2)];
    const double dk = SCALE ? Ds[kk] : 1.0;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int nn = n_off + j * 8 + (lane >> 2);
      bf[j] = BNMAJ ? Bs[nn * LDBN + kk] : Bs[kk * LDBK + nn];
      if (SCALE) bf[j] = scal(bf[j], dk);
    }
    if constexpr (!CPLX) {
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j)
          if (j <= i || !tri) dmma884(acc.re[i][j][0], acc.re[i][j][1], af[i], bf[j]);
    } else {
      // a*b:       re += ar br - ai bi ;  im += ar bi + ai br
      // a*conj(b): re += ar br + ai bi ;  im += ai br - ar bi
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const double ar = re(af[i]), ai = im(af[i]);
        const double s_ai = CONJ ? ai : -ai, s_ar = CONJ ? -ar : ar;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double br = re(bf[j]), bi = im(bf[j]);
          dmma884(acc.re[i][j][0], acc.re[i][j][1], ar, br);
          dmma884(acc.re[i][j][0], acc.re[i][j][1], s_ai, bi);
          dmma884(acc.im[CPLX ? i : 0][CPLX ? j : 0][0], acc.im[CPLX ? i : 0][CPLX ? j : 0][1], s_ar, bi);
          dmma884(acc.im[CPLX ? i : 0][CPLX ? j : 0][0], acc.im[CPLX ? i : 0][CPLX ? j : 0][1], ai, br);
        }
      }
    }
  }
}

}  // namespace dpp
