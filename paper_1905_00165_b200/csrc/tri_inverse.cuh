// tri_inverse.cuh -- inverse of a small lower-triangular matrix held block-packed in shared
// memory (one CTA), shared by the diag-tile kernel (stage-2 operators) and the L-ensemble
// conversion (tile inverses of a factored kernel).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace dpp {

__device__ __forceinline__ double madd(double c, double a, double b) { return fma(a, b, c); }
__device__ __forceinline__ double2 madd(double2 c, double2 a, double2 b) {
  double rx = fma(a.x, b.x, c.x);
  rx = fma(-a.y, b.y, rx);
  double ry = fma(a.x, b.y, c.y);
  ry = fma(a.y, b.x, ry);
  return make_double2(rx, ry);
}
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double neg(double a) { return -a; }
__device__ __forceinline__ double2 neg(double2 a) { return make_double2(-a.x, -a.y); }
__device__ __forceinline__ float madd(float c, float a, float b) { return fmaf(a, b, c); }
__device__ __forceinline__ float2 madd(float2 c, float2 a, float2 b) {
  float rx = fmaf(a.x, b.x, c.x);
  rx = fmaf(-a.y, b.y, rx);
  float ry = fmaf(a.x, b.y, c.y);
  ry = fmaf(a.y, b.x, ry);
  return make_float2(rx, ry);
}
__device__ __forceinline__ float neg(float a) { return -a; }
__device__ __forceinline__ float2 neg(float2 a) { return make_float2(-a.x, -a.y); }

// block-packed lower-triangular storage: 16x16 blocks (I >= J), column-major inside a block with a
// column pitch of BLK_LD = 20 elements.  With a pitch of 16 every column of a block starts on the
// same bank, and the DMMA fragment loads below (lane -> (row lane/4, k lane%4) for A, (k lane%4,
// column lane/4) for B) hit each bank 4 (A) or 8 (B) times per request; with 20 they are
// conflict-free (each 8-byte bank pair serves two lanes: the minimum of two wavefronts).
constexpr int BLK_LD = 20, BLK_SZ = 16 * BLK_LD;
__device__ __forceinline__ int bp(int i, int k) {
  const int I = i >> 4, J = k >> 4;
  return (I * (I + 1) / 2 + J) * BLK_SZ + (i & 15) + (k & 15) * BLK_LD;
}

// C (16x16) += A (16x16) B (16x16) on 16x16 column-major blocks in shared memory, one warp, with
// DMMA.8x8x4: 2x2 output tiles of 8x8, four k-steps of 4.  Fragments of mma.m8n8k4.row.col:
// a = A[m = lane>>2][k = lane&3], b = B[k = lane&3][n = lane>>2], c = C[lane>>2][2(lane&3) + e].
// Complex blocks take four real products (re/im parts of the fragments).
template <typename T> struct BlockAcc16;
template <> struct BlockAcc16<double> {
  double c[2][2][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  }
  __device__ __forceinline__ void mma(const double* A, const double* B, int lane, int lda = BLK_LD, int ldb = BLK_LD) {
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kk = k4 * 4 + (lane & 3);
      double a[2], b[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        a[t] = A[t * 8 + (lane >> 2) + kk * lda];
        b[t] = B[kk + (t * 8 + (lane >> 2)) * ldb];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(c[i][j][0], c[i][j][1], a[i], b[j]);
    }
  }
  // block -> C (the layout store() writes)
  __device__ __forceinline__ void load(const double* C, int lane, int ldc = BLK_LD) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) c[i][j][e] = C[i * 8 + (lane >> 2) + (j * 8 + 2 * (lane & 3) + e) * ldc];
  }
  // C -> block (neg: store -C)
  __device__ __forceinline__ void store(double* C, int lane, bool neg, int ldc = BLK_LD) const {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          C[i * 8 + (lane >> 2) + (j * 8 + 2 * (lane & 3) + e) * ldc] = neg ? -c[i][j][e] : c[i][j][e];
  }
};
template <> struct BlockAcc16<double2> {
  double cr[2][2][2], ci[2][2][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  }
  __device__ __forceinline__ void mma(const double2* A, const double2* B, int lane, int lda = BLK_LD, int ldb = BLK_LD) {
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
      const int kk = k4 * 4 + (lane & 3);
      double2 a[2], b[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        a[t] = A[t * 8 + (lane >> 2) + kk * lda];
        b[t] = B[kk + (t * 8 + (lane >> 2)) * ldb];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          dmma884(cr[i][j][0], cr[i][j][1], a[i].x, b[j].x);
          dmma884(cr[i][j][0], cr[i][j][1], -a[i].y, b[j].y);
          dmma884(ci[i][j][0], ci[i][j][1], a[i].x, b[j].y);
          dmma884(ci[i][j][0], ci[i][j][1], a[i].y, b[j].x);
        }
    }
  }
  __device__ __forceinline__ void store(double2* C, int lane, bool neg, int ldc = BLK_LD) const {
    const double sg = neg ? -1.0 : 1.0;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          C[i * 8 + (lane >> 2) + (j * 8 + 2 * (lane & 3) + e) * ldc] = make_double2(sg * cr[i][j][e], sg * ci[i][j][e]);
  }
};

// Single precision has no exact tensor-core path: the same block product on the FP32 pipe, each
// lane computing the 8 outputs it would hold as DMMA accumulators.
template <typename T> struct BlockAccSimt {
  T c[2][2][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) c[i][j][0] = c[i][j][1] = dpp::zero<T>();
  }
  __device__ __forceinline__ void mma(const T* A, const T* B, int lane, int lda = BLK_LD, int ldb = BLK_LD) {
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      T a[2], b[2][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = A[i * 8 + (lane >> 2) + k * lda];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) b[j][e] = B[k + (j * 8 + 2 * (lane & 3) + e) * ldb];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) c[i][j][e] = madd(c[i][j][e], a[i], b[j][e]);
    }
  }
  __device__ __forceinline__ void store(T* C, int lane, bool ng, int ldc = BLK_LD) const {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          C[i * 8 + (lane >> 2) + (j * 8 + 2 * (lane & 3) + e) * ldc] = ng ? neg(c[i][j][e]) : c[i][j][e];
  }
  __device__ __forceinline__ void load(const T* C, int lane, int ldc = BLK_LD) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) c[i][j][e] = C[i * 8 + (lane >> 2) + (j * 8 + 2 * (lane & 3) + e) * ldc];
  }
};
template <> struct BlockAcc16<float> : BlockAccSimt<float> {};
template <> struct BlockAcc16<float2> : BlockAccSimt<float2> {};

// X = L^{-1} for a lower-triangular L (unit or not) of order 16*nblk; X block-packed in smem, L
// given by a block accessor Lblk(I, K) -> pointer to its 16x16 block (I >= K), element (i, k) at
// [i + k * ldl].  Tb: scratch for (nblk - 1) 16x16 blocks.  All NT threads participate.  X (and
// Tb) blocks: column pitch xld, xld * 16 elements per block (bp's layout by default).
template <typename T, bool UNIT, int NT, class LBlk>
__device__ void tri_inverse_lower_g(LBlk Lblk_of, int ldl, T* Xb, T* Tb, int nblk, int xld = BLK_LD) {
  const int xsz = 16 * xld;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARPS = NT / 32;
  // diagonal blocks: warp w inverts block w; lane c < 16 forms column c of the inverse by forward
  // substitution in column (axpy) order -- after x[l] is final it is eliminated from all later
  // rows at once, so the dependent chain is 16 steps long, not 120
  for (int I = warp; I < nblk; I += NWARPS) {
    if (lane < 16) {
      const int c = lane;
      const T* Lblk = Lblk_of(I, I);
      T x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = (i == c) ? make_real(1.0, zero<T>()) : zero<T>();
#pragma unroll
      for (int l = 0; l < 16; ++l) {
        if (!UNIT) x[l] = mul(x[l], recip(Lblk[l + l * ldl]));
#pragma unroll
        for (int i = l + 1; i < 16; ++i) x[i] = fms(x[i], Lblk[i + l * ldl], x[l]);
      }
      T* Xblk = Xb + (I * (I + 1) / 2 + I) * xsz;
#pragma unroll
      for (int i = 0; i < 16; ++i) Xblk[i + c * xld] = x[i];
    }
  }
  __syncthreads();
  // off-diagonal blocks, by block diagonals d = I - J (plain triangular inversion):
  //   X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ
  // one warp per block, both 16x16x16 products on the FP64 tensor pipe (DMMA.8x8x4)
  for (int d = 1; d < nblk; ++d) {
    for (int q = warp; q + d < nblk; q += NWARPS) {
      const int I = d + q, J = q;
      BlockAcc16<T> acc;
      acc.zero();
      for (int K = J; K < I; ++K) acc.mma(Lblk_of(I, K), Xb + (K * (K + 1) / 2 + J) * xsz, lane, ldl, xld);
      T* Tq = Tb + q * xsz;
      acc.store(Tq, lane, false, xld);
      __syncwarp();
      BlockAcc16<T> acc2;
      acc2.zero();
      acc2.mma(Xb + (I * (I + 1) / 2 + I) * xsz, Tq, lane, xld, xld);
      acc2.store(Xb + (I * (I + 1) / 2 + J) * xsz, lane, true, xld);
      __syncwarp();
    }
    __syncthreads();
  }
}

// the same with L block-packed in smem
template <typename T, bool UNIT, int NT>
__device__ void tri_inverse_lower(const T* Lb, T* Xb, T* Tb, int nblk) {
  tri_inverse_lower_g<T, UNIT, NT>([=](int I, int K) { return Lb + (I * (I + 1) / 2 + K) * BLK_SZ; }, BLK_LD, Xb,
                                   Tb, nblk);
}

}  // namespace dpp
