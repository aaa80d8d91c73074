// update_simt.cu -- Stage 3 (and the stage-2 GEMMs) of the SINGLE-PRECISION samplers (SURVEY §8(f)
// rank 2; the paper's single-precision runs): C -= A op(B)^T, the same
// operation and UpdateArgs contract as update.cu / update_ws.cu (Listing 3,
// PAPER.md:586; Hermitian: A22 -= W21 L21^H on the lower triangle, LU: A22 -= L21 U12).
//
// sm_100a has no exact-fp32 tensor-core MMA (kind::tf32 rounds the operands to 10 mantissa bits),
// so single precision runs on the FP32 SIMT pipe (FFMA: 148 SMs x 128 lanes x 2 flop x 1.965 GHz =
// 74.4 TFLOP/s): a register-blocked outer-product kernel --
//   * one CTA of 256 threads per 128x128 (real) / 64x64 (complex) tile, 8x8 (4x4 complex) outputs
//     per thread in registers, split in two 4-row/4-column halves 64 (32) apart so the fragment
//     loads are 16-byte vector loads from conflict-free shared-memory rows;
//   * K-chunks of 16 (8 complex) double-buffered in shared memory with cp.async;
//   * epilogue: read-modify-write of C straight from the registers (masked to the lower triangle for
//     Hermitian diagonal tiles).
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "update_common.cuh"

namespace dpp {

template <typename T> struct SimtCfg;
template <> struct SimtCfg<float> { static constexpr int BM = 128, BN = 128, TM = 8, TN = 8, KC = 16; };
template <> struct SimtCfg<float2> { static constexpr int BM = 64, BN = 64, TM = 4, TN = 4, KC = 8; };

__device__ __forceinline__ void cfma(float& c, float a, float b) { c = fmaf(a, b, c); }

template <typename T, bool MASK, bool CONJ>
__global__ void __launch_bounds__(256) update_simt_kernel(const UpdateArgs a) {
  using C = SimtCfg<T>;
  constexpr bool CPLX = sizeof(T) == 8;
  constexpr int BM = C::BM, BN = C::BN, TM = C::TM, TN = C::TN, KC = C::KC;
  constexpr int HM = TM / 2, HN = TN / 2;  // each thread: rows {ty*HM + r, BM/2 + ty*HM + r}
  __shared__ __align__(16) T As[2][KC][BM];
  __shared__ __align__(16) T Bs[2][KC][BN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int tiles_per_sample = a.tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  const int ntiles = tiles_per_sample * a.batch;
  const int nchunks = (a.K + KC - 1) / KC;
  constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte copy
  const bool vec = a.vec != 0;

  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const TileInfo ti = tile_info<BM, BN>(a, t, tiles_per_sample, MASK);
    if (!ti.valid) continue;
    const T* Ag = reinterpret_cast<const T*>(a.Aop) + (int64_t)ti.s * a.strideA;
    const T* Bg = reinterpret_cast<const T*>(a.Bop) + (int64_t)ti.s * a.strideB;
    T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)ti.s * a.strideC;

    auto load = [&](int buf, int k0) {
      // A: KC x BM, B: KC x BN; rows beyond the operand / k beyond K are zero-filled
      for (int idx = tid; idx < KC * (BM / EPV); idx += 256) {
        const int kk = idx / (BM / EPV), r = (idx % (BM / EPV)) * EPV;
        const int gk = k0 + kk, gr = ti.grow0 + r;
        if (vec) {
          int valid = gk < a.K ? min(EPV, a.a_rows - gr) : 0;
          valid = max(valid, 0);
          cp_async16(&As[buf][kk][r], valid > 0 ? Ag + gr + (int64_t)gk * a.lda : Ag, valid * (int)sizeof(T));
        } else {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            As[buf][kk][r + e] = (gk < a.K && gr + e < a.a_rows) ? Ag[gr + e + (int64_t)gk * a.lda] : T{};
        }
      }
      for (int idx = tid; idx < KC * (BN / EPV); idx += 256) {
        const int kk = idx / (BN / EPV), c = (idx % (BN / EPV)) * EPV;
        const int gk = k0 + kk, gc = ti.gcol0 + c;
        if (vec) {
          int valid = gk < a.K ? min(EPV, a.b_rows - gc) : 0;
          valid = max(valid, 0);
          cp_async16(&Bs[buf][kk][c], valid > 0 ? Bg + gc + (int64_t)gk * a.ldb : Bg, valid * (int)sizeof(T));
        } else {
#pragma unroll
          for (int e = 0; e < EPV; ++e)
            Bs[buf][kk][c + e] = (gk < a.K && gc + e < a.b_rows) ? Bg[gc + e + (int64_t)gk * a.ldb] : T{};
        }
      }
    };

    float acc[TM][TN][CPLX ? 2 : 1];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int e = 0; e < (CPLX ? 2 : 1); ++e) acc[i][j][e] = 0.f;

    load(0, 0);
    cp_async_commit();
    for (int kc = 0; kc < nchunks; ++kc) {
      const int buf = kc & 1;
      if (kc + 1 < nchunks) load(buf ^ 1, (kc + 1) * KC);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        T av[TM], bv[TN];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int r = 0; r < HM; ++r) av[h * HM + r] = As[buf][kk][h * (BM / 2) + ty * HM + r];
#pragma unroll
          for (int c = 0; c < HN; ++c) bv[h * HN + c] = Bs[buf][kk][h * (BN / 2) + tx * HN + c];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            if constexpr (!CPLX) {
              cfma(acc[i][j][0], av[i], bv[j]);
            } else {
              // a * op(b), op = conj for the Hermitian update
              const float ar = reinterpret_cast<const float2&>(av[i]).x, ai = reinterpret_cast<const float2&>(av[i]).y;
              const float br = reinterpret_cast<const float2&>(bv[j]).x;
              const float bi = CONJ ? -reinterpret_cast<const float2&>(bv[j]).y : reinterpret_cast<const float2&>(bv[j]).y;
              cfma(acc[i][j][0], ar, br);
              cfma(acc[i][j][0], -ai, bi);
              cfma(acc[i][j][1], ar, bi);
              cfma(acc[i][j][1], ai, br);
            }
          }
      }
      __syncthreads();
    }
    cp_async_wait<0>();
    // epilogue: C -= acc (Hermitian: never above the diagonal)
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = (i / HM) * (BM / 2) + ty * HM + (i % HM);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = (j / HN) * (BN / 2) + tx * HN + (j % HN);
        if (r < ti.nrows && c < ti.ncols && (!MASK || ti.grow0 + r >= ti.gcol0 + c)) {
          T* p = Cg + ti.grow0 + r + (int64_t)(ti.gcol0 + c - ti.cshift) * a.ldc;
          if constexpr (!CPLX) {
            *p = *p - acc[i][j][0];
          } else {
            float2 v = *reinterpret_cast<float2*>(p);
            v.x -= acc[i][j][0];
            v.y -= acc[i][j][1];
            *reinterpret_cast<float2*>(p) = v;
          }
        }
      }
    }
  }
}

template <typename T, bool MASK, bool CONJ>
static cudaError_t launch_simt_t(UpdateArgs a, cudaStream_t s) {
  using C = SimtCfg<T>;
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  a.tiles_m = (a.rows + C::BM - 1) / C::BM;
  if (a.bcc_P == 0) a.tiles_n = (a.cols + C::BN - 1) / C::BN;
  const long long per = a.tri ? (long long)a.tiles_m * (a.tiles_m + 1) / 2 : (long long)a.tiles_m * a.tiles_n;
  const long long total = per * a.batch;
  if (total <= 0) return cudaSuccess;
  long long g = total;
  if (a.grid_limit > 0 && g > (long long)a.grid_limit * 2) g = (long long)a.grid_limit * 2;  // 2 CTAs per SM
  update_simt_kernel<T, MASK, CONJ><<<(unsigned)g, 256, 0, s>>>(a);
  return cudaGetLastError();
}

// Dispatch for the single-precision kinds (mirrors launch_update's operand conventions).
cudaError_t launch_update_simt(Kind kind, UpdateArgs a, cudaStream_t s) {
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  if (a.dscale || a.bnmajor) return cudaErrorInvalidValue;  // pre-scaled / K-major operands only
  if (kind == HERM_S) {
    if (a.conj) return cudaErrorInvalidValue;
    return a.mask ? launch_simt_t<float, true, false>(a, s) : launch_simt_t<float, false, false>(a, s);
  }
  if (kind == LU_C) {
    if (a.mask || a.conj) return cudaErrorInvalidValue;
    return launch_simt_t<float2, false, false>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dpp
