// update_simt.cu -- Stage 3 (and the stage-2 GEMMs) of the SINGLE-PRECISION samplers (SURVEY §8(f)
// rank 2; the paper's single-precision runs): C -= A op(B)^T, the same
// operation and UpdateArgs contract as update.cu / update_ws.cu (Listing 3,
// PAPER.md:586; Hermitian: A22 -= W21 L21^H on the lower triangle, LU: A22 -= L21 U12).
//
// sm_100a has no exact-fp32 tensor-core MMA (kind::tf32 rounds the operands to 10 mantissa bits),
// so single precision runs on the FP32 SIMT pipe (FFMA: 148 SMs x 128 lanes x 2 flop x 1.965 GHz =
// 74.4 TFLOP/s): a register-blocked outer-product kernel --
//   * one CTA of 512 threads (4 warps per SM sub-partition) per 256x128 (real) / 128x64 (complex)
//     tile, 8x8 (4x4 complex) outputs per thread in registers, split in two halves so the fragment
//     loads are 16-byte vector loads;
//   * persistent CTAs (one per SM, the SMs of the lookahead stream left free); K-chunks of 32 (16
//     complex) double-buffered in shared memory with cp.async, the first chunk of the next tile
//     prefetched while the last one of the current tile is consumed;
//   * epilogue: read-modify-write of C straight from the registers with 16-byte accesses (masked to
//     the lower triangle on Hermitian diagonal tiles).
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "update_common.cuh"

namespace dpp {

// 512 threads = 32 (rows) x 16 (columns); each thread TM x TN outputs in two halves of HM x HN.
template <typename T> struct SimtCfg;
template <> struct SimtCfg<float> { static constexpr int BM = 256, BN = 128, TM = 8, TN = 8, KC = 32; };
template <> struct SimtCfg<float2> { static constexpr int BM = 128, BN = 64, TM = 4, TN = 4, KC = 16; };
constexpr int SIMT_NT = 512;

__device__ __forceinline__ void cfma(float& c, float a, float b) { c = fmaf(a, b, c); }

template <typename T, bool MASK, bool CONJ>
__global__ void __launch_bounds__(SIMT_NT, 1) update_simt_kernel(const UpdateArgs a) {
  using C = SimtCfg<T>;
  constexpr bool CPLX = sizeof(T) == 8;
  constexpr int BM = C::BM, BN = C::BN, TM = C::TM, TN = C::TN, KC = C::KC;
  constexpr int HM = TM / 2, HN = TN / 2;  // each thread: rows {tx*HM + r, BM/2 + tx*HM + r}
  // Dynamic shared memory (see launch_simt_t): [2][KC][BM] A stages, [2][KC][BN] B stages.
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T (*As)[KC][BM] = reinterpret_cast<T (*)[KC][BM]>(smem_raw);
  T (*Bs)[KC][BN] = reinterpret_cast<T (*)[KC][BN]>(smem_raw + sizeof(T) * 2 * KC * BM);
  // rows of the register tile from the fast thread index: the epilogue then moves HM contiguous
  // rows (16 bytes) per thread and a warp covers 2 x 256 contiguous bytes per column
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  static_assert(BM == 64 * HM && BN == 32 * HN, "thread grid 32 x 16");
  const int tiles_per_sample = a.tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  const int ntiles = tiles_per_sample * a.batch;
  const int nchunks = (a.K + KC - 1) / KC;
  constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte copy
  const bool vec = a.vec != 0;

  auto load = [&](const TileInfo& ti, int buf, int k0) {
    const T* Ag = reinterpret_cast<const T*>(a.Aop) + (int64_t)ti.s * a.strideA;
    const T* Bg = reinterpret_cast<const T*>(a.Bop) + (int64_t)ti.s * a.strideB;
    // A: KC x BM, B: KC x BN; rows beyond the operand / k beyond K are zero-filled
    for (int idx = tid; idx < KC * (BM / EPV); idx += SIMT_NT) {
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
    for (int idx = tid; idx < KC * (BN / EPV); idx += SIMT_NT) {
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
  auto next_valid = [&](int t) {  // the next tile of this CTA that has work (ntiles if none)
    for (; t < ntiles; t += gridDim.x)
      if (tile_info<BM, BN>(a, t, tiles_per_sample, MASK).valid) return t;
    return ntiles;
  };

  int t = next_valid(blockIdx.x);
  int buf = 0;
  if (t < ntiles) load(tile_info<BM, BN>(a, t, tiles_per_sample, MASK), 0, 0);
  cp_async_commit();
  while (t < ntiles) {
    const TileInfo ti = tile_info<BM, BN>(a, t, tiles_per_sample, MASK);
    const int tn = next_valid(t + gridDim.x);
    float acc[TM][TN][CPLX ? 2 : 1];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
#pragma unroll
        for (int e = 0; e < (CPLX ? 2 : 1); ++e) acc[i][j][e] = 0.f;
    for (int kc = 0; kc < nchunks; ++kc, buf ^= 1) {
      // prefetch the next chunk -- or, after the last one, the first chunk of the next tile
      if (kc + 1 < nchunks) load(ti, buf ^ 1, (kc + 1) * KC);
      else if (tn < ntiles) load(tile_info<BM, BN>(a, tn, tiles_per_sample, MASK), buf ^ 1, 0);
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        T av[TM], bv[TN];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int r = 0; r < HM; ++r) av[h * HM + r] = As[buf][kk][h * (BM / 2) + tx * HM + r];
#pragma unroll
          for (int c = 0; c < HN; ++c) bv[h * HN + c] = Bs[buf][kk][h * (BN / 2) + ty * HN + c];
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
    // epilogue: C -= acc (Hermitian: never above the diagonal).  Per group of HN columns x HM rows:
    // 16-byte accesses when the whole group lies inside the tile and below the diagonal (vec: ldc
    // keeps every column of the group 16-byte aligned like the first), element accesses otherwise.
    // The group's loads are all issued before its stores (a load after a store to the same array
    // waits for it: one serialized global round trip per group, not per column).
    T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)ti.s * a.strideC;
#pragma unroll
    for (int hg = 0; hg < 4; ++hg) {
      const int h = hg >> 1, jg = (hg & 1) * HN;
      const int r0 = h * (BM / 2) + tx * HM;
      const int cb = (hg & 1) * (BN / 2) + ty * HN;  // first column of the group
      T* pb = Cg + ti.grow0 + r0 + (int64_t)(ti.gcol0 + cb - ti.cshift) * a.ldc;
      const bool full = vec && cb + HN <= ti.ncols && r0 + HM <= ti.nrows &&
                        (!MASK || ti.grow0 + r0 >= ti.gcol0 + cb + HN - 1) &&
                        (reinterpret_cast<uintptr_t>(pb) & 15) == 0;
      if (full) {
        float4 cv[HN];
#pragma unroll
        for (int jj = 0; jj < HN; ++jj) cv[jj] = *reinterpret_cast<const float4*>(pb + (int64_t)jj * a.ldc);
#pragma unroll
        for (int jj = 0; jj < HN; ++jj) {
          const int j = jg + jj;
          float4 v = cv[jj];
          if constexpr (!CPLX) {
            v.x -= acc[h * HM + 0][j][0]; v.y -= acc[h * HM + 1][j][0];
            v.z -= acc[h * HM + 2][j][0]; v.w -= acc[h * HM + 3][j][0];
          } else {
            v.x -= acc[h * HM + 0][j][0]; v.y -= acc[h * HM + 0][j][1];
            v.z -= acc[h * HM + 1][j][0]; v.w -= acc[h * HM + 1][j][1];
          }
          *reinterpret_cast<float4*>(pb + (int64_t)jj * a.ldc) = v;
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < HN; ++jj) {
          const int j = jg + jj, c = cb + jj;
          if (c >= ti.ncols) continue;
          T* p = pb + (int64_t)jj * a.ldc;
#pragma unroll
          for (int r = 0; r < HM; ++r) {
            const int rr = r0 + r;
            if (rr < ti.nrows && (!MASK || ti.grow0 + rr >= ti.gcol0 + c)) {
              if constexpr (!CPLX) {
                p[r] = p[r] - acc[h * HM + r][j][0];
              } else {
                float2 v = *reinterpret_cast<float2*>(p + r);
                v.x -= acc[h * HM + r][j][0];
                v.y -= acc[h * HM + r][j][1];
                *reinterpret_cast<float2*>(p + r) = v;
              }
            }
          }
        }
      }
    }
    t = tn;
  }
  cp_async_wait<0>();
}

template <typename T, bool MASK, bool CONJ>
static cudaError_t launch_simt_t(UpdateArgs a, cudaStream_t s) {
  using C = SimtCfg<T>;
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  a.tri = 0;  // rectangular tiles: rectangular enumeration, tiles above the diagonal are skipped
  a.tiles_m = (a.rows + C::BM - 1) / C::BM;
  if (a.bcc_P == 0) a.tiles_n = (a.cols + C::BN - 1) / C::BN;
  const long long per = a.tri ? (long long)a.tiles_m * (a.tiles_m + 1) / 2 : (long long)a.tiles_m * a.tiles_n;
  const long long total = per * a.batch;
  if (total <= 0) return cudaSuccess;
  // One CTA per SM: the operand stages need 32 KB, but the launch asks for 120 KB of dynamic shared
  // memory so that no second CTA (and no diag kernel of the lookahead stream) shares an SM with it;
  // with grid_limit = SMs - R the R reserved SMs then stay free for the sequential chain.
  constexpr size_t SMEM = 120 * 1024;
  static_assert(sizeof(T) * 2 * C::KC * (C::BM + C::BN) <= SMEM, "stages fit");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long g = a.grid_limit > 0 ? a.grid_limit : sms;
  if (g > total) g = total;
  auto* fn = update_simt_kernel<T, MASK, CONJ>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)g, SIMT_NT, SMEM, s>>>(a);
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
