// update.cu -- Stage 3 (and stage-2 GEMMs): C -= A op(B)^T on FP64 tensor cores -- generic path.
//
// Listing 3:  A_{J2} -= A_{J2,J1} A_{J1,J2}.  "Asymptotically, all of the
// work is performed in the outer-product updates which form the Schur complements"
// (PAPER.md:608-609).  Hermitian specialisation:
//   A22 -= L21 D1 L21^H   on the lower triangle only   (B = L21, scaled by D1 on the fly)
// Non-Hermitian (LU):
//   A22 -= L21 U12.
// The same contraction, with the small operators of diag.cu, performs the panel solves of stage 2.
//
// This file holds the launcher and the cp.async-fed fallback kernel used when an operand is not
// 16-byte aligned (real matrices with odd ld).  The fast path is update_ws.cu.  sm_100a has no
// tcgen05 kind::f64, so the FP64 tensor path is the warp-level DMMA.8x8x4 (mma.sync m8n8k4 f64),
// measured at 37.1 TFLOP/s on this part (profiles/r01_fp64_peak.jsonl).  Complex products are
// 4 real DMMAs each (no 3M trick: keeps the textbook rounding and the paper's flop count).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "update_common.cuh"

namespace dpp {

template <bool CPLX> struct Cfg;
template <> struct Cfg<false> { static constexpr int BM = 128, BN = 128, WM = 2, WN = 4, KC = 8, STAGES = 4; };
template <> struct Cfg<true> { static constexpr int BM = 64, BN = 64, WM = 2, WN = 4, KC = 8, STAGES = 4; };

template <bool CPLX, bool BNMAJ>
struct Layout {
  using C = Cfg<CPLX>;
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr int PAD = CPLX ? 2 : 4;
  static constexpr int LDA = C::BM + PAD;
  static constexpr int LDBK = C::BN + PAD;
  static constexpr int LDBN = C::KC + PAD;
  static constexpr int A_ELEMS = C::KC * LDA;
  static constexpr int B_ELEMS = BNMAJ ? C::BN * LDBN : C::KC * LDBK;
  static constexpr int D_ELEMS = (C::KC * 8 + ES - 1) / ES;  // per-k scale of B (doubles)
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS + D_ELEMS;
  static constexpr size_t RING = (size_t)STAGE_ELEMS * C::STAGES * ES;
  static constexpr int LDC = CPLX ? C::BM + 1 : C::BM + 2;
  static constexpr size_t SMEM = RING + (size_t)C::BN * LDC * ES;
};

template <bool CPLX, bool BNMAJ, bool SCALE, bool VEC>
__device__ __forceinline__ void load_stage(typename Elem<CPLX>::T* As, const typename Elem<CPLX>::T* Ag,
                                           const typename Elem<CPLX>::T* Bg, const double* dsc, const UpdateArgs& a,
                                           int grow0, int gcol0, int k0) {
  using T = typename Elem<CPLX>::T;
  using C = Cfg<CPLX>;
  using LY = Layout<CPLX, BNMAJ>;
  constexpr int NT = C::WM * C::WN * 32;
  constexpr int EPC = (CPLX || VEC) ? (16 / sizeof(T)) : 1;  // elements per copy
  const int tid = threadIdx.x;
  T* Bs = As + LY::A_ELEMS;
  if (SCALE && tid < C::KC) {
    double* Ds = reinterpret_cast<double*>(Bs + LY::B_ELEMS);
    Ds[tid] = (k0 + tid < a.K) ? dsc[k0 + tid] : 0.0;
  }
  {
    constexpr int PER_K = C::BM / EPC;
    for (int idx = tid; idx < C::KC * PER_K; idx += NT) {
      const int kk = idx / PER_K, r = (idx % PER_K) * EPC;
      const int gk = k0 + kk, gr = grow0 + r;
      int valid = (gk < a.K) ? min(EPC, a.a_rows - gr) : 0;
      if (valid < 0) valid = 0;
      const T* src = valid > 0 ? Ag + gr + (int64_t)gk * a.lda : Ag;
      if (EPC * sizeof(T) == 16) cp_async16(As + kk * LY::LDA + r, src, valid * (int)sizeof(T));
      else cp_async8(As + kk * LY::LDA + r, src, valid * (int)sizeof(T));
    }
  }
  if (!BNMAJ) {
    constexpr int PER_K = C::BN / EPC;
    for (int idx = tid; idx < C::KC * PER_K; idx += NT) {
      const int kk = idx / PER_K, c = (idx % PER_K) * EPC;
      const int gk = k0 + kk, gc = gcol0 + c;
      int valid = (gk < a.K) ? min(EPC, a.b_rows - gc) : 0;
      if (valid < 0) valid = 0;
      const T* src = valid > 0 ? Bg + gc + (int64_t)gk * a.ldb : Bg;
      if (EPC * sizeof(T) == 16) cp_async16(Bs + kk * LY::LDBK + c, src, valid * (int)sizeof(T));
      else cp_async8(Bs + kk * LY::LDBK + c, src, valid * (int)sizeof(T));
    }
  } else {
    constexpr int PER_N = C::KC / EPC;
    for (int idx = tid; idx < C::BN * PER_N; idx += NT) {
      const int c = idx / PER_N, kk = (idx % PER_N) * EPC;
      const int gk = k0 + kk, gc = gcol0 + c;
      int valid = (gc < a.b_rows) ? min(EPC, a.K - gk) : 0;
      if (valid < 0) valid = 0;
      const T* src = valid > 0 ? Bg + gk + (int64_t)gc * a.ldb : Bg;
      if (EPC * sizeof(T) == 16) cp_async16(Bs + c * LY::LDBN + kk, src, valid * (int)sizeof(T));
      else cp_async8(Bs + c * LY::LDBN + kk, src, valid * (int)sizeof(T));
    }
  }
}

template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ, bool VEC>
__global__ void __launch_bounds__(Cfg<CPLX>::WM * Cfg<CPLX>::WN * 32, 1) update_kernel(const UpdateArgs a) {
  using T = typename Elem<CPLX>::T;
  using C = Cfg<CPLX>;
  using LY = Layout<CPLX, BNMAJ>;
  constexpr int NT = C::WM * C::WN * 32;
  constexpr int TM = C::BM / C::WM, TN = C::BN / C::WN, MI = TM / 8, NI = TN / 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);
  T* Cs = reinterpret_cast<T*>(smem_raw + LY::RING);

  const int tiles_per_sample = a.tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  const TileInfo ti = tile_info<C::BM, C::BN>(a, blockIdx.x, tiles_per_sample, MASK);
  if (!ti.valid) return;
  const T* Ag = reinterpret_cast<const T*>(a.Aop) + (int64_t)ti.s * a.strideA;
  const T* Bg = reinterpret_cast<const T*>(a.Bop) + (int64_t)ti.s * a.strideB;
  T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)ti.s * a.strideC;
  const double* dsc = SCALE ? a.dscale + (int64_t)ti.s * a.dstride : nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WM, wn = warp / C::WM;

  MmaAcc<CPLX, MI, NI> acc;
  acc.zero();
  const int nchunks = (a.K + C::KC - 1) / C::KC;
#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    if (st < nchunks) {
      T* As = sm + st * LY::STAGE_ELEMS;
      load_stage<CPLX, BNMAJ, SCALE, VEC>(As, Ag, Bg, dsc, a, ti.grow0, ti.gcol0, st * C::KC);
    }
    cp_async_commit();
  }
  for (int kc = 0; kc < nchunks; ++kc) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kc + C::STAGES - 1;
      if (nk < nchunks) {
        T* As = sm + (nk % C::STAGES) * LY::STAGE_ELEMS;
        load_stage<CPLX, BNMAJ, SCALE, VEC>(As, Ag, Bg, dsc, a, ti.grow0, ti.gcol0, nk * C::KC);
      }
      cp_async_commit();
    }
    const T* As = sm + (kc % C::STAGES) * LY::STAGE_ELEMS;
    mma_chunk<CPLX, BNMAJ, SCALE, CONJ, C::KC, MI, NI, LY::LDA, LY::LDBK, LY::LDBN>(
        acc, As, As + LY::A_ELEMS, reinterpret_cast<const double*>(As + LY::A_ELEMS + LY::B_ELEMS), wm * TM,
        wn * TN, lane);
  }
  cp_async_wait<0>();
  __syncthreads();
  // epilogue: C tile -> smem, subtract, write back (Hermitian: never above the diagonal)
  for (int idx = tid; idx < ti.ncols * ti.nrows; idx += NT) {
    const int c = idx / ti.nrows, r = idx % ti.nrows;
    Cs[c * LY::LDC + r] = Cg[ti.grow0 + r + (ti.gcol0 + c - ti.cshift) * a.ldc];
  }
  __syncthreads();
  acc.template subtract_into<MASK, TM, TN, LY::LDC>(Cs, wm, wn, lane, ti);
  __syncthreads();
  for (int idx = tid; idx < ti.ncols * ti.nrows; idx += NT) {
    const int c = idx / ti.nrows, r = idx % ti.nrows;
    if (!MASK || ti.grow0 + r >= ti.gcol0 + c) Cg[ti.grow0 + r + (ti.gcol0 + c - ti.cshift) * a.ldc] = Cs[c * LY::LDC + r];
  }
}

template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ, bool VEC>
static cudaError_t launch_generic(UpdateArgs a, cudaStream_t s) {
  using C = Cfg<CPLX>;
  a.tiles_m = (a.rows + C::BM - 1) / C::BM;
  if (a.bcc_P == 0) a.tiles_n = (a.cols + C::BN - 1) / C::BN;
  const long long per = a.tri ? (long long)a.tiles_m * (a.tiles_m + 1) / 2 : (long long)a.tiles_m * a.tiles_n;
  if (per * a.batch <= 0) return cudaSuccess;
  const size_t smem = Layout<CPLX, BNMAJ>::SMEM;
  auto* fn = update_kernel<CPLX, BNMAJ, MASK, SCALE, CONJ, VEC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)(per * a.batch), C::WM * C::WN * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ>
cudaError_t launch_update_ws_t(UpdateArgs a, cudaStream_t s);

// W(i, k) = L(i, k) * d[k] for i < rows, k < cols: the pre-scaled panel W21 = L21 D1 of the
// Hermitian trailing update (A operand), so the DMMA loop needs no per-k scaling.
template <typename T>
__global__ void __launch_bounds__(256) scale_cols_kernel(const T* L, int64_t ldl, int64_t strideL, T* W, int64_t ldw,
                                                         int64_t strideW, const double* d, int64_t strideD, int rows,
                                                         int cols) {
  const int s = blockIdx.z, k = blockIdx.y;
  const double dk = d[(int64_t)s * strideD + k];
  const T* src = L + (int64_t)s * strideL + (int64_t)k * ldl;
  T* dst = W + (int64_t)s * strideW + (int64_t)k * ldw;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < rows; i += gridDim.x * 256) dst[i] = scal(src[i], dk);
}

cudaError_t launch_scale_cols(Kind kind, const void* L, int64_t ldl, int64_t strideL, void* W, int64_t ldw,
                              int64_t strideW, const double* d, int64_t strideD, int rows, int cols, int batch,
                              cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((rows + 255) / 256, 16), cols, batch);
#define DPP_SC(T) scale_cols_kernel<T><<<grid, 256, 0, s>>>(reinterpret_cast<const T*>(L), ldl, strideL, \
      reinterpret_cast<T*>(W), ldw, strideW, d, strideD, rows, cols)
  switch (kind) {
    case HERM_D: DPP_SC(double); break;
    case HERM_Z: case LU_Z: DPP_SC(double2); break;
    case HERM_S: DPP_SC(float); break;
    case LU_C: DPP_SC(float2); break;
  }
#undef DPP_SC
  return cudaGetLastError();
}

// dst <- src for columns [c0, c1) of `batch` n x n column-major matrices; lower = true copies only
// rows >= column (the part a Hermitian sampler reads).  Persistent warps walk (sample, column)
// items; each warp moves one column with four 16-byte loads in flight per lane (the one-CTA-per-
// column kernel it replaces wrote the UST batch's 40 GB at 3.6 TB/s).  V = 16-byte vectors when
// both sides are 16-byte aligned (ld, stride, base), else one element per access.
template <typename T, bool V>
__global__ void __launch_bounds__(256) copy_matrix_kernel(const T* src, int64_t lds, int64_t strideS, T* dst,
                                                          int64_t ldd, int64_t strideD, int n, int c0, int ncols,
                                                          int batch, bool lower) {
  constexpr int E = V ? 16 / (int)sizeof(T) : 1;  // elements per access
  const int lane = threadIdx.x & 31;
  const int64_t items = (int64_t)ncols * batch;
  for (int64_t it = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); it < items; it += (int64_t)gridDim.x * 8) {
    const int64_t s = it / ncols;
    const int j = c0 + (int)(it % ncols);
    const T* a = src + s * strideS + (int64_t)j * lds;
    T* b = dst + s * strideD + (int64_t)j * ldd;
    int i0 = lower ? j : 0;
    if (V) {  // scalar head up to the first 16-byte boundary (same offset on both sides)
      const int head = min(n - i0, (int)((E - (i0 % E)) % E));
      if (lane < head) b[i0 + lane] = a[i0 + lane];
      i0 += head;
      const int nv = (n - i0) / E;
      const uint4* av = reinterpret_cast<const uint4*>(a + i0);
      uint4* bv = reinterpret_cast<uint4*>(b + i0);
      int v = lane;
      for (; v + 96 < nv; v += 128) {
        const uint4 x0 = av[v], x1 = av[v + 32], x2 = av[v + 64], x3 = av[v + 96];
        bv[v] = x0; bv[v + 32] = x1; bv[v + 64] = x2; bv[v + 96] = x3;
      }
      for (; v < nv; v += 32) bv[v] = av[v];
      for (int i = i0 + nv * E + lane; i < n; i += 32) b[i] = a[i];
    } else {
      for (int i = i0 + lane; i < n; i += 32) b[i] = a[i];
    }
  }
}

cudaError_t launch_copy_matrix(size_t es, const void* src, int64_t lds, int64_t strideS, void* dst, int64_t ldd,
                               int64_t strideD, int n, int batch, bool lower, cudaStream_t s, int c0, int c1) {
  if (c1 < 0 || c1 > n) c1 = n;
  if (n <= 0 || batch <= 0 || c0 >= c1) return cudaSuccess;
  const int ncols = c1 - c0;
  const bool v = reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0 &&
                 (lds * (int64_t)es) % 16 == 0 && (ldd * (int64_t)es) % 16 == 0 &&
                 (strideS * (int64_t)es) % 16 == 0 && (strideD * (int64_t)es) % 16 == 0;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t items = (int64_t)ncols * batch;
  const int64_t grid = std::min<int64_t>((items + 7) / 8, (int64_t)sms * 8);
#define DPP_CP(T)                                                                                             \
  do {                                                                                                        \
    if (v)                                                                                                    \
      copy_matrix_kernel<T, true><<<(unsigned)grid, 256, 0, s>>>(reinterpret_cast<const T*>(src), lds, strideS, \
          reinterpret_cast<T*>(dst), ldd, strideD, n, c0, ncols, batch, lower);                               \
    else                                                                                                      \
      copy_matrix_kernel<T, false><<<(unsigned)grid, 256, 0, s>>>(reinterpret_cast<const T*>(src), lds, strideS, \
          reinterpret_cast<T*>(dst), ldd, strideD, n, c0, ncols, batch, lower);                               \
  } while (0)
  if (es == 4) DPP_CP(float);
  else if (es == 8) DPP_CP(double);
  else DPP_CP(double2);
#undef DPP_CP
  return cudaGetLastError();
}

// 32 x 32 tiles through shared memory: coalesced 16-byte reads of src columns and dst columns.
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T* src, int64_t lds, int64_t strideS, T* dst,
                                                        int64_t ldd, int64_t strideD, int rows, int cols) {
  __shared__ T t[32][33];
  const int s = blockIdx.z;
  const int k0 = blockIdx.x * 32, j0 = blockIdx.y * 32;  // src rows k (< rows), src cols j (< cols)
  const T* S = src + (int64_t)s * strideS;
  T* D = dst + (int64_t)s * strideD;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int jj = ty; jj < 32; jj += 8) {
    const int k = k0 + tx, j = j0 + jj;
    if (k < rows && j < cols) t[jj][tx] = S[k + (int64_t)j * lds];
  }
  __syncthreads();
  for (int kk = ty; kk < 32; kk += 8) {
    const int j = j0 + tx, k = k0 + kk;
    if (k < rows && j < cols) D[j + (int64_t)k * ldd] = t[tx][kk];
  }
}

cudaError_t launch_transpose(size_t es, const void* src, int64_t lds, int64_t strideS, void* dst, int64_t ldd,
                             int64_t strideD, int rows, int cols, int batch, cudaStream_t s) {
  if (rows <= 0 || cols <= 0 || batch <= 0) return cudaSuccess;
  dim3 grid((rows + 31) / 32, (cols + 31) / 32, batch);
  if (es == 16)
    transpose_kernel<double2><<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(src), lds, strideS,
                                                   reinterpret_cast<double2*>(dst), ldd, strideD, rows, cols);
  else
    transpose_kernel<float2><<<grid, 256, 0, s>>>(reinterpret_cast<const float2*>(src), lds, strideS,
                                                  reinterpret_cast<float2*>(dst), ldd, strideD, rows, cols);
  return cudaGetLastError();
}

// Dispatch on (kind, operand layout, flags).  Fast path: update_ws.cu (persistent,
// warp-specialized, TMA-fed) for 16-byte-aligned operands; this file's cp.async kernel otherwise.
static cudaError_t launch_update_core(Kind kind, UpdateArgs a, cudaStream_t s, bool ws);

cudaError_t launch_update(Kind kind, UpdateArgs a, cudaStream_t s) {
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  const bool ws = a.vec && !a.generic && kind != HERM_S && kind != LU_C;
  // a separate C source is read only by the warp-specialized kernel (16-byte aligned, no bcc)
  if (a.csrc && (!ws || a.bcc_P > 0 || reinterpret_cast<uintptr_t>(a.csrc) % 16 || (a.ldcs * kind_esize(kind)) % 16 ||
                 (a.strideCs * kind_esize(kind)) % 16))
    return cudaErrorInvalidValue;
  // the second output W: fused into the warp-specialized panel kernel (no mask, Hermitian) or the
  // 3xTF32 kernel's epilogue (real single precision), else a column-scaling pass over the region
  const bool tc32 = kind == HERM_S && a.vec && !a.generic && !a.fp32_simt && !a.dscale && !a.conj && !a.bnmajor &&
                    a.batch == 1 && a.bcc_P == 0 && a.tcs &&
                    a.tcs_bytes >= (int64_t)tc32_scratch_bytes(a.rows, a.cols, a.K, false);
  const bool fuse = a.wout && !a.mask && a.bcc_P == 0 && ((ws && (kind == HERM_D || kind == HERM_Z)) || tc32);
  UpdateArgs k = a;
  if (!fuse) k.wout = nullptr;
  cudaError_t e = launch_update_core(kind, k, s, ws);
  if (e == cudaSuccess && a.wout && !fuse) {
    const size_t es = kind_esize(kind);
    e = launch_scale_cols(kind, reinterpret_cast<const char*>(a.C) + (size_t)(a.row0 + (int64_t)a.col0 * a.ldc) * es,
                          a.ldc, a.strideC,
                          reinterpret_cast<char*>(a.wout) + (size_t)(a.row0 + (int64_t)a.col0 * a.ldw) * es, a.ldw,
                          a.strideWo, a.wscale + a.col0, a.wsstride, a.rows, a.cols, a.batch, s);
  }
  return e;
}

static cudaError_t launch_update_core(Kind kind, UpdateArgs a, cudaStream_t s, bool ws) {
  // single precision: tcgen05 3xTF32 for aligned operands of one sample (update_tc32.cu), else FP32 SIMT
  if ((kind == HERM_S || (kind == LU_C && !a.mask)) && a.vec && !a.generic && !a.fp32_simt && !a.dscale && !a.conj &&
      !a.bnmajor && a.batch == 1 && a.bcc_P == 0 && a.tcs &&
      a.tcs_bytes >= (int64_t)tc32_scratch_bytes(a.rows, a.cols, a.K, kind == LU_C))
    return launch_update_tc32(a, s, kind == LU_C);
  if (kind == HERM_S || kind == LU_C) return launch_update_simt(kind, a, s);
  const bool scale = a.dscale != nullptr;
#define DPP_GO(CP, BN_, MK, SC, CJ)                                         \
  return ws ? launch_update_ws_t<CP, BN_, MK, SC, CJ>(a, s)                \
            : (a.vec ? launch_generic<CP, BN_, MK, SC, CJ, true>(a, s)     \
                     : launch_generic<CP, BN_, MK, SC, CJ, false>(a, s))
  if (kind == HERM_D) {
    if (a.bnmajor || a.conj) return cudaErrorInvalidValue;
    if (a.mask && scale) DPP_GO(false, false, true, true, false);      // trailing update, B scaled by D1
    if (a.mask && !scale) DPP_GO(false, false, true, false, false);    // trailing update, A = W21
    if (!a.mask && !scale) DPP_GO(false, false, false, false, false);  // panel GEMM
  } else if (kind == HERM_Z) {
    if (a.bnmajor) return cudaErrorInvalidValue;
    if (a.mask && scale && a.conj) DPP_GO(true, false, true, true, true);
    if (a.mask && !scale && a.conj) DPP_GO(true, false, true, false, true);
    if (!a.mask && !scale && a.conj) DPP_GO(true, false, false, false, true);  // L-ensemble: B conjugated
    if (!a.mask && !scale && !a.conj) DPP_GO(true, false, false, false, false);
  } else {
    if (a.mask || scale || a.conj) return cudaErrorInvalidValue;
    if (a.bnmajor) DPP_GO(true, true, false, false, false);  // trailing update, row panel
    DPP_GO(true, false, false, false, false);                // column panel
  }
#undef DPP_GO
  return cudaErrorInvalidValue;
}

}  // namespace dpp
