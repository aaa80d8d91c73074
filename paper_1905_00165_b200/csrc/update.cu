// update.cu -- Stage 3: the trailing Schur-complement update on FP64 tensor cores.
//
// Listing 3:  A_{J2} -= A_{J2,J1} A_{J1,J2}.  "Asymptotically, all of the
// work is performed in the outer-product updates which form the Schur complements"
// (PAPER.md:608-609).  Hermitian specialisation:
//   A22 -= L21 W21^H   on the lower triangle only   (W21 = L21 D1 from stage 2)
// Non-Hermitian (LU):
//   A22 -= L21 U12.
//
// B200 design: sm_100a has no tcgen05 kind::f64, so the FP64 tensor path is the warp-level
// DMMA.8x8x4 (mma.sync m8n8k4 f64), measured at 37.1 TFLOP/s on this part
// (profiles/r01_fp64_peak.jsonl).  Operand K-chunks stream from L2/HBM into a STAGES-deep
// cp.async ring in shared memory (padded layouts: conflict-free 64-bit fragment loads); the
// accumulator tile lives in registers; C is prefetched into L2 (cp.async.bulk.prefetch) when the
// CTA starts so the read-modify-write epilogue hits L2.  Complex products are 4 real DMMAs each
// (no 3M trick: keeps the rounding of the textbook product and the paper's flop count).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dpp {

template <bool CPLX> struct Cfg;
// real: CTA 128x128, 8 warps as 2(M) x 4(N), warp tile 64x32, K chunk 8, 4 stages
template <> struct Cfg<false> {
  static constexpr int BM = 128, BN = 128, WM = 2, WN = 4, KC = 8, STAGES = 4;
};
// complex: CTA 64x64, 8 warps as 2 x 4, warp tile 32x16, K chunk 8, 4 stages
template <> struct Cfg<true> {
  static constexpr int BM = 64, BN = 64, WM = 2, WN = 4, KC = 8, STAGES = 4;
};

template <bool CPLX, bool BLU>
struct Layout {
  using C = Cfg<CPLX>;
  static constexpr int ES = CPLX ? 16 : 8;  // element bytes
  // A (and Hermitian B): [KC][BM + PADA]; row = k, BM contiguous elements.  PAD keeps the
  // 16 lanes of a 64-bit (or 8 lanes of a 128-bit) fragment load on distinct banks.
  static constexpr int PAD = CPLX ? 2 : 4;
  static constexpr int LDA = C::BM + PAD;
  static constexpr int LDBK = C::BN + PAD;   // Hermitian B: [KC][BN + PAD]
  static constexpr int LDBN = C::KC + PAD;   // LU B: [BN][KC + PAD]
  static constexpr int A_ELEMS = C::KC * LDA;
  static constexpr int B_ELEMS = BLU ? C::BN * LDBN : C::KC * LDBK;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t RING = (size_t)STAGE_ELEMS * C::STAGES * ES;
  // C tile staged in shared memory, column j at j*LDC: LDC = 130 (real) / 65 (complex) keeps
  // the accumulator-fragment access pattern (8 rows x 4 column pairs per warp) conflict-free
  // and every column 16-byte aligned for the bulk (TMA) copies.
  static constexpr int LDC = CPLX ? C::BM + 1 : C::BM + 2;
  static constexpr size_t CTILE = (size_t)C::BN * LDC * ES;
  static constexpr size_t SMEM = RING + CTILE;
};

template <bool CPLX> struct Elem { using T = double; };
template <> struct Elem<true> { using T = double2; };

template <bool CPLX, bool BLU, bool VEC>
__device__ __forceinline__ void load_stage(typename Elem<CPLX>::T* As, typename Elem<CPLX>::T* Bs,
                                           const typename Elem<CPLX>::T* Ag, const typename Elem<CPLX>::T* Bg,
                                           const UpdateArgs& a, int grow0, int gcol0, int k0) {
  using T = typename Elem<CPLX>::T;
  using C = Cfg<CPLX>;
  using LY = Layout<CPLX, BLU>;
  constexpr int NT = C::WM * C::WN * 32;
  constexpr int EPC = (CPLX || VEC) ? (16 / sizeof(T)) : 1;  // elements per copy
  const int tid = threadIdx.x;
  // A: KC x BM (rows contiguous)
  {
    constexpr int PER_K = C::BM / EPC;
    for (int idx = tid; idx < C::KC * PER_K; idx += NT) {
      const int kk = idx / PER_K, r = (idx % PER_K) * EPC;
      const int gk = k0 + kk, gr = grow0 + r;
      int valid = (gk < a.K) ? min(EPC, a.m_total - gr) : 0;
      if (valid < 0) valid = 0;
      const T* src = valid > 0 ? Ag + gr + (int64_t)gk * a.lda : Ag;
      if (EPC * sizeof(T) == 16) cp_async16(As + kk * LY::LDA + r, src, valid * (int)sizeof(T));
      else cp_async8(As + kk * LY::LDA + r, src, valid * (int)sizeof(T));
    }
  }
  if (!BLU) {
    constexpr int PER_K = C::BN / EPC;
    for (int idx = tid; idx < C::KC * PER_K; idx += NT) {
      const int kk = idx / PER_K, c = (idx % PER_K) * EPC;
      const int gk = k0 + kk, gc = gcol0 + c;
      int valid = (gk < a.K) ? min(EPC, a.m_total - gc) : 0;
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
      int valid = (gc < a.m_total) ? min(EPC, a.K - gk) : 0;
      if (valid < 0) valid = 0;
      const T* src = valid > 0 ? Bg + gk + (int64_t)gc * a.ldb : Bg;
      if (EPC * sizeof(T) == 16) cp_async16(Bs + c * LY::LDBN + kk, src, valid * (int)sizeof(T));
      else cp_async8(Bs + c * LY::LDBN + kk, src, valid * (int)sizeof(T));
    }
  }
}

template <bool CPLX, bool BLU, bool VEC>
__global__ void __launch_bounds__(Cfg<CPLX>::WM * Cfg<CPLX>::WN * 32, 1)
update_kernel(const UpdateArgs a) {
  using T = typename Elem<CPLX>::T;
  using C = Cfg<CPLX>;
  using LY = Layout<CPLX, BLU>;
  constexpr int NT = C::WM * C::WN * 32;
  constexpr int TM = C::BM / C::WM, TN = C::BN / C::WN;  // warp tile
  constexpr int MI = TM / 8, NI = TN / 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);

  // ---- which tile
  int ti, tj;
  if (a.tri) {
    const int t = blockIdx.x;
    int r = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    ti = r;
    tj = t - r * (r + 1) / 2;
  } else {
    ti = blockIdx.x % a.tiles_m;
    tj = blockIdx.x / a.tiles_m;
  }
  const int s = blockIdx.z;
  const int grow0 = a.row0 + ti * C::BM;  // A22-relative
  const int row_end = a.row0 + a.rows;
  int gcol0, col_end;
  int64_t cshift = 0;  // storage column of A22-relative column gc is gc - cshift
  if (a.bcc_P > 0) {
    const int64_t q = a.bcc_q0 + tj;
    const int64_t gcs = (a.bcc_r + q * a.bcc_P) * (int64_t)a.bcc_nb;
    gcol0 = (int)(gcs - a.bcc_j1);
    col_end = min(gcol0 + a.bcc_nb, a.m_total);
    cshift = gcol0 - q * a.bcc_nb;
  } else {
    gcol0 = a.col0 + tj * C::BN;
    col_end = a.col0 + a.cols;
  }
  if (grow0 >= row_end || gcol0 >= col_end) return;
  if (!BLU && gcol0 > grow0 + C::BM - 1) return;  // strictly above the diagonal (Hermitian)

  const T* Ag = reinterpret_cast<const T*>(a.Aop) + (int64_t)s * a.strideA;
  const T* Bg = reinterpret_cast<const T*>(a.Bop) + (int64_t)s * a.strideB;
  T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)s * a.strideC;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WM, wn = warp / C::WM;

  // ---- C tile -> shared memory with TMA bulk copies, issued now, awaited in the epilogue
  __shared__ __align__(8) uint64_t cbar;
  T* Cs = reinterpret_cast<T*>(smem_raw + LY::RING);
  const int nrows = min(C::BM, row_end - grow0);         // rows of this tile inside the region
  const int ncols = min(C::BN, col_end - gcol0);
  const bool diag_tile = !BLU && (gcol0 + ncols - 1 > grow0);  // some element above the diagonal
  const bool bulk = VEC && ((nrows * (int)sizeof(T)) % 16 == 0);
  if (tid == 0) {
    mbar_init(&cbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (bulk && warp == 0) {
    if (lane == 0) mbar_arrive_expect_tx(&cbar, (uint32_t)(ncols * nrows * (int)sizeof(T)));
    __syncwarp();
    for (int c = lane; c < ncols; c += 32)
      bulk_g2s(Cs + c * LY::LDC, Cg + grow0 + (gcol0 + c - cshift) * a.ldc, (uint32_t)(nrows * sizeof(T)), &cbar);
  }

  // ---- accumulators
  double acc[MI][NI][2];
  double acci[CPLX ? MI : 1][CPLX ? NI : 1][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      if (CPLX) acci[CPLX ? i : 0][CPLX ? j : 0][0] = acci[CPLX ? i : 0][CPLX ? j : 0][1] = 0.0;
    }

  const int nchunks = (a.K + C::KC - 1) / C::KC;
  // ---- prologue
#pragma unroll
  for (int st = 0; st < C::STAGES - 1; ++st) {
    if (st < nchunks) {
      T* As = sm + st * LY::STAGE_ELEMS;
      load_stage<CPLX, BLU, VEC>(As, As + LY::A_ELEMS, Ag, Bg, a, grow0, gcol0, st * C::KC);
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
        load_stage<CPLX, BLU, VEC>(As, As + LY::A_ELEMS, Ag, Bg, a, grow0, gcol0, nk * C::KC);
      }
      cp_async_commit();
    }
    const T* As = sm + (kc % C::STAGES) * LY::STAGE_ELEMS;
    const T* Bs = As + LY::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < C::KC / 4; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      T af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = As[kk * LY::LDA + wm * TM + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int n = wn * TN + j * 8 + (lane >> 2);
        bf[j] = BLU ? Bs[n * LY::LDBN + kk] : Bs[kk * LY::LDBK + n];
      }
      if constexpr (!CPLX) {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NI; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      } else {
        // product term a*b (LU) or a*conj(w) (Hermitian, b = w):
        //   LU:   re += ar br - ai bi ;  im += ar bi + ai br
        //   Herm: re += ar wr + ai wi ;  im += ai wr - ar wi
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const double ar = re(af[i]), ai = im(af[i]);
          const double nai = -ai, nar = -ar;
#pragma unroll
          for (int j = 0; j < NI; ++j) {
            const double br = re(bf[j]), bi = im(bf[j]);
            dmma884(acc[i][j][0], acc[i][j][1], ar, br);
            dmma884(acc[i][j][0], acc[i][j][1], BLU ? nai : ai, bi);
            dmma884(acci[CPLX ? i : 0][CPLX ? j : 0][0], acci[CPLX ? i : 0][CPLX ? j : 0][1], BLU ? ar : nar, bi);
            dmma884(acci[CPLX ? i : 0][CPLX ? j : 0][0], acci[CPLX ? i : 0][CPLX ? j : 0][1], ai, br);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: C -= acc in shared memory, then write the tile back
  if (bulk) {
    mbar_wait(&cbar, 0);
  } else {
    // unaligned / odd-row tiles: cooperative loads (the slow path; ragged tails only)
    for (int idx = tid; idx < ncols * nrows; idx += NT) {
      const int c = idx / nrows, r = idx % nrows;
      Cs[c * LY::LDC + r] = Cg[grow0 + r + (gcol0 + c - cshift) * a.ldc];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int r = wm * TM + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < NI; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wn * TN + j * 8 + 2 * (lane & 3) + e;
        if (r < nrows && c < ncols && (BLU || grow0 + r >= gcol0 + c)) {
          T* p = Cs + c * LY::LDC + r;
          if constexpr (!CPLX) {
            *p = *p - acc[i][j][e];
          } else {
            T v = *p;
            v.x -= acc[i][j][e];
            v.y -= acci[CPLX ? i : 0][CPLX ? j : 0][e];
            *p = v;
          }
        }
      }
    }
  }
  if (bulk && !diag_tile) {
    fence_proxy_async_smem();
    __syncthreads();
    if (warp == 0) {
      for (int c = lane; c < ncols; c += 32)
        bulk_s2g(Cg + grow0 + (gcol0 + c - cshift) * a.ldc, Cs + c * LY::LDC, (uint32_t)(nrows * sizeof(T)));
      bulk_commit();
      bulk_wait_read0();
    }
  } else {
    __syncthreads();
    // element stores; Hermitian diagonal tiles never write the strict upper triangle
    for (int idx = tid; idx < ncols * nrows; idx += NT) {
      const int c = idx / nrows, r = idx % nrows;
      if (BLU || grow0 + r >= gcol0 + c) Cg[grow0 + r + (gcol0 + c - cshift) * a.ldc] = Cs[c * LY::LDC + r];
    }
  }
}

int update_tile_m(Kind kind) { return kind == HERM_D ? Cfg<false>::BM : Cfg<true>::BM; }
int update_tile_n(Kind kind) { return kind == HERM_D ? Cfg<false>::BN : Cfg<true>::BN; }

template <bool CPLX, bool BLU, bool VEC>
static cudaError_t launch_update_t(UpdateArgs a, cudaStream_t s) {
  using C = Cfg<CPLX>;
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  a.tiles_m = (a.rows + C::BM - 1) / C::BM;
  if (a.bcc_P == 0) a.tiles_n = (a.cols + C::BN - 1) / C::BN;
  unsigned nblk;
  if (a.tri) nblk = (unsigned)a.tiles_m * (a.tiles_m + 1) / 2;
  else nblk = (unsigned)a.tiles_m * a.tiles_n;
  const size_t smem = Layout<CPLX, BLU>::SMEM;
  auto* fn = update_kernel<CPLX, BLU, VEC>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(nblk, 1, a.batch);
  fn<<<grid, C::WM * C::WN * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <bool CPLX, bool BLU> cudaError_t launch_update_ws_t(UpdateArgs a, cudaStream_t s);

// Fast path (update_ws.cu: persistent, warp-specialized, TMA-fed) for 16-byte-aligned operands;
// the cp.async kernel above handles unaligned real matrices (odd ld) and forced fallback.
static int g_force_generic = -1;
cudaError_t launch_update(Kind kind, UpdateArgs a, cudaStream_t s) {
  if (g_force_generic < 0) {
    const char* e = getenv("DPP_UPDATE_GENERIC");  // test hook: exercise the generic kernel
    g_force_generic = (e && e[0] == '1') ? 1 : 0;
  }
  const bool ws = a.vec && !g_force_generic;
  switch (kind) {
    case HERM_D:
      if (ws) return launch_update_ws_t<false, false>(a, s);
      return a.vec ? launch_update_t<false, false, true>(a, s) : launch_update_t<false, false, false>(a, s);
    case HERM_Z:
      if (ws) return launch_update_ws_t<true, false>(a, s);
      return launch_update_t<true, false, true>(a, s);
    case LU_Z:
      if (ws) return launch_update_ws_t<true, true>(a, s);
      return launch_update_t<true, true, true>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace dpp
