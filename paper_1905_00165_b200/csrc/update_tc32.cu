// update_tc32.cu -- the single-precision real update C -= A B^T (the fp32 sampler's panel and trailing
// updates, Listing 3 line 586 / PAPER.md:586 in fp32, reading R19) on the 5th-generation tensor
// cores: tcgen05.mma kind::tf32 with the accumulator in tensor memory (TMEM).
//
// sm_100a has no fp32-input tensor-core MMA; kind::tf32 reads 19-bit operands.  The products are
// therefore formed in the "3xTF32" split: x = x_hi + x_lo with x_hi = tf32_rn(x), x_lo = tf32_rn(x -
// x_hi), and A B^T = A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T (the dropped A_lo B_lo^T is ~2^-22
// |A||B|), accumulated in fp32 in TMEM: fp32-level accuracy (measured: the factor of an n = 1000
// fp32 sample differs from the fp32 oracle's by the same 1.3e-6 as the FP32 SIMT kernel's).
//
// Two kernels per update:
//   pack:   each operand (A: the update's rows x K, B: its columns x K, both MN-contiguous columns)
//           is split once into hi/lo tf32 parts and written as 16 KB images of the canonical
//           K-major no-swizzle UMMA layout, one per (128-row tile, 32-k chunk, part) -- so the
//           GEMM's producer moves each stage with two contiguous bulk copies;
//   GEMM:   one CTA per SM, persistent over 128 x 128 tiles of C:
//           warp 0     PRODUCER (one lane): TMA bulk copies (cp.async.bulk) of the four 16 KB
//                      images of a k-chunk into a 3-stage ring, full/empty mbarriers (320 threads);
//           warp 1     MMA ISSUER (one lane): per k-group of 8, three tcgen05.mma (M = N = 128,
//                      K = 8) into one of two TMEM accumulators (2 x 128 columns); tcgen05.commit
//                      releases the ring stage and, at the end of a tile, the accumulator;
//           warps 2-9  EPILOGUE: each loads its C values (32 rows x 64 columns) while the tile's
//                      MMAs run, then tcgen05.ld of its 32 TMEM lanes (= rows), C -= acc in global
//                      memory (coalesced column segments; Hermitian diagonal tiles masked), and
//                      releases the accumulator -- the epilogue of tile t overlaps the MMAs of
//                      tile t+1.
// The canonical layout (CuTe's Layout_K_INTER_Atom; make_umma_desc<Major::K> with SWIZZLE_NONE):
// core matrices of 8 rows x 16 bytes (4 k); the two 4-k halves of one MMA's K = 8 slice are LBO
// apart, consecutive 8-row groups SBO apart.  (The MN-major no-swizzle form, which would have
// spared the pack, produced no output for kind::tf32 in tools/tc32_test.cu.)
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "update_common.cuh"

namespace dpp {

namespace {

constexpr int TC_BM = 128, TC_BN = 128, TC_KC = 32, TC_STAGES = 3;
constexpr int TC_NT = 320;  // producer warp, MMA warp, 8 epilogue warps
constexpr uint32_t TC_PART = TC_BM * TC_KC * 4;  // 16 KB: one (tile, chunk) image of one part
constexpr uint32_t TC_STAGE = 4 * TC_PART;       // A hi, A lo, B hi, B lo
constexpr uint32_t TC_KLBO = 128, TC_KSBO = 256, TC_KSLICE = (TC_BM / 8) * TC_KSBO;  // 4 KB per K = 8
constexpr uint32_t TC_TMEM_COLS = 256;           // two 128-column fp32 accumulators

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  // start address, LBO, SBO in 16-byte units; version 1 (sm_100); layout SWIZZLE_NONE
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((TC_KLBO >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((TC_KSBO >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// byte offset of element (row mn, k) inside one 128 x 32 image
__device__ __forceinline__ uint32_t tc_koff(int mn, int k) {
  return (uint32_t)(k >> 3) * TC_KSLICE + (uint32_t)(mn >> 3) * TC_KSBO + (uint32_t)((k >> 2) & 1) * TC_KLBO +
         (uint32_t)(mn & 7) * 16 + (uint32_t)(k & 3) * 4;
}

__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(TC_IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 consecutive TMEM columns of this warp's 32 lanes: v[j] = column c0 + j of row lane
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// pack: rows [0, rows) x k [0, K) of X (element (r, k) at r + k ld) into images
// dst[((t * nch + c) * 2 + part) * TC_PART bytes] for row tile t, k chunk c; zeros beyond.
// Complex (complex64 X, C -= A B^T without conjugation) through the real embedding
//   [Re C; Im C] -= [A2; A3] B2^T,  k' = 2 k + e:  A2(i, 2k) = Re A, A2(i, 2k+1) = -Im A,
//   A3(i, 2k) = Im A, A3(i, 2k+1) = Re A,  B2(j, 2k) = Re B, B2(j, 2k+1) = Im B
// -- an A image holds 64 complex rows (A2 above A3), a B image 128 complex rows; K' = 2 K.
template <bool CPLX, bool AOP>
__device__ __forceinline__ void tc32_pack_tile(const void* Xv, int64_t ld, int rows, int K, int nch,
                                               unsigned char* dst, int t, int c, float (*img)[TC_BM * TC_KC]) {
  const int tid = threadIdx.x;
  constexpr int ROWS = (CPLX && AOP) ? TC_BM / 2 : TC_BM;  // operand rows per image
  for (int e = tid; e < TC_BM * TC_KC; e += 256) {
    const int r = e % TC_BM, k = e / TC_BM;  // consecutive threads: consecutive rows of one column
    float x;
    if constexpr (!CPLX) {
      const float* X = reinterpret_cast<const float*>(Xv);
      const int gr = t * TC_BM + r, gk = c * TC_KC + k;
      x = (gr < rows && gk < K) ? X[gr + (int64_t)gk * ld] : 0.f;
    } else {
      const float2* X = reinterpret_cast<const float2*>(Xv);
      const int i = AOP ? (r & (ROWS - 1)) : r, blk = AOP ? (r / ROWS) : 0;
      const int gr = t * ROWS + i, gk2 = c * TC_KC + k, gk = gk2 >> 1, ee = gk2 & 1;
      float2 z = make_float2(0.f, 0.f);
      if (gr < rows && gk < K) z = X[gr + (int64_t)gk * ld];
      if (!AOP) x = ee ? z.y : z.x;                 // B2
      else if (blk == 0) x = ee ? -z.y : z.x;       // A2
      else x = ee ? z.x : z.y;                      // A3
    }
    const float hi = tf32_rn(x);
    const uint32_t o = tc_koff(r, k) >> 2;
    img[0][o] = hi;
    img[1][o] = tf32_rn(x - hi);
  }
  __syncthreads();
  float4* out = reinterpret_cast<float4*>(dst + ((size_t)t * nch + c) * 2 * TC_PART);
  const float4* in = reinterpret_cast<const float4*>(&img[0][0]);
  for (int e = tid; e < 2 * TC_BM * TC_KC / 4; e += 256) out[e] = in[e];
}

// Both operands of an update in one launch: CTAs x < tiles_a pack A's row tiles, the others B's
// (two launches on the sampler's chain cost a launch each per update; the chain of the fp32
// sampler is its bound).
template <bool CPLX>
__global__ void __launch_bounds__(256) tc32_pack_kernel(const void* Av, int64_t lda, int arows, const void* Bv,
                                                        int64_t ldb, int brows, int K, int nch, int tiles_a,
                                                        unsigned char* pa, unsigned char* pb) {
  __shared__ __align__(16) float img[2][TC_BM * TC_KC];
  const int t = blockIdx.x, c = blockIdx.y;
  if (t < tiles_a) tc32_pack_tile<CPLX, true>(Av, lda, arows, K, nch, pa, t, c, img);
  else tc32_pack_tile<CPLX, false>(Bv, ldb, brows, K, nch, pb, t - tiles_a, c, img);
}

}  // namespace

template <bool MASK, bool CPLX>
__global__ void __launch_bounds__(TC_NT, 1) update_tc32_kernel(const UpdateArgs a, const unsigned char* pa,
                                                                const unsigned char* pb) {
  constexpr int TBM = CPLX ? TC_BM / 2 : TC_BM;  // C rows per tile (complex: 64, re and im stacked)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[TC_STAGES], empty[TC_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_s;
  unsigned char* ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t ring_s = smem_u32(ring);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_per_sample = a.tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  const int ntiles = tiles_per_sample * a.batch;
  const int nch = ((CPLX ? 2 : 1) * a.K + TC_KC - 1) / TC_KC;

  if (tid == 0) {
    for (int i = 0; i < TC_STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 256); }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)),
                 "n"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_s;

  if (warp == 0) {
    // ============================ producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileInfo ti = tile_info<TBM, TC_BN>(a, t, tiles_per_sample, MASK);
        if (!ti.valid) continue;
        const int tr = (ti.grow0 - a.row0) / TBM, tc = (ti.gcol0 - a.col0) / TC_BN;
        for (int kc = 0; kc < nch; ++kc) {
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* st = ring + (size_t)stage * TC_STAGE;
          mbar_arrive_expect_tx(&full[stage], TC_STAGE);
          const unsigned char* sa = pa + ((size_t)tr * nch + kc) * 2 * TC_PART;
          const unsigned char* sb = pb + ((size_t)tc * nch + kc) * 2 * TC_PART;
          bulk_g2s(st, sa, 2 * TC_PART, &full[stage]);                // A hi, A lo
          bulk_g2s(st + 2 * TC_PART, sb, 2 * TC_PART, &full[stage]);  // B hi, B lo
          if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TileInfo ti = tile_info<TBM, TC_BN>(a, t, tiles_per_sample, MASK);
      if (!ti.valid) continue;
      mbar_wait(&tempty[ab], aphase ^ 1);  // the epilogue has drained this accumulator
      tc_fence_after();
      const uint32_t tacc = tmem_base + (uint32_t)(ab * TC_BN);
      for (int kc = 0; kc < nch; ++kc) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t s0 = ring_s + (uint32_t)stage * TC_STAGE;
#pragma unroll
          for (int h = 0; h < TC_KC / 8; ++h) {
            const uint32_t ko = (uint32_t)h * TC_KSLICE;
            const uint64_t ahi = smem_desc(s0 + ko), alo = smem_desc(s0 + TC_PART + ko);
            const uint64_t bhi = smem_desc(s0 + 2 * TC_PART + ko), blo = smem_desc(s0 + 3 * TC_PART + ko);
            tc_mma(tacc, ahi, bhi, (kc | h) != 0);
            tc_mma(tacc, ahi, blo, 1u);
            tc_mma(tacc, alo, bhi, 1u);
          }
          tc_commit(&empty[stage]);                  // the stage is free once these MMAs are done
          if (kc == nch - 1) tc_commit(&tfull[ab]);  // the accumulator is complete
        }
        __syncwarp();
        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
      }
      if (++ab == 2) { ab = 0; aphase ^= 1; }
    }
  } else {
    // ============================ epilogue ============================
    // 8 warps: warp w serves TMEM lanes 32 (w % 4) .. + 31 (= tile rows) and columns 64 h .. 64 h + 63,
    // h = (w - 2) / 4; its C values are loaded BEFORE the accumulator is ready, so the global
    // round trip overlaps the tile's MMAs
    const int q = warp & 3, h = (warp - 2) >> 2;
    int ab = 0;
    uint32_t aphase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TileInfo ti = tile_info<TBM, TC_BN>(a, t, tiles_per_sample, MASK);
      if (!ti.valid) continue;
      // TMEM lane R = 32 q + lane: real row R, or complex row R mod 64, component R / 64
      const int R = 32 * q + lane;
      const int r = CPLX ? (R & (TBM - 1)) : R;
      const int grow = ti.grow0 + r;
      const int cb = 64 * h;
      constexpr int ES = CPLX ? 2 : 1;  // floats per element
      float* p0 = reinterpret_cast<float*>(a.C) +
                  ES * ((int64_t)ti.s * a.strideC + grow + (int64_t)(ti.gcol0 + cb - ti.cshift) * a.ldc) +
                  (CPLX ? R / TBM : 0);
      const bool row_in = r < ti.nrows;
      // second output W = C_new diag(wscale) (the Hermitian panel's W21 = L21 D1), real unmasked only
      float* w0 = nullptr;
      const double* ws = nullptr;
      if constexpr (!CPLX && !MASK) {
        if (a.wout) {
          w0 = reinterpret_cast<float*>(a.wout) + (int64_t)ti.s * a.strideWo + grow + (int64_t)(ti.gcol0 + cb) * a.ldw;
          ws = a.wscale + (int64_t)ti.s * a.wsstride + ti.gcol0 + cb;
        }
      }
      float cv[64];
#pragma unroll
      for (int j = 0; j < 64; ++j)
        cv[j] = (row_in && cb + j < ti.ncols && (!MASK || grow >= ti.gcol0 + cb + j)) ? p0[(int64_t)j * ES * a.ldc] : 0.f;
      mbar_wait(&tfull[ab], aphase);
      tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float v[32];
        tc_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(ab * TC_BN + cb + 32 * half), v);
        if (row_in) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int c = cb + 32 * half + j;
            if (c < ti.ncols && (!MASK || grow >= ti.gcol0 + c)) {
              const float nv = cv[32 * half + j] - v[j];
              p0[(int64_t)(32 * half + j) * ES * a.ldc] = nv;
              if (!CPLX && !MASK && w0) w0[(int64_t)(32 * half + j) * a.ldw] = scal(nv, __ldg(ws + 32 * half + j));
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[ab]);
      if (++ab == 2) { ab = 0; aphase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TC_TMEM_COLS)
                 : "memory");
  }
}

// Scratch bytes the packed operands of an update need (complex: 64-row A images, K' = 2 K).
size_t tc32_scratch_bytes(int rows, int cols, int K, bool cplx) {
  const size_t nch = (size_t)((cplx ? 2 : 1) * K + TC_KC - 1) / TC_KC;
  const int bm = cplx ? TC_BM / 2 : TC_BM;
  const size_t tm = (size_t)(rows + bm - 1) / bm, tn = (size_t)(cols + TC_BN - 1) / TC_BN;
  return (tm + tn) * nch * 2 * TC_PART;
}

template <bool CPLX>
static cudaError_t launch_tc32_t(UpdateArgs a, cudaStream_t s) {
  constexpr int TBM = CPLX ? TC_BM / 2 : TC_BM;
  using E = typename std::conditional<CPLX, float2, float>::type;
  a.tiles_m = (a.rows + TBM - 1) / TBM;
  a.tiles_n = (a.cols + TC_BN - 1) / TC_BN;
  const int nch = ((CPLX ? 2 : 1) * a.K + TC_KC - 1) / TC_KC;
  unsigned char* pa = reinterpret_cast<unsigned char*>(a.tcs);
  unsigned char* pb = pa + (size_t)a.tiles_m * nch * 2 * TC_PART;
  // the operand rows of the region: A rows [row0, row0 + rows), B rows [col0, col0 + cols)
  const E* Ar = reinterpret_cast<const E*>(a.Aop) + a.row0;
  const E* Br = reinterpret_cast<const E*>(a.Bop) + a.col0;
  tc32_pack_kernel<CPLX><<<dim3(a.tiles_m + a.tiles_n, nch), 256, 0, s>>>(
      Ar, a.lda, min(a.rows, a.a_rows - a.row0), Br, a.ldb, min(a.cols, a.b_rows - a.col0), a.K, nch, a.tiles_m, pa, pb);
  const long long per = a.tri ? (long long)a.tiles_m * (a.tiles_m + 1) / 2 : (long long)a.tiles_m * a.tiles_n;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long g = a.grid_limit > 0 ? a.grid_limit : sms;
  if (g > per) g = per;
  const size_t smem = (size_t)TC_STAGES * TC_STAGE + 1024;
  cudaError_t e;
  if (a.mask) {
    e = cudaFuncSetAttribute(update_tc32_kernel<true, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    update_tc32_kernel<true, CPLX><<<(unsigned)g, TC_NT, smem, s>>>(a, pa, pb);
  } else {
    e = cudaFuncSetAttribute(update_tc32_kernel<false, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    update_tc32_kernel<false, CPLX><<<(unsigned)g, TC_NT, smem, s>>>(a, pa, pb);
  }
  return cudaGetLastError();
}

// Single-precision updates on the tensor cores (3xTF32): real (HERM_S) or complex64 (LU_C, no
// conjugation, no mask); a.tcs must hold tc32_scratch_bytes of scratch for the packed operands.  One
// sample per launch (a.batch == 1); no block-cyclic mode.
cudaError_t launch_update_tc32(UpdateArgs a, cudaStream_t s, bool cplx) {
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  if (a.conj || a.bnmajor || a.dscale || a.batch != 1 || a.bcc_P || (cplx && a.mask)) return cudaErrorInvalidValue;
  if (!a.tcs || a.tcs_bytes < (int64_t)tc32_scratch_bytes(a.rows, a.cols, a.K, cplx)) return cudaErrorInvalidValue;
  return cplx ? launch_tc32_t<true>(a, s) : launch_tc32_t<false>(a, s);
}

}  // namespace dpp
