// update_ws.cu -- Stage 3 fast path (also stage-2 GEMMs): persistent, warp-specialized FP64
// tensor-core contraction C -= A op(B)^T (see update.cu for the operation and the citations:
// Listing 3; Hermitian specialisation PAPER.md:396-398, 626-628).
//
// Organised the Blackwell way for 16-byte-aligned operands:
//  * persistent CTAs walk the tile list round-robin (<= 4 tiles each, so the high-priority
//    lookahead stream still finds SMs between tiles);
//  * one PRODUCER warp streams operand K-chunks with TMA bulk copies (cp.async.bulk, one 1-D copy
//    per column segment into padded shared rows) into a STAGES-deep ring guarded by full/empty
//    mbarriers; a second warp owns the C tile (bulk load -> consumers subtract -> bulk store);
//  * CONSUMER warps (real: 16 of 32x32; complex: 8 of 32x16) run
//    DMMA.8x8x4 (mma.sync m8n8k4 f64) out of the ring with no CTA-wide barrier in the main loop and
//    subtract their accumulators from the C tile in shared memory.
// Ragged edges: rows/columns beyond the tile are left stale in shared memory (they only feed
// masked outputs); K-columns beyond jb are zero-filled; an odd trailing row (real) is moved with
// ordinary loads/stores.
#include <cuda_runtime.h>


#include "common.cuh"
#include "kernels.h"
#include "update_common.cuh"


// Ring geometry (tools/gpu_update_ab.sh).  A chunk boundary (barrier round, first fragment loads) is
// reached by the four warps of a sub-partition together and idles its FP64 pipe, so FEW LARGE chunks
// beat a deep ring of small ones: real kernels 2 stages of 16 k (64 DMMAs per warp and chunk) --
// probe K = 384: 33.8 TF/s against 32.9 for 5 x 8 k and 32.1 for 11 x 4 k; 3 x 12 k the same but
// K = 128 is not a multiple of 12 (profiles/r02/update_ab.txt).
#ifndef DPP_WS_KC
#define DPP_WS_KC 16      // real kernels: k per ring stage ...
#define DPP_WS_STAGES 2   // ... and ring stages
#endif
#ifndef DPP_WS_KCZ
#define DPP_WS_KCZ 16     // complex kernels (64 x 64 tiles): 4 stages of 16 k -- Aztec d = 80 33.3 -> 34.3 TF/s,
#define DPP_WS_STAGESZ 4  // n = 32768 block-cyclic 31.1 -> 32.5, n = 8192 Hermitian / LU +2.8 / +2.2 % over 4 x 8 k
#endif

namespace dpp {

template <bool CPLX, int V> struct WsCfg;
template <> struct WsCfg<false, 1> {  // real: 128x128 tile, 16 consumer warps 4 x 4 of 32x32
  static constexpr int BM = 128, BN = 128, WM = 4, WN = 4, KC = DPP_WS_KC, STAGES = DPP_WS_STAGES;
};
template <> struct WsCfg<true, 0> {   // complex: 64x64 tile, consumer warps 2 x 4 of 32x16
  static constexpr int BM = 64, BN = 64, WM = 2, WN = 4, KC = DPP_WS_KCZ, STAGES = DPP_WS_STAGESZ;
};

template <bool CPLX, bool BNMAJ, int V>
struct WsLayoutT {
  using C = WsCfg<CPLX, V>;
  using T = typename Elem<CPLX>::T;
  static constexpr int ES = CPLX ? 16 : 8;
  static constexpr int PAD = CPLX ? 2 : 4;     // conflict-free 64/128-bit fragment loads
  static constexpr int LDA = C::BM + PAD;      // A: [KC][LDA]
  static constexpr int LDBK = C::BN + PAD;     // K-major B: [KC][LDBK]
  static constexpr int LDBN = C::KC + PAD;     // N-major B: [BN][LDBN]
  static constexpr int A_ELEMS = C::KC * LDA;
  static constexpr int B_ELEMS = BNMAJ ? C::BN * LDBN : C::KC * LDBK;
  static constexpr int D_ELEMS = (C::KC * 8 + ES - 1) / ES;  // per-k scale of B
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS + D_ELEMS;
  static constexpr int LDC = CPLX ? C::BM + 1 : C::BM + 2;
  static constexpr size_t RING = (size_t)STAGE_ELEMS * C::STAGES * ES;
  static constexpr size_t CTILE = (size_t)C::BN * LDC * ES;
  static constexpr size_t BAR_OFF = RING + CTILE;
  static constexpr size_t SMEM = BAR_OFF + (2 * C::STAGES + 2) * 8;
  static constexpr int NCONS = C::WM * C::WN;  // consumer warps
  static constexpr int NT = (NCONS + 2) * 32;   // + operand producer warp + C-tile warp
};

__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ, int V>
__global__ void __launch_bounds__(WsLayoutT<CPLX, BNMAJ, V>::NT, 1) update_ws_kernel(const UpdateArgs a) {
  using LY = WsLayoutT<CPLX, BNMAJ, V>;
  using C = WsCfg<CPLX, V>;
  using T = typename LY::T;
  constexpr int TM = C::BM / C::WM, TN = C::BN / C::WN, MI = TM / 8, NI = TN / 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  T* Cs = reinterpret_cast<T*>(smem_raw + LY::RING);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + LY::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* cfull = empty + C::STAGES;
  uint64_t* cready = cfull + 1;  // consumers finished C -= acc (count: consumer warps)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_per_sample = a.tri ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  const int ntiles = tiles_per_sample * a.batch;
  const int nchunks = (a.K + C::KC - 1) / C::KC;

  if (tid == 0) {
    for (int i = 0; i < C::STAGES; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], LY::NCONS); }
    mbar_init(cfull, 1);
    mbar_init(cready, LY::NCONS);
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == LY::NCONS + 1) {
    // ============================ C-tile warp ============================
    // Owns the life of the C region: load C(t) -> (consumers subtract) -> bulk-store C(t) ->
    // load C(t+1); runs beside the operand producer so neither ever blocks the other.
    uint32_t rphase = 0;
    bool have_prev = false;
    TileInfo prev{};
    auto flush_prev = [&]() {  // store the previous tile's C once the consumers are done with it
      if (!have_prev) return;
      mbar_wait(cready, rphase);
      rphase ^= 1;
      if (!prev.diag) {
        T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)prev.s * a.strideC;
        const int cbulk = CPLX ? prev.nrows : (prev.nrows & ~1);
        if (cbulk > 0)
          for (int c = lane; c < prev.ncols; c += 32)
            bulk_s2g(Cg + prev.grow0 + (prev.gcol0 + c - prev.cshift) * a.ldc, Cs + c * LY::LDC,
                     (uint32_t)(cbulk * LY::ES));
        bulk_commit();
        if (!CPLX && (prev.nrows & 1))
          for (int c = lane; c < prev.ncols; c += 32)
            Cg[prev.grow0 + prev.nrows - 1 + (prev.gcol0 + c - prev.cshift) * a.ldc] = Cs[c * LY::LDC + prev.nrows - 1];
        bulk_wait_read0();
      }
      __syncwarp();
      have_prev = false;
    };
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TileInfo ti = tile_info<C::BM, C::BN>(a, t, tiles_per_sample, MASK);
      if (!ti.valid) continue;
      // C values are read from csrc when the driver deferred the workspace copy to this launch
      const T* Cg = a.csrc ? reinterpret_cast<const T*>(a.csrc) + (int64_t)ti.s * a.strideCs
                           : reinterpret_cast<const T*>(a.C) + (int64_t)ti.s * a.strideC;
      const int64_t ldr = a.csrc ? a.ldcs : a.ldc;
      const int cbulk = CPLX ? ti.nrows : (ti.nrows & ~1);
      flush_prev();
      if (!CPLX && (ti.nrows & 1)) {  // odd trailing row: ordinary copies
        for (int c = lane; c < ti.ncols; c += 32)
          Cs[c * LY::LDC + ti.nrows - 1] = Cg[ti.grow0 + ti.nrows - 1 + (ti.gcol0 + c - ti.cshift) * ldr];
      }
      fence_proxy_async_smem();  // generic smem accesses before the async-proxy writes
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(cfull, (uint32_t)(ti.ncols * cbulk * LY::ES));
      __syncwarp();
      if (cbulk > 0)
        for (int c = lane; c < ti.ncols; c += 32)
          bulk_g2s(Cs + c * LY::LDC, Cg + ti.grow0 + (ti.gcol0 + c - ti.cshift) * ldr, (uint32_t)(cbulk * LY::ES),
                   cfull);
      prev = ti;
      have_prev = true;
    }
    flush_prev();
    bulk_wait_all();  // the last stores are complete (visible) before the CTA retires
    return;
  }

  if (warp == LY::NCONS) {
    // ============================ operand producer warp ============================
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const TileInfo ti = tile_info<C::BM, C::BN>(a, t, tiles_per_sample, MASK);
      if (!ti.valid) continue;
      const T* Ag = reinterpret_cast<const T*>(a.Aop) + (int64_t)ti.s * a.strideA;
      const T* Bg = reinterpret_cast<const T*>(a.Bop) + (int64_t)ti.s * a.strideB;
      const double* dsc = SCALE ? a.dscale + (int64_t)ti.s * a.dstride : nullptr;
      const int arows = min(C::BM, a.a_rows - ti.grow0);   // operand rows that exist
      const int bcols = min(C::BN, a.b_rows - ti.gcol0);
      const int abulk = CPLX ? arows : (arows & ~1), bbulk = CPLX ? bcols : (bcols & ~1);
      for (int kc = a.ktri ? ti.grow0 / C::KC : 0; kc < nchunks; ++kc) {
        mbar_wait(&empty[stage], phase ^ 1);
        T* As = ring + stage * LY::STAGE_ELEMS;
        T* Bs = As + LY::A_ELEMS;
        const int k0 = kc * C::KC;
        const int kv = min(C::KC, a.K - k0);  // valid k in this chunk
        if (SCALE && lane < C::KC) reinterpret_cast<double*>(Bs + LY::B_ELEMS)[lane] = lane < kv ? dsc[k0 + lane] : 0.0;
        // zero-fill k beyond K; odd trailing operand rows by ordinary copies
        for (int idx = lane; idx < (C::KC - kv) * C::BM; idx += 32) As[(kv + idx / C::BM) * LY::LDA + idx % C::BM] = zero<T>();
        if (!BNMAJ) {
          for (int idx = lane; idx < (C::KC - kv) * C::BN; idx += 32) Bs[(kv + idx / C::BN) * LY::LDBK + idx % C::BN] = zero<T>();
        } else {
          for (int idx = lane; idx < (C::KC - kv) * C::BN; idx += 32)
            Bs[(idx % C::BN) * LY::LDBN + kv + idx / C::BN] = zero<T>();
        }
        if (!CPLX) {
          if (arows & 1)
            for (int kk = lane; kk < kv; kk += 32)
              As[kk * LY::LDA + arows - 1] = Ag[ti.grow0 + arows - 1 + (int64_t)(k0 + kk) * a.lda];
          if (!BNMAJ && (bcols & 1))
            for (int kk = lane; kk < kv; kk += 32)
              Bs[kk * LY::LDBK + bcols - 1] = Bg[ti.gcol0 + bcols - 1 + (int64_t)(k0 + kk) * a.ldb];
        }
        fence_proxy_async_smem();
        __syncwarp();
        uint32_t bytes = (uint32_t)(kv * abulk * LY::ES);
        bytes += BNMAJ ? (uint32_t)(bcols * kv * LY::ES) : (uint32_t)(kv * bbulk * LY::ES);
        if (lane == 0) mbar_arrive_expect_tx(&full[stage], bytes);
        __syncwarp();
        if (abulk > 0)
          for (int kk = lane; kk < kv; kk += 32)
            bulk_g2s(As + kk * LY::LDA, Ag + ti.grow0 + (int64_t)(k0 + kk) * a.lda, (uint32_t)(abulk * LY::ES),
                     &full[stage]);
        if (!BNMAJ) {
          if (bbulk > 0)
            for (int kk = lane; kk < kv; kk += 32)
              bulk_g2s(Bs + kk * LY::LDBK, Bg + ti.gcol0 + (int64_t)(k0 + kk) * a.ldb, (uint32_t)(bbulk * LY::ES),
                       &full[stage]);
        } else {
          for (int c = lane; c < bcols; c += 32)
            bulk_g2s(Bs + c * LY::LDBN, Bg + k0 + (int64_t)(ti.gcol0 + c) * a.ldb, (uint32_t)(kv * LY::ES),
                     &full[stage]);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }

  // ============================ consumer warps ============================
  // Warp -> warp tile.  A warp's DMMAs run on its sub-partition's FP64 pipe (SMSP = warp & 3, one
  // warp saturates it: tools/dmma_tput.cu), so a tile takes as long as its busiest sub-partition.
  // Real 4 x 4 layout: the plain map wm = warp & 3 would put the four working warps of row 3 of a
  // masked diagonal tile on one sub-partition (the tile as slow as a full one); this table gives
  // every sub-partition one warp tile per column with, on a diagonal tile, (below, below, idle, idle)
  // on two of them and (diag, diag, below, idle) on the other two: 2 / 2.25 warp tiles of DMMAs
  // instead of 4 (diagonal warp tiles skip their 6 of 16 fragments above the diagonal).
  int wm = warp % C::WM;
  const int wn = warp / C::WM;
  if constexpr (MASK && !CPLX && C::WM == 4 && C::WN == 4) {
    // wm[s = warp & 3][wn]: s0 {0,1,3,0}, s1 {1,0,2,3}, s2 {2,2,0,1}, s3 {3,3,1,2}; each column a permutation
    constexpr uint32_t TBL = (0u | 1u << 2 | 3u << 4 | 0u << 6) | (1u | 0u << 2 | 2u << 4 | 3u << 6) << 8 |
                             (2u | 2u << 2 | 0u << 4 | 1u << 6) << 16 | (3u | 3u << 2 | 1u << 4 | 2u << 6) << 24;
    wm = (TBL >> (8 * (warp & 3) + 2 * wn)) & 3;
  }
  int stage = 0;
  uint32_t phase = 0, cphase = 0;
  bool ready = false;  // the current stage's full barrier was already seen complete
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const TileInfo ti = tile_info<C::BM, C::BN>(a, t, tiles_per_sample, MASK);
    if (!ti.valid) continue;
    MmaAcc<CPLX, MI, NI> acc;
    acc.zero();
    // a warp tile strictly above the diagonal of a masked diagonal tile writes nothing: it only
    // keeps pace with the ring (waits and releases every stage) and leaves the DMMA pipe to the others
    const bool idle = MASK && ti.diag && ti.gcol0 + wn * TN > ti.grow0 + wm * TM + TM - 1;
    const bool wdiag = !CPLX && MASK && TM == TN && ti.diag && ti.gcol0 + wn * TN == ti.grow0 + wm * TM;
    const int kc0 = a.ktri ? ti.grow0 / C::KC : 0;
    // triangular B (stage-2 operators): the warp's columns need k <= its last column only; the
    // chunks past it are waited for and released without DMMA (the ring is shared by all warps)
    const int kcend = a.btri ? min(nchunks, (ti.gcol0 + wn * TN + TN + C::KC - 1) / C::KC) : nchunks;
    if (idle) {
      for (int kc = kc0; kc < nchunks; ++kc) {
        if (!ready) mbar_wait(&full[stage], phase);
        ready = false;
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    } else {
      // One copy of the chunk body per ring stage (s is a constant in each): the operand and barrier
      // addresses are base + immediate, so nothing but the fragment loads sits between a chunk's
      // wait and its first DMMA; and the NEXT stage's barrier is tested a whole chunk early
      // (`ready`), so the wait itself leaves the chunk boundary when the producer is ahead.  The four
      // warps of a sub-partition reach a chunk boundary together (they share one FP64 pipe fairly):
      // whatever a boundary costs beyond the other warps' three DMMA slots idles the pipe.
      int kc = kc0;
      while (kc < nchunks) {
#pragma unroll
        for (int s = 0; s < C::STAGES; ++s) {
          if (s == stage && kc < nchunks) {
            if (!ready) mbar_wait(&full[s], phase);
            ready = mbar_test(&full[(s + 1) % C::STAGES], s + 1 == C::STAGES ? phase ^ 1 : phase);
            if (kc < kcend) {
              const T* As = ring + s * LY::STAGE_ELEMS;
              mma_chunk<CPLX, BNMAJ, SCALE, CONJ, C::KC, MI, NI, LY::LDA, LY::LDBK, LY::LDBN>(
                  acc, As, As + LY::A_ELEMS, reinterpret_cast<const double*>(As + LY::A_ELEMS + LY::B_ELEMS), wm * TM,
                  wn * TN, lane, wdiag);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            ++kc;
            if (s + 1 == C::STAGES) { stage = 0; phase ^= 1; } else { stage = s + 1; }
          }
        }
      }
    }
    // ---- epilogue: C -= acc in shared memory; the C warp writes the tile back
    // (the W21 scale of this lane's column is loaded first: its latency hides behind the wait and
    // the subtraction instead of sitting, once per column, inside the store loop below)
    double dl = 0.0;
    if constexpr (!MASK) {
      static_assert(MASK || TN <= 32, "one W21 scale per lane");
      if (a.wout && lane < TN && wn * TN + lane < ti.ncols)
        dl = __ldg(a.wscale + (int64_t)ti.s * a.wsstride + ti.gcol0 + wn * TN + lane);
    }
    mbar_wait(cfull, cphase);
    cphase ^= 1;
    acc.template subtract_into<MASK, TM, TN, LY::LDC>(Cs, wm, wn, lane, ti);
    if constexpr (!MASK) {
      if (a.wout) {
        // second output W = C_new diag(wscale) (the Hermitian panel's W21 = L21 D1): each warp
        // re-reads its own TM x TN part of the updated tile, one row per lane, coalesced stores
        __syncwarp();
        T* Wg = reinterpret_cast<T*>(a.wout) + (int64_t)ti.s * a.strideWo + ti.grow0 + (int64_t)ti.gcol0 * a.ldw;
#pragma unroll 8
        for (int cc = 0; cc < TN; ++cc) {
          const int c = wn * TN + cc;
          const double dc = __shfl_sync(0xffffffffu, dl, cc);
          if (c < ti.ncols)
            for (int r = wm * TM + lane; r < wm * TM + TM && r < ti.nrows; r += 32)
              Wg[r + (int64_t)c * a.ldw] = scal(Cs[c * LY::LDC + r], dc);
        }
      }
    }
    if (ti.diag) {
      // Hermitian diagonal tile: element stores that never touch the strict upper triangle
      T* Cg = reinterpret_cast<T*>(a.C) + (int64_t)ti.s * a.strideC;
      consumer_sync(LY::NCONS * 32);
      for (int idx = tid; idx < ti.ncols * ti.nrows; idx += LY::NCONS * 32) {
        const int c = idx / ti.nrows, r = idx % ti.nrows;
        if (ti.grow0 + r >= ti.gcol0 + c) Cg[ti.grow0 + r + (ti.gcol0 + c - ti.cshift) * a.ldc] = Cs[c * LY::LDC + r];
      }
    }
    fence_proxy_async_smem();  // make this thread's smem writes visible to the bulk store
    __syncwarp();
    if (lane == 0) mbar_arrive(cready);
  }
}

#ifndef DPP_WS_TPC
#define DPP_WS_TPC 8  // tiles per short-lived CTA (tools/gpu_tpc_sweep.sh: UST 2913 / 2929 / 2925 samples/s for 4 / 8 / 16, 2860 for 2; C4 flat)
#endif

static int num_sms() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] > 0 ? sms[dev] : 148;
}

template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ, int V>
cudaError_t launch_update_ws_v(UpdateArgs a, cudaStream_t s) {
  using C = WsCfg<CPLX, V>;
  using LY = WsLayoutT<CPLX, BNMAJ, V>;
  if (a.rows <= 0 || a.cols <= 0 || a.K <= 0) return cudaSuccess;
  constexpr int CPS = 1;  // CTAs per SM
  a.tiles_m = (a.rows + C::BM - 1) / C::BM;
  if (a.bcc_P == 0) a.tiles_n = (a.cols + C::BN - 1) / C::BN;
  const long long per = a.tri ? (long long)a.tiles_m * (a.tiles_m + 1) / 2 : (long long)a.tiles_m * a.tiles_n;
  const long long total = per * a.batch;
  if (total <= 0) return cudaSuccess;
  // short-lived CTAs walk <= TPC = 8 tiles each (at least one wave of the SMs), so the high-priority
  // lookahead stream still finds SMs between tiles; persistent launches take the CTAs granted
  constexpr long long TPC = DPP_WS_TPC;
  long long g;
  if (a.grid_limit > 0) {
    const long long lim = (long long)a.grid_limit * CPS;
    g = total < lim ? total : lim;  // persistent over the CTAs granted
  } else {
    g = (total + TPC - 1) / TPC;
    if (g < num_sms() * CPS) g = total < num_sms() * CPS ? total : num_sms() * CPS;
  }
  auto* fn = update_ws_kernel<CPLX, BNMAJ, MASK, SCALE, CONJ, V>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LY::SMEM);
  if (e != cudaSuccess) return e;
  fn<<<(unsigned)g, LY::NT, LY::SMEM, s>>>(a);
  return cudaGetLastError();
}

// Real kernels: 128 x 128 tiles, 16 consumer warps of 32 x 32 (96 registers; 85.9 % tensor-active
// against 81.6 % for 8 consumer warps of 64 x 32 at the 168-register cap, and faster than 64 x 128
// tiles with two CTAs per SM, which double the operand traffic per flop -- round-1 measurements,
// DESIGN.md §6).  Complex kernels: 64 x 64 tiles, 8 consumer warps of 32 x 16.
template <bool CPLX, bool BNMAJ, bool MASK, bool SCALE, bool CONJ>
cudaError_t launch_update_ws_t(UpdateArgs a, cudaStream_t s) {
  return launch_update_ws_v<CPLX, BNMAJ, MASK, SCALE, CONJ, CPLX ? 0 : 1>(a, s);
}

template cudaError_t launch_update_ws_t<false, false, true, true, false>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<false, false, false, false, false>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<true, false, true, true, true>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<true, false, false, false, false>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<true, true, false, false, false>(UpdateArgs, cudaStream_t);
// Hermitian trailing update with a pre-scaled A operand (W21 = L21 D1): no per-k scaling
template cudaError_t launch_update_ws_t<false, false, true, false, false>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<true, false, true, false, true>(UpdateArgs, cudaStream_t);
template cudaError_t launch_update_ws_t<true, false, false, false, true>(UpdateArgs, cudaStream_t);

}  // namespace dpp
