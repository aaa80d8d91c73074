// driver.cu -- host driver of the blocked sampler and the C ABI of include/dpp.h.
//
// Blocked, right-looking DPP sampling = Listing 3's loop with line 583
// replaced by the unblocked sampler (Listing 4):
//   for j0 in 0, nb, 2nb, ...:
//     stage 1  diag(j0):   sample-and-factor the diagonal tile; form the small inverse operators
//     stage 2  panel(j0):  L21 = A21 L11^-H D1^-1 (Hermitian) or L21 = A21 U11^-1, U12 = L11^-1 A12
//                          (LU), as DMMA GEMMs with those operators (update kernels)
//     stage 3  update(j0): A22 -= L21 D1 L21^H (lower) or A22 -= L21 U12 (DMMA)
// With lookahead (the GPU analogue of the paper's tile-dependency task
// scheduling) the update of step k is split into
//   (a) the next block column (and, for LU, the next block row), on the high-priority stream S1,
//       immediately followed by diag(k+1) and panel(k+1), and
//   (b) the rest of the trailing matrix, on stream S2,
// so the sequential diag/panel chain of step k+1 runs under the big update of step k.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace dpp;

// schedule constants (compile-time; measured values, DESIGN.md §6 "Schedules tried")
#ifndef DPP_DIAG_TILES
#define DPP_DIAG_TILES 2.5        // one sample's diag tile in update-tile times (K = nb)
#endif
#ifndef DPP_DIAG_TILES_BATCH
#define DPP_DIAG_TILES_BATCH 5.0  // the same in the batched cost model
#endif
#ifndef DPP_GROUP_MIN_ROWS
#define DPP_GROUP_MIN_ROWS 6144   // 128-wide Hermitian blocks: no grouping at or below this many rows
#endif
#ifndef DPP_SPLIT_ROWS
#define DPP_SPLIT_ROWS 3072       // split chain at or below this many trailing rows
#endif

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x, size_t a = ALIGN) { return (x + a - 1) / a * a; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct Opts {
  int nb;          // the diag / update tile width (32, 64, 128 real; 32, 64 complex)
  int lookahead;
  double tie_tol, range_tol;
  const uint8_t* forced;
  int64_t batch_chunk;
  int group;             // G: trailing updates of G consecutive steps applied as one K = G nb pass
  int64_t group_min_rows;  // -1: defaults; else group only while more than this many rows remain
  bool generic;          // DPP_FLAG_GENERIC_UPDATE
  bool fp32_simt;        // DPP_FLAG_FP32_SIMT
  bool no_split;         // DPP_FLAG_NO_SPLIT_CHAIN
};

// opts->nb larger than the kind's tile (256 real; 128 or 256 complex) is the blocked algorithm with
// that block width whose diagonal-block factorization is itself blocked by the tile width: the
// block's trailing update is one K = nb pass (a group of nb / tile steps, lookahead on).  Prop. 5
// makes every blocking sample the same decisions in exact arithmetic.
int resolve_opts(Kind kind, const dpp_opts_t* o, Opts* r) {
  const int tile_max = kind_cplx(kind) ? 64 : 128;
  int nb = (o && o->nb) ? o->nb : tile_max;
  r->lookahead = o ? o->lookahead : 1;
  r->tie_tol = (o && o->tie_tol > 0) ? o->tie_tol : 1e-9;
  r->range_tol = (o && o->range_tol > 0) ? o->range_tol : 1e-8;
  r->forced = o ? o->forced : nullptr;
  r->batch_chunk = o ? o->batch_chunk : 0;
  r->generic = o && (o->flags & DPP_FLAG_GENERIC_UPDATE);
  r->fp32_simt = o && (o->flags & DPP_FLAG_FP32_SIMT);
  r->no_split = o && (o->flags & DPP_FLAG_NO_SPLIT_CHAIN);
  if (nb != 32 && nb != 64 && nb != 128 && nb != 256) return DPP_EINVAL;
  if (o && (o->group < 0 || o->group > 8)) return DPP_EINVAL;
  // G = 3 by default (round 2: C4 31.2 vs 30.8 TF/s with G = 2, UST 2675 vs 2643 samples/s,
  // complex samples within noise; round 1, with the slower diag kernel, had measured G = 2 best)
  r->group = (o && o->group) ? o->group : 3;
  // internal: -1 = the library's default thresholds (group_threshold below), else group only while
  // more than this many trailing rows remain (0: at every size)
  const int64_t gm = o ? o->group_min_rows : 0;
  r->group_min_rows = gm == 0 ? -1 : (gm < 0 ? 0 : gm);
  if (nb > tile_max) {
    r->group = nb / tile_max;
    r->group_min_rows = 0;
    nb = tile_max;
  }
  r->nb = nb;
  if (r->lookahead < 0 || r->lookahead > 1) return DPP_EINVAL;
  if (r->batch_chunk < 0) return DPP_EINVAL;
  return DPP_OK;
}

size_t esize(Kind k) { return kind_esize(k); }


// Workspace layout (all regions 256-byte aligned):
//   [SampleState x chunk]
//   [panel operators: Bm (and Am for LU), nb x nb per sample]
//   [D1 double buffer (Hermitian): 2 x chunk x nb doubles]
//   [operand panels: two group buffers of max(G, 2) panels of ldk x nb per sample -- W21 = L21 D1
//    (Hermitian, the pre-scaled trailing-update operand) or U12^T (LU, the row panel K-major)]
//   [K copies: chunk x ldk x n (batched / host)][host staging: mask, loglik, info (host)]
struct WsLayout {
  size_t state_off, bm_off, am_off, d_off, ut_off, tcs_off, k_off, mask_off, ll_off, info_off, total;
  size_t tcs_bytes;  // per stream region (two regions: the chain's stream and the trailing stream)
  int64_t ldk, strideK, strideM, strideU;
};

WsLayout layout(Kind kind, int64_t chunk, int64_t n, const Opts& o, bool copies, bool host) {
  WsLayout L{};
  const size_t es = esize(kind);
  const int nb = o.nb;
  L.ldk = std::max<int64_t>(round_up(n, 16), 16);
  L.strideK = L.ldk * std::max<int64_t>(n, 1);
  L.strideM = (int64_t)nb * nb;
  L.strideU = L.ldk * std::min<int64_t>(nb, std::max<int64_t>(n, 1));  // panel buffers: ldk x min(nb, n)
  size_t off = 0;
  L.state_off = off; off = align_up(off + sizeof(SampleState) * (size_t)chunk);
  L.bm_off = off; off = align_up(off + (size_t)chunk * L.strideM * es);
  L.am_off = off;
  if (!kind_herm(kind)) off = align_up(off + (size_t)chunk * L.strideM * es);
  L.d_off = off;
  if (kind_herm(kind)) off = align_up(off + 2 * (size_t)chunk * nb * 8);
  L.ut_off = off;
  off = align_up(off + 2 * (size_t)std::max(o.group, 2) * chunk * (size_t)L.strideU * es);
  // single precision, one sample: the 3xTF32 tensor-core updates' packed operands, one region
  // per stream (the lookahead and the trailing updates run concurrently)
  L.tcs_off = off;
  L.tcs_bytes = 0;
  if ((kind == HERM_S || kind == LU_C) && chunk == 1 && !o.fp32_simt && n > 0) {
    const int kmax = std::max(o.group, 1) * nb;
    L.tcs_bytes = align_up(tc32_scratch_bytes((int)n, (int)n, kmax, kind == LU_C));
    off = align_up(off + 2 * L.tcs_bytes);
  }
  L.k_off = off;
  if (copies) off = align_up(off + (size_t)chunk * (size_t)L.strideK * es);
  L.mask_off = off;
  if (host) off = align_up(off + (size_t)chunk * (size_t)std::max<int64_t>(n, 1));
  L.ll_off = off;
  if (host) off = align_up(off + 8 * (size_t)chunk);
  L.info_off = off;
  if (host) off = align_up(off + sizeof(dpp_info_t) * (size_t)chunk);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------- stream pair per device
struct DeviceStreams {
  cudaStream_t s1 = nullptr, s2 = nullptr, s3 = nullptr;  // chain, trailing, split-off chain work
  cudaEvent_t ev_start, ev_panel, ev_rest, ev_done1, ev_done2, ev_diag, ev_p0, ev_p1, ev_lr, ev_done3;
  std::recursive_mutex mu;
  bool init = false;
};
// Per device, a few stream pairs (with their events): calls made on different caller streams get
// different pairs, so independent samplers in flight on two caller streams run concurrently (one
// step's copy and first block steps under the previous step's chain-bound tail); calls on the
// same caller stream share a pair and stay in call order.
constexpr int NPAIRS = 4;
DeviceStreams g_streams[64][NPAIRS];
cudaStream_t g_pair_owner[64][NPAIRS];
int g_pair_next[64];
std::mutex g_streams_mu;

int get_streams(DeviceStreams** out, cudaStream_t caller = nullptr) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DPP_ECUDA;
  std::lock_guard<std::mutex> lk(g_streams_mu);
  int slot = -1;
  for (int i = 0; i < NPAIRS && slot < 0; ++i)
    if (g_streams[dev][i].init && g_pair_owner[dev][i] == caller) slot = i;
  if (slot < 0) {  // a new caller stream: the next pair, round robin
    slot = g_pair_next[dev];
    g_pair_next[dev] = (slot + 1) % NPAIRS;
    g_pair_owner[dev][slot] = caller;
  }
  DeviceStreams& d = g_streams[dev][slot];
  if (!d.init) {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return DPP_ECUDA;
    if (cudaStreamCreateWithPriority(&d.s1, cudaStreamNonBlocking, hi) != cudaSuccess) return DPP_ECUDA;
    if (cudaStreamCreateWithPriority(&d.s2, cudaStreamNonBlocking, lo) != cudaSuccess) return DPP_ECUDA;
    if (cudaStreamCreateWithPriority(&d.s3, cudaStreamNonBlocking, hi) != cudaSuccess) return DPP_ECUDA;
    for (cudaEvent_t* e : {&d.ev_start, &d.ev_panel, &d.ev_rest, &d.ev_done1, &d.ev_done2, &d.ev_diag, &d.ev_p0,
                           &d.ev_p1, &d.ev_lr, &d.ev_done3})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return DPP_ECUDA;
    d.init = true;
  }
  *out = &d;
  return DPP_OK;
}

int check_device() {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DPP_ECUDA;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return DPP_ECUDA;
  return major == 10 ? DPP_OK : DPP_EUNSUPPORTED;
}

#define CK(x) do { if ((x) != cudaSuccess) return DPP_ECUDA; } while (0)

// ---------------------------------------------------------------- stage profiling
struct ProfRec { int stage; double flops; cudaEvent_t e0, e1; };
struct Profiler {
  bool on = false;
  unsigned mask = 0x1f;  // stages recorded
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) { cudaEvent_t e; cudaEventCreate(&e); pool.push_back(e); }
    return pool[used++];
  }
};
thread_local Profiler g_prof;

struct ProfScope {  // brackets one launch with events on its stream
  int stage; double flops; cudaStream_t s; cudaEvent_t e1 = nullptr;
  ProfScope(int st, double fl, cudaStream_t str) : stage(st), flops(fl), s(str) {
    if (g_prof.on && (g_prof.mask >> st & 1u)) {
      cudaEvent_t e0 = g_prof.get();
      e1 = g_prof.get();
      cudaEventRecord(e0, s);
      g_prof.recs.push_back({stage, flops, e0, e1});
    }
  }
  ~ProfScope() { if (e1) cudaEventRecord(e1, s); }
};

double cplx_mult(Kind k) { return kind_cplx(k) ? 4.0 : 1.0; }
// algorithmic flops of a Hermitian update region (lower elements only) or an LU rectangle
double region_flops(Kind kind, int64_t row0, int64_t col0, int64_t rows, int64_t cols, int K) {
  double elems;
  if (!kind_herm(kind)) {
    elems = (double)rows * (double)cols;
  } else {
    elems = 0;  // count (i, j) with i >= j, i in [row0, row0+rows), j in [col0, col0+cols)
    for (int64_t j = col0; j < col0 + cols; ++j) {
      const int64_t lo = std::max(j, row0), hi = row0 + rows;
      if (hi > lo) elems += (double)(hi - lo);
    }
  }
  return elems * 2.0 * K * cplx_mult(kind);
}

int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// SMs to leave to the lookahead stream while the trailing update (b) of this step runs
// persistently on the rest: minimise max(T1, T2) in units of one (K = nb) update tile, with
//   T1 = (a) this step's lookahead update: ceil(jn / tile) block columns x K = g nb
//      + the next group's chain beside (b): g diag tiles, g panel GEMMs and the g - 1 non-last
//        lookahead updates (K = nb, 2 nb, ... (g-1) nb, one column each)
//   T2 = (b): its tiles at K = g nb on SMs - R.
// g = G at the last step of a group (its (a) covers the next group's G blocks with K = G nb), 1
// otherwise.  (Round 2: the (a) term had counted one column at K = nb whatever g -- a 4x
// underestimate at the paired steps, which starved the next pair's chain of SMs: a timeline of one
// C4 sample showed the trailing kernel idle 5.3 ms, mostly at those steps.)
//
// Split-chain steps (see run_blocked): the chain stream s1 carries only the diag tile, P0 and LT
// (one tile each), s3 the one-wave launches P1 and LR beside the next diag tile, (b) the rest.
// With the period T = max(chain, (b)'s tiles on SMs - R, P1 + LR on R - 1 SMs).
int reserve_sms(int64_t m2, int jn, int sms, int batch, int tile, bool herm, int g = 1, bool split = false) {
  const double side = (double)((m2 + tile - 1) / tile), side_b = (double)((m2 - jn + tile - 1) / tile);
  const double lu = herm ? 1.0 : 2.0;
  const double tb = (herm ? side_b * (side_b + 1) / 2 : side_b * side_b) * batch;  // (b) tiles
  double diag_tiles, chain;
  if (batch == 1 && tile == 128) {
    // the diag tile in update-tile times (~49 us vs ~20-30 us per tile at K = nb)
    diag_tiles = DPP_DIAG_TILES;
    const double cols_a = (double)((jn + tile - 1) / tile);
    const double ta = lu * side * cols_a * g;                 // (a) now
    const double tp = lu * side_b;                            // one panel GEMM (K = nb)
    const double tn = lu * side_b * (g * (g - 1) / 2.0);      // the next non-last (a) updates
    chain = ta + g * tp + tn;
  } else {
    // batches (every launch spans the batch, the diag tiles of all samples share the free SMs
    // with the chain's GEMMs) and the 64-wide complex tiles: the round-1 model, tuned on the UST
    // batch and the complex workloads (the corrected terms above cost 10 % on the UST batch and
    // 1.5-2.6 % on complex samples with three in flight; on one real C4 sample they save 1 ms)
    diag_tiles = DPP_DIAG_TILES_BATCH;
    chain = lu * side * batch + g * lu * side_b * batch;
  }
  int best = 8;
  double best_t = 1e300;
  if (split) {
    const double rest = side - 1.0;  // P1 / LR row tiles
    for (int R = 4; R <= sms / 2; R += 2) {
      const double t1 = diag_tiles + 1.0;
      const double t2 = tb / (sms - R);
      const double t3 = 2.0 * std::ceil(rest / (R - 1));
      const double t = std::max(t1, std::max(t2, t3));
      if (t < best_t - 1e-9) { best_t = t; best = R; }
    }
    return best;
  }
  for (int R = 4; R <= sms / 2; R += 2) {
    const double t1 = g * diag_tiles + chain / R;
    const double t2 = g * tb / (sms - R);
    const double t = t1 > t2 ? t1 : t2;
    if (t < best_t) { best_t = t; best = R; }
  }
  return best;
}

UpdateArgs base_update(Kind kind, int batch, bool vec) {
  UpdateArgs u{};
  u.batch = batch;
  u.vec = vec ? 1 : 0;
  (void)kind;
  return u;
}

// ---------------------------------------------------------------- the blocked factorization
// Grouped trailing updates (lookahead on): the trailing updates of G consecutive steps are applied
// by the group's last step as ONE DMMA pass with K = G nb (the G panels are adjacent columns of the
// factor; their operand copies -- W21 = L21 D1, or U12^T -- are stacked in one buffer), so the
// update kernel's per-tile epilogue and the C read/write are amortized over G times the work.
// G = 3 by default (opts->group; G = 2 is "paired updates").
//
// Default grouping thresholds (opts->group_min_rows = 0): no grouping once the trailing size is
// <= 6144 rows for 128-wide Hermitian blocks, where the diag tile makes the chain the bound near
// the end (measured C4 25.8 -> 26.1 TF/s); 0 for 64-wide Hermitian blocks, whose chain is short
// (complex Hermitian n = 8192: 27.0 vs 26.6 TF/s with 6144); 8192 for LU (two panel GEMMs and two
// lookahead updates per step: n = 8192 27.6 TF/s unpaired vs 26.1 paired; Aztec n = 25600 33.3
// paired vs 32.0); 0 for batches of >= 8 (the chain is shared by the batch and the updates
// dominate throughout: UST 40x40, 256 per launch, 2373 paired vs 2275 samples/s).
int64_t group_threshold(const Opts& o, bool herm, int batch) {
  if (o.group_min_rows >= 0) return o.group_min_rows;
  if (batch >= 8) return 0;
  if (!herm) return 8192;
  return o.nb >= 128 ? DPP_GROUP_MIN_ROWS : 0;
}

// Factors `batch` matrices A + s*strideA (in place), samples b0 + s.
int run_blocked(Kind kind, const Opts& o, int64_t n, void* A, int64_t ld, int64_t strideA, int batch,
                uint64_t seed, uint64_t b0, uint8_t* mask, const uint8_t* forced, double* loglik,
                dpp_info_t* info, char* work, const WsLayout& L, cudaStream_t caller, bool map = false,
                const void* dsrc = nullptr, int64_t dld = 0, int64_t dstride = 0) {
  void* state = work + L.state_off;
  if (n == 0) { CK(launch_zero_state(state, loglik, info, batch, caller)); return DPP_OK; }
  static const char* const kname[] = {"herm_d", "herm_z", "lu_z", "herm_s", "lu_c"};
  NvtxRange call_range("dpp %s n=%lld batch=%d", kname[kind], (long long)n, batch);
  DeviceStreams* ds = nullptr;
  int rc = get_streams(&ds, caller);
  if (rc) return rc;
  std::lock_guard<std::recursive_mutex> lk(ds->mu);
  const int nb = o.nb;
  const bool la = o.lookahead > 0;
  cudaStream_t s1 = la ? ds->s1 : caller, s2 = la ? ds->s2 : caller, s3 = la ? ds->s3 : caller;
  if (la) {
    CK(cudaEventRecord(ds->ev_start, caller));
    CK(cudaStreamWaitEvent(s1, ds->ev_start, 0));
    CK(cudaStreamWaitEvent(s2, ds->ev_start, 0));
    CK(cudaStreamWaitEvent(s3, ds->ev_start, 0));
  }
  const size_t es = esize(kind);
  const bool herm = kind_herm(kind);
  char* Ab = reinterpret_cast<char*>(A);
  // 16-byte aligned columns: the TMA / cp.async 16-byte operand paths
  const bool vec = ((size_t)ld * es) % 16 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
                   ((size_t)strideA * es) % 16 == 0;
  auto upd = [&](UpdateArgs u, cudaStream_t s) -> cudaError_t {
    u.generic = o.generic ? 1 : 0;
    u.fp32_simt = o.fp32_simt ? 1 : 0;
    if (L.tcs_bytes) {
      u.tcs = work + L.tcs_off + ((la && s == s2) ? L.tcs_bytes : 0);
      u.tcs_bytes = (int64_t)L.tcs_bytes;
    }
    return launch_update(kind, u, s);
  };
  void* Bm = work + L.bm_off;
  void* Am = work + L.am_off;
  // Deferred copy (dsrc != null: the batched entry points with a device kernel K at dsrc, leading
  // dimension dld, stride dstride): instead of copying K's lower triangle into the workspace before
  // the factorization, columns [0, copied) are valid in the workspace and the first update launch
  // touching a block column range at `copied` reads its C values from K itself (UpdateArgs::csrc)
  // and writes the workspace -- the lookahead updates of the first block columns and the first
  // trailing update (the rest of the matrix), so only the first block column is ever copied.  Any
  // other first touch copies the columns it needs beforehand (ensure_cols).  Hermitian
  // warp-specialized path only (its updates never write above the diagonal; the sampler reads only
  // the lower triangle).
  int64_t copied = dsrc ? 0 : n;
  auto ensure_cols = [&](int64_t c1, cudaStream_t s) -> int {
    if (c1 <= copied) return DPP_OK;
    ProfScope pa(4, 0.0, s);
    CK(launch_copy_matrix(esize(kind), dsrc, dld, dstride, A, ld, strideA, (int)n, batch, true, s, (int)copied,
                          (int)c1));
    copied = c1;
    return DPP_OK;
  };
  // a launch whose C region starts at column c0 (and row c0) and ends at column c1: read from K if
  // nothing in [c0, c1) has been touched yet
  auto defer_to = [&](UpdateArgs& ua, int64_t c0, int64_t c1) {
    if (copied != c0 || !vec || o.generic) return false;
    ua.csrc = reinterpret_cast<const char*>(dsrc) + (size_t)(c0 + c0 * dld) * esize(kind);
    ua.ldcs = dld; ua.strideCs = dstride;
    copied = c1;
    return true;
  };
  int step = 0;
  bool have_rest = false;
  int gpos = -1;            // position of the previous step in its group (-1: none)
  bool prev_glast = false;  // the previous step was the last of a group
  bool lr_pending = false;  // the previous step's lookahead rows below its diagonal tile run on s3
  bool used_s3 = false;
  const int sms = device_sms();
  // Head block: when nb does not divide n, the FIRST block takes the remainder (n mod nb) so that
  // every trailing region is a whole number of tiles (a ragged last block would leave a partly
  // empty tile row and column in every trailing update: UST n = 3120, 2472 -> 2574 samples/s).
  // Only when the remainder keeps every block origin 16-byte aligned (the TMA operand copies): a
  // multiple of 16 / element-size rows.  Pivot draws are by global index (reading R2), so the
  // blocking does not change the sample.
  const int64_t rem = n % nb;
  const int64_t head = (n > nb && rem && rem % (int64_t)(16 / es) == 0) ? rem : 0;
  // With grouping the head block is position 0 of group 0 (its trailing update deferred like any
  // non-last position: a separate K = head pass over the whole trailing matrix is HBM-bound -- the
  // UST batch, n = 3120, spent 28 ms of a 381 ms step in it).  Position gp of a group starts at
  // column offset goff(gp) from the group's first column (the head shifts group 0's later blocks).
  const int G = o.group;
  const int64_t gthr = group_threshold(o, herm, batch);
  auto blk = [&](int64_t j) -> int64_t { return (head && j == 0) ? head : std::min<int64_t>(nb, n - j); };
  for (int64_t j0 = 0; j0 < n; j0 += blk(j0), ++step) {
    const int jb = (int)blk(j0);
    const int64_t j1 = j0 + jb, m2 = n - j1;
    NvtxRange step_range("step %d j0=%lld", step, (long long)j0);
    double* dvec = herm ? reinterpret_cast<double*>(work + L.d_off) + (size_t)(step & 1) * batch * nb : nullptr;
    // LU: U12^T (m2 x jb, ld = ldk, K-major GEMM operand); Hermitian: W21 = L21 D1 (same shape);
    // double-buffered like D1
    const int64_t strideU = L.strideU;
    char* UT = work + L.ut_off + (size_t)(step & 1) * batch * strideU * es;
    // grouping: steps (G g .. G g + G-1) share the group buffer (g & 1) of G panels per sample
    const bool grouping = la && G > 1 && nb == (int)std::min<int64_t>(nb, n);
    const int64_t strideW = (int64_t)std::max(G, 2) * strideU;
    const int gstep = step;
    char* WP = work + L.ut_off + (size_t)((gstep / G) & 1) * batch * strideW * es;
    const int64_t w0 = (head && gstep < G) ? head : nb;  // width of the group's position 0
    auto goff = [&](int g) -> int64_t { return g == 0 ? 0 : w0 + (int64_t)(g - 1) * nb; };
    // group roles: a group starts at a step that is a multiple of G when all its G blocks are full
    // width, its last step has a trailing region of its own, and the trailing updates still dominate
    // (near the end the chain is the bound, and a group's G-wide lookahead update lengthens it).
    // Every step but the last defers its trailing update; the last applies all G panels.  Each
    // step's operand panel (W21 or U12^T) goes to its slot of the group buffer, slot i shifted down
    // by i nb rows so that row r of every slot is the same matrix row.
    int gp = -1;  // this step's position in its group
    if (grouping) {
      if (gpos >= 0 && gpos < G - 1) {
        gp = gpos + 1;
      } else if (gstep >= 0 && gstep % G == 0 && m2 - (int64_t)(G - 1) * nb > 0 && m2 > gthr) {
        gp = 0;
      }
    }
    const bool glast = gp == G - 1, gnonlast = gp >= 0 && !glast;
    // Split chain (ungrouped Hermitian steps of one fp64 sample): the only work the next diag tile
    // waits for is the panel's first row tile P0 (the rows of the next block) and the lookahead
    // update LT of the next diagonal tile; they stay on the chain stream s1, while the panel's other
    // rows P1 and the lookahead update of the rows below the next tile LR run on s3 beside the next
    // diag tile.  Same tiles, same arithmetic as the unsplit launches: bit-identical results.
    // Only near the end (m2 <= 3072: the steps whose chain is the bound; above it the one-wave P1 /
    // LR launches cost the trailing update more SMs than the chain saves -- measured on C4).
    const bool split = la && !o.no_split && batch == 1 && herm && kind != HERM_S && gp < 0 && m2 > nb &&
                       m2 <= DPP_SPLIT_ROWS;
    const int64_t jsp = std::min<int64_t>(nb, m2);  // rows of P0 / LT (= the ungrouped jn)
    // real 128-blocks: P0 and LT as ONE single-CTA launch (next_tile.cu)
    const bool fuse = split && kind == HERM_D && nb == 128 && jb == 128 && vec && !o.generic;
    // my slot: its columns at goff(gp) of the group buffer, shifted down by gp nb rows so that row
    // r of the stacked operand is the same matrix row in every slot
    char* const PH = WP + (size_t)(gp >= 0 ? goff(gp) * L.ldk + (int64_t)gp * nb : (step % G) * strideU) * es;
    char* const WG = WP + (size_t)(gp > 0 ? gp * nb : 0) * es;  // the stacked operand of panels 0..gp
    const int64_t jg0 = gp > 0 ? j0 - goff(gp) : j0;  // the group's first column
    bool copyback = false;  // LU: the U12^T -> A12 copy deferred to the trailing stream
    const char* cb_src = nullptr;
    char* cb_dst = nullptr;
    int64_t cb_stride = 0;
    // ---- stage 1
    DiagArgs d{};
    d.A = A; d.ld = ld; d.strideA = strideA; d.n = n; d.j0 = j0; d.tcol = j0; d.jb = jb; d.seed = seed; d.b0 = b0;
    d.mask = mask; d.forced = forced; d.state = state; d.loglik = loglik; d.info = info;
    d.tie_tol = o.tie_tol; d.range_tol = o.range_tol; d.batch = batch; d.map = map ? 1 : 0;
    d.need_ops = m2 > 0; d.Bm = Bm; d.Am = Am; d.dvec = dvec; d.ldm = nb; d.strideM = L.strideM;
    // the diag tile and the panel read block column j0; a split step's LT / LR (s3, ordered after P0
    // only) also the next block's columns, copied here ahead of everything the step launches
    if ((rc = ensure_cols(split ? j1 + jsp : j1, s1))) return rc;
    {
      const double fl = (herm ? 1.0 : 2.0) * jb * (double)jb * jb / 3.0 * cplx_mult(kind) * batch;
      ProfScope ps(0, fl, s1);
      CK(launch_diag(kind, nb, d, s1));
    }
    if (m2 <= 0) break;
    if (split) CK(cudaEventRecord(ds->ev_diag, s1));
    // the panel reads this block column below the diagonal tile: the previous step's LR (s3)
    if (lr_pending) { CK(cudaStreamWaitEvent(s1, ds->ev_lr, 0)); lr_pending = false; }
    // ---- stage 2: panel GEMMs with the tile operators (in place)
    {
      const double fl = (herm ? 1.0 : 2.0) * (double)m2 * jb * jb * cplx_mult(kind) * batch;  // TRSM count
      // (split: P1's share is bracketed on s3, P0's with the fused launch when there is one)
      ProfScope ps(1, split ? (fuse ? 0.0 : fl * jsp / m2) : fl, s1);
      UpdateArgs p = base_update(kind, batch, vec);
      p.Aop = Ab + (size_t)(j1 + j0 * ld) * es; p.lda = ld; p.strideA = strideA;   // A21
      p.Bop = Bm; p.ldb = nb; p.strideB = L.strideM;
      p.C = Ab + (size_t)(j1 + j0 * ld) * es; p.ldc = ld; p.strideC = strideA;    // L21 in place
      p.a_rows = (int)m2; p.b_rows = jb; p.K = jb; p.btri = 1;
      p.row0 = 0; p.col0 = 0; p.rows = (int)m2; p.cols = jb;
      if (herm) {
        // and the pre-scaled copy W21 = L21 D1 (the trailing-update operand) into its panel slot
        // (written by the panel kernel's epilogue when it is the warp-specialized one)
        p.wout = grouping ? PH : UT; p.ldw = L.ldk; p.strideWo = grouping ? strideW : strideU;
        p.wscale = dvec; p.wsstride = nb;
      }
      if (split) {
        UpdateArgs p0 = p, p1 = p;
        if (!fuse) {
          p0.rows = (int)jsp;
          CK(upd(p0, s1));
          CK(cudaEventRecord(ds->ev_p0, s1));
        }
        CK(cudaStreamWaitEvent(s3, ds->ev_diag, 0));
        p1.row0 = (int)jsp; p1.rows = (int)(m2 - jsp);
        { ProfScope ps1(1, fl * (m2 - jsp) / m2, s3); CK(upd(p1, s3)); }
        CK(cudaEventRecord(ds->ev_p1, s3));
        used_s3 = true;
      } else {
        CK(upd(p, s1));
      }
      if (!herm) {
        // U12 = L11^-1 A12 = A12 - Am A12 (Am = I - L11^-1), computed transposed so that every
        // operand is K-major:  U12^T = A12^T - A12^T Am^T  in the U12^T buffer, then copied back.
        char* A12 = Ab + (size_t)(j0 + j1 * ld) * es;
        char* const UTs = grouping ? PH : UT;  // my U12^T panel (grouping: my slot of the group buffer)
        const int64_t sU = grouping ? strideW : strideU;
        { ProfScope pa(4, 0.0, s1); CK(launch_transpose(es, A12, ld, strideA, UTs, L.ldk, sU, jb, (int)m2, batch, s1)); }
        UpdateArgs q = base_update(kind, batch, vec);
        q.Aop = UTs; q.lda = L.ldk; q.strideA = sU;                                // A12^T (j, k)
        q.Bop = Am; q.ldb = nb; q.strideB = L.strideM;                             // Am (i, k)
        q.C = UTs; q.ldc = L.ldk; q.strideC = sU;                                  // U12^T in place
        q.a_rows = (int)m2; q.b_rows = jb; q.K = jb; q.btri = 1;
        q.row0 = 0; q.col0 = 0; q.rows = (int)m2; q.cols = jb;
        CK(upd(q, s1));
        if (!la) {
          ProfScope pa(4, 0.0, s1);
          CK(launch_transpose(es, UTs, L.ldk, sU, A12, ld, strideA, (int)m2, jb, batch, s1));  // U12 -> K
        } else {
          // U12 -> K is only output (no later step reads A12): off the chain, on the trailing
          // stream once the panel is done (below)
          copyback = true; cb_src = UTs; cb_stride = sU; cb_dst = A12;
        }
      }
    }
    // ---- stage 3 operands
    UpdateArgs u = base_update(kind, batch, vec);
    u.Aop = Ab + (size_t)(j1 + j0 * ld) * es; u.lda = ld; u.strideA = strideA;  // L21
    if (herm && grouping) {
      // W21 of this step is in its slot of the group buffer (written with the panel; the
      // K = (gp+1) nb operand of group position gp starts at row gp nb of slot 0)
      u.Aop = gp >= 0 ? WG : PH; u.lda = L.ldk; u.strideA = strideW;  // W21 of panels 0..gp
      u.Bop = Ab + (size_t)(j1 + jg0 * ld) * es; u.ldb = ld; u.strideB = strideA;
      u.mask = 1; u.conj = (kind == HERM_Z);
    } else if (herm) {
      // A22 -= W21 L21^H with W21 = L21 D1 (pre-scaled copy written with the panel; the DMMA loop
      // does no scaling)
      u.Aop = UT; u.lda = L.ldk; u.strideA = strideU;  // W21
      u.Bop = Ab + (size_t)(j1 + j0 * ld) * es; u.ldb = ld; u.strideB = strideA;  // L21 (conjugated on load)
      u.mask = 1; u.conj = (kind == HERM_Z);
    } else if (grouping) {
      u.Aop = Ab + (size_t)(j1 + jg0 * ld) * es;                                    // L21 of panels 0..gp
      u.Bop = gp >= 0 ? WG : PH; u.ldb = L.ldk; u.strideB = strideW;                // U12^T of panels 0..gp
    } else {
      u.Bop = UT; u.ldb = L.ldk; u.strideB = strideU;  // U12^T (j, k), K-major
    }
    u.C = Ab + (size_t)(j1 + j1 * ld) * es; u.ldc = ld; u.strideC = strideA;
    u.a_rows = (int)m2; u.b_rows = (int)m2; u.K = (int)((gp > 0 ? goff(gp) : 0) + jb);
    // width of the lookahead region: the next block -- or, at the last step of a group, the next
    // group's G blocks, so the next group's whole diag/panel chain runs under this group's update
    const int jn = (int)std::min<int64_t>(glast ? (int64_t)G * nb : nb, m2);
    if (!la) {
      u.row0 = 0; u.col0 = 0; u.rows = (int)m2; u.cols = (int)m2; u.tri = herm;
      if (!defer_to(u, j1, n) && (rc = ensure_cols(n, s1))) return rc;
      ProfScope ps(3, region_flops(kind, 0, 0, m2, m2, jb) * batch, s1);
      CK(upd(u, s1));
      continue;
    }
    if (!split) CK(cudaEventRecord(ds->ev_panel, s1));
    if (copyback) {
      CK(cudaStreamWaitEvent(s2, ds->ev_panel, 0));
      ProfScope pa(4, 0.0, s2);
      CK(launch_transpose(es, cb_src, L.ldk, cb_stride, cb_dst, ld, strideA, (int)m2, jb, batch, s2));  // U12 -> K
      copyback = false;
    }
    // (a) next block column [0, jn) x rows [0, m2)  (+ LU: next block row [0, jn) x cols [jn, m2))
    // (a non-last step of a group needs no wait: its lookahead block was covered by the previous
    // group's lookahead update and is not part of the previous trailing update)
    if (have_rest && !(gnonlast && (gp > 0 || prev_glast))) CK(cudaStreamWaitEvent(s1, ds->ev_rest, 0));
    prev_glast = glast;
    if (split) {
      // LT: the next diagonal tile (chain, s1); LR: the rows below it (s3, after P0 and P1)
      UpdateArgs lt = u, lr = u;
      lt.row0 = 0; lt.col0 = 0; lt.rows = (int)jsp; lt.cols = (int)jsp; lt.tri = 0;
      if (fuse) {
        NextTileArgs nt{};
        nt.A21 = reinterpret_cast<double*>(Ab + (size_t)(j1 + j0 * ld) * es); nt.ld = ld;
        nt.Bm = reinterpret_cast<const double*>(Bm); nt.ldm = nb; nt.d = dvec;
        nt.W21 = reinterpret_cast<double*>(grouping ? PH : UT); nt.ldw = L.ldk;
        nt.C = reinterpret_cast<double*>(Ab + (size_t)(j1 + j1 * ld) * es);
        ProfScope ps(2, region_flops(kind, 0, 0, jsp, jsp, u.K) + (double)jsp * jb * jb, s1);
        CK(launch_next_tile(nt, s1));
        CK(cudaEventRecord(ds->ev_p0, s1));
      } else {
        ProfScope ps(2, region_flops(kind, 0, 0, jsp, jsp, u.K), s1);
        CK(upd(lt, s1));
      }
      CK(cudaStreamWaitEvent(s3, ds->ev_p0, 0));
      if (have_rest) CK(cudaStreamWaitEvent(s3, ds->ev_rest, 0));
      lr.row0 = (int)jsp; lr.col0 = 0; lr.rows = (int)(m2 - jsp); lr.cols = (int)jsp; lr.tri = 0;
      {
        ProfScope ps(2, region_flops(kind, jsp, 0, m2 - jsp, jsp, u.K), s3);
        CK(upd(lr, s3));
      }
      CK(cudaEventRecord(ds->ev_lr, s3));
      lr_pending = true;
    } else {
      UpdateArgs ua = u;
      ua.row0 = 0; ua.col0 = 0; ua.rows = (int)m2; ua.cols = jn; ua.tri = 0;
      if (!defer_to(ua, j1, j1 + jn) && (rc = ensure_cols(j1 + jn, s1))) return rc;
      double fl = region_flops(kind, 0, 0, m2, jn, ua.K);
      if (!herm && m2 > jn) fl += region_flops(kind, 0, jn, jn, m2 - jn, jb);
      ProfScope ps(2, fl * batch, s1);
      CK(upd(ua, s1));
      if (!herm && m2 > jn) {
        UpdateArgs ur = u;
        ur.row0 = 0; ur.col0 = jn; ur.rows = jn; ur.cols = (int)(m2 - jn); ur.tri = 0;
        CK(upd(ur, s1));
      }
    }
    // (b) the rest [jn, m2)^2 on S2, persistently on the SMs the lookahead chain leaves free
    gpos = gp;  // a non-last position: the group's last step applies this step's trailing update
    if (m2 > jn && !gnonlast) {
      if (split) {
        CK(cudaStreamWaitEvent(s2, ds->ev_p0, 0));
        CK(cudaStreamWaitEvent(s2, ds->ev_p1, 0));
      } else {
        CK(cudaStreamWaitEvent(s2, ds->ev_panel, 0));
      }
      UpdateArgs ub = u;
      ub.row0 = jn; ub.col0 = jn; ub.rows = (int)(m2 - jn); ub.cols = (int)(m2 - jn);
      ub.tri = herm;
      if (defer_to(ub, j1 + jn, n)) {
        ub.csrc = reinterpret_cast<const char*>(ub.csrc) - (size_t)(jn + jn * dld) * esize(kind);  // origin at u.C's
      } else if ((rc = ensure_cols(n, s2))) {
        return rc;
      }
      if (vec)
        ub.grid_limit = sms - reserve_sms(m2, jn, sms, batch, kind_cplx(kind) ? 64 : 128, herm, glast ? G : 1, split);
      {
        ProfScope ps(3, region_flops(kind, jn, jn, m2 - jn, m2 - jn, ub.K) * batch, s2);
        CK(upd(ub, s2));
      }
      CK(cudaEventRecord(ds->ev_rest, s2));
      have_rest = true;
    }
  }
  if (la) {
    CK(cudaEventRecord(ds->ev_done1, s1));
    CK(cudaEventRecord(ds->ev_done2, s2));
    CK(cudaStreamWaitEvent(caller, ds->ev_done1, 0));
    CK(cudaStreamWaitEvent(caller, ds->ev_done2, 0));
    if (used_s3) {
      CK(cudaEventRecord(ds->ev_done3, s3));
      CK(cudaStreamWaitEvent(caller, ds->ev_done3, 0));
    }
  }
  return DPP_OK;
}

int validate(int64_t n, int64_t ld, const void* K, const uint8_t* mask, const double* loglik) {
  if (n < 0 || ld < std::max<int64_t>(1, n)) return DPP_EINVAL;
  if (n > (int64_t)1 << 30) return DPP_EINVAL;
  if (n > 0 && (!K || !mask)) return DPP_EINVAL;
  if (!loglik) return DPP_EINVAL;
  return DPP_OK;
}

int sample_inplace(Kind kind, int64_t n, void* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                   dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, cudaStream_t st,
                   bool map = false) {
  Opts o;
  int rc = resolve_opts(kind, opts, &o);
  if (rc) return rc;
  if ((rc = validate(n, ld, K, mask, loglik))) return rc;
  if ((rc = check_device())) return rc;
  WsLayout L = layout(kind, 1, n, o, false, false);
  if (!work || work_bytes < L.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  if (reinterpret_cast<uintptr_t>(K) % esize(kind)) return DPP_EINVAL;
  return run_blocked(kind, o, n, K, ld, 0, 1, seed, 0, mask, o.forced, loglik, info, reinterpret_cast<char*>(work),
                     L, st, map);
}

int sample_batched(Kind kind, int64_t batch, int64_t n, const void* K, int64_t ld, int64_t strideK, uint64_t seed,
                   uint64_t b0, uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                   size_t work_bytes, cudaStream_t st, bool host, bool sync = true) {
  Opts o;
  int rc = resolve_opts(kind, opts, &o);
  if (rc) return rc;
  if (batch < 0 || strideK < 0) return DPP_EINVAL;
  if (batch == 0) return DPP_OK;
  if ((rc = validate(n, ld, K, mask, loglik))) return rc;
  if (strideK > 0 && strideK < ld * std::max<int64_t>(n, 1)) return DPP_EINVAL;
  if ((rc = check_device())) return rc;
  const int64_t chunk = o.batch_chunk > 0 ? std::min(o.batch_chunk, batch) : batch;
  if (chunk > 65535) return DPP_EINVAL;
  WsLayout L = layout(kind, chunk, n, o, true, host);
  if (!work || work_bytes < L.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  char* w = reinterpret_cast<char*>(work);
  const size_t es = esize(kind);
  const cudaMemcpyKind ck = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  char* Kc = w + L.k_off;
  // Kernels are copied into their workspace slots.  Hermitian kernels read only the lower
  // triangle, so only it is moved: device sources with one batched copy kernel, host sources with
  // one 2-D DMA copy per 128-column block of rows [c, n) -- about half the bytes of the full
  // matrix (this halves the host->device time of the _host entry points).
  const bool lower = kind_herm(kind);
  // device kernels of the fp64 Hermitian samplers: the copy into the workspace is deferred into the
  // first updates (run_blocked), which read K directly -- needs the lookahead schedule, the
  // warp-specialized update kernel and 16-byte aligned K columns
  const bool defer = !host && n > 0 && (kind == HERM_D || kind == HERM_Z) && o.lookahead > 0 && !o.generic &&
                     reinterpret_cast<uintptr_t>(K) % 16 == 0 && ((size_t)ld * es) % 16 == 0 &&
                     ((size_t)strideK * es) % 16 == 0 && ((size_t)L.ldk * es) % 16 == 0;
  auto h2d = [&](char* dst, const char* src) -> int {
    if (!lower) {
      CK(cudaMemcpy2DAsync(dst, (size_t)L.ldk * es, src, (size_t)ld * es, (size_t)n * es, (size_t)n, ck, st));
      return DPP_OK;
    }
    constexpr int64_t CB = 128;
    for (int64_t c = 0; c < n; c += CB) {
      const int64_t w_ = std::min<int64_t>(CB, n - c);
      CK(cudaMemcpy2DAsync(dst + (size_t)(c + c * L.ldk) * es, (size_t)L.ldk * es, src + (size_t)(c + c * ld) * es,
                           (size_t)ld * es, (size_t)(n - c) * es, (size_t)w_, ck, st));
    }
    return DPP_OK;
  };
  for (int64_t c0 = 0; c0 < batch; c0 += chunk) {
    const int cb = (int)std::min<int64_t>(chunk, batch - c0);
    if (n > 0) {
      if (host && strideK == 0) {
        // one host->device transfer of the shared kernel, then device-side replication
        if ((rc = h2d(Kc, reinterpret_cast<const char*>(K)))) return rc;
        ProfScope pa(4, 0.0, st);
        if (cb > 1)
          CK(launch_copy_matrix(es, Kc, L.ldk, 0, Kc + (size_t)L.strideK * es, L.ldk, L.strideK, (int)n,
                                cb - 1, lower, st));
      } else if (host) {
        for (int s = 0; s < cb; ++s)
          if ((rc = h2d(Kc + (size_t)s * L.strideK * es,
                        reinterpret_cast<const char*>(K) + (size_t)(strideK * (c0 + s)) * es))) return rc;
      } else if (!defer) {
        ProfScope pa(4, 0.0, st);
        CK(launch_copy_matrix(es, reinterpret_cast<const char*>(K) + (size_t)(strideK * c0) * es, ld,
                              strideK, Kc, L.ldk, L.strideK, (int)n, cb, lower, st));
      }
    }
    uint8_t* mk = host ? reinterpret_cast<uint8_t*>(w + L.mask_off) : mask + c0 * n;
    double* llk = host ? reinterpret_cast<double*>(w + L.ll_off) : loglik + c0;
    dpp_info_t* ifo = host ? (info ? reinterpret_cast<dpp_info_t*>(w + L.info_off) : nullptr) : (info ? info + c0 : nullptr);
    const uint8_t* fz = o.forced ? o.forced + c0 * n : nullptr;
    rc = run_blocked(kind, o, n, Kc, L.ldk, L.strideK, cb, seed, b0 + (uint64_t)c0, mk, fz, llk, ifo, w, L, st,
                     false, defer ? reinterpret_cast<const char*>(K) + (size_t)(strideK * c0) * es : nullptr, ld,
                     strideK);
    if (rc) return rc;
    if (host) {
      if (n > 0) CK(cudaMemcpyAsync(mask + c0 * n, mk, (size_t)cb * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(loglik + c0, llk, 8 * (size_t)cb, cudaMemcpyDeviceToHost, st));
      if (info) CK(cudaMemcpyAsync(info + c0, ifo, sizeof(dpp_info_t) * (size_t)cb, cudaMemcpyDeviceToHost, st));
    }
  }
  if (host && sync) CK(cudaStreamSynchronize(st));
  return DPP_OK;
}

}  // namespace

extern "C" {

size_t dpp_workspace_bytes(int op, int64_t batch, int64_t n, const dpp_opts_t* opts) {
  if ((op & 0x7) > 4 || n < 0 || batch < 0) return 0;
  const Kind kind = (Kind)(op & 0x7);
  Opts o;
  if (resolve_opts(kind, opts, &o)) return 0;
  const bool batched = (op & (DPP_OP_BATCHED | DPP_OP_HOST)) != 0;
  const bool host = (op & DPP_OP_HOST) != 0;
  int64_t chunk = batched ? batch : 1;
  if (batched && o.batch_chunk > 0) chunk = std::min(chunk, o.batch_chunk);
  chunk = std::max<int64_t>(chunk, 1);
  return layout(kind, chunk, n, o, batched, host).total;
}

int dpp_sample_herm_d(int64_t n, double* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                      dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(HERM_D, n, K, ld, seed, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream);
}
int dpp_sample_herm_z(int64_t n, dpp_complex_t* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                      dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(HERM_Z, n, K, ld, seed, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream);
}
int dpp_sample_lu_z(int64_t n, dpp_complex_t* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                    dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(LU_Z, n, K, ld, seed, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream);
}

// single precision (reading R19)
int dpp_sample_herm_s(int64_t n, float* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                      dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(HERM_S, n, K, ld, seed, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream);
}
int dpp_sample_lu_c(int64_t n, dpp_complex64_t* K, int64_t ld, uint64_t seed, uint8_t* mask, double* loglik,
                    dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(LU_C, n, K, ld, seed, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream);
}

// greedy MAP inference: the same blocked factorization, decisions Re p >= 1/2
int dpp_map_herm_d(int64_t n, double* K, int64_t ld, uint8_t* mask, double* loglik, dpp_info_t* info,
                   const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(HERM_D, n, K, ld, 0, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream, true);
}
int dpp_map_herm_z(int64_t n, dpp_complex_t* K, int64_t ld, uint8_t* mask, double* loglik, dpp_info_t* info,
                   const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(HERM_Z, n, K, ld, 0, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream, true);
}
int dpp_map_lu_z(int64_t n, dpp_complex_t* K, int64_t ld, uint8_t* mask, double* loglik, dpp_info_t* info,
                 const dpp_opts_t* opts, void* work, size_t work_bytes, dpp_stream_t stream) {
  return sample_inplace(LU_Z, n, K, ld, 0, mask, loglik, info, opts, work, work_bytes, (cudaStream_t)stream, true);
}

#define BATCHED(name, kind, T, host, sync)                                                                    \
  int name(int64_t batch, int64_t n, const T* K, int64_t ld, int64_t strideK, uint64_t seed, uint64_t b0,     \
           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,                 \
           size_t work_bytes, dpp_stream_t stream) {                                                           \
    return sample_batched(kind, batch, n, K, ld, strideK, seed, b0, mask, loglik, info, opts, work, work_bytes, \
                          (cudaStream_t)stream, host, sync);                                                   \
  }
BATCHED(dpp_sample_herm_d_batched, HERM_D, double, false, true)
BATCHED(dpp_sample_herm_z_batched, HERM_Z, dpp_complex_t, false, true)
BATCHED(dpp_sample_lu_z_batched, LU_Z, dpp_complex_t, false, true)
BATCHED(dpp_sample_herm_d_host, HERM_D, double, true, true)
BATCHED(dpp_sample_herm_z_host, HERM_Z, dpp_complex_t, true, true)
BATCHED(dpp_sample_lu_z_host, LU_Z, dpp_complex_t, true, true)
BATCHED(dpp_sample_herm_d_host_async, HERM_D, double, true, false)
BATCHED(dpp_sample_herm_z_host_async, HERM_Z, dpp_complex_t, true, false)
BATCHED(dpp_sample_lu_z_host_async, LU_Z, dpp_complex_t, true, false)
BATCHED(dpp_sample_herm_s_batched, HERM_S, float, false, true)
BATCHED(dpp_sample_lu_c_batched, LU_C, dpp_complex64_t, false, true)
#undef BATCHED

int dpp_philox_uniforms(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u, dpp_stream_t stream) {
  if (count < 0 || (count > 0 && !u)) return DPP_EINVAL;
  return launch_uniforms(seed, j0, b, count, u, (cudaStream_t)stream) == cudaSuccess ? DPP_OK : DPP_ECUDA;
}

int dpp_probe_update_d(int64_t m, int32_t K, const double* W, const double* L, int64_t ldo, double* C, int64_t ldc,
                       float* ms, dpp_stream_t stream) {
  if (m <= 0 || K <= 0 || !W || !L || !C || !ms || ldo < m || ldc < m) return DPP_EINVAL;
  int rc = check_device();
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  UpdateArgs u{};
  u.Aop = W; u.lda = ldo; u.Bop = L; u.ldb = ldo; u.mask = 1;
  u.C = C; u.ldc = ldc;
  u.a_rows = (int)m; u.b_rows = (int)m; u.K = K; u.batch = 1;
  u.vec = (ldo % 2 == 0 && ldc % 2 == 0 && reinterpret_cast<uintptr_t>(W) % 16 == 0 &&
           reinterpret_cast<uintptr_t>(L) % 16 == 0 && reinterpret_cast<uintptr_t>(C) % 16 == 0) ? 1 : 0;
  u.row0 = 0; u.col0 = 0; u.rows = (int)m; u.cols = (int)m; u.tri = 1;
  u.grid_limit = device_sms();  // persistent over every SM, as the trailing update with nothing beside it
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  const cudaError_t le = launch_update(HERM_D, u, st);
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  CK(le);
  CK(cudaEventElapsedTime(ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return DPP_OK;
}

int dpp_profile_begin_stages(unsigned stage_mask) {
  if (!(stage_mask & 0x1fu)) return DPP_EINVAL;
  g_prof.recs.clear();
  g_prof.used = 0;
  g_prof.mask = stage_mask & 0x1fu;
  g_prof.on = true;
  return DPP_OK;
}

int dpp_profile_begin(void) { return dpp_profile_begin_stages(0x1fu); }

int dpp_profile_end(dpp_profile_t* out) { return dpp_profile_end_records(out, nullptr, 0, nullptr); }

int dpp_profile_end_records(dpp_profile_t* out, double* records, int64_t max_records, int64_t* count) {
  g_prof.on = false;
  if (!out || max_records < 0 || (max_records > 0 && !records)) return DPP_EINVAL;
  if (count) *count = (int64_t)g_prof.recs.size();
  std::memset(out, 0, sizeof(*out));
  std::vector<std::pair<double, double>> iv[5];  // launch intervals per stage, from the first event
  const cudaEvent_t ref = g_prof.recs.empty() ? nullptr : g_prof.recs.front().e0;
  for (auto& r : g_prof.recs) {
    if (cudaEventSynchronize(r.e1) != cudaSuccess) return DPP_ECUDA;
    float ms = 0.f, t0 = 0.f, t1 = 0.f;
    if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) return DPP_ECUDA;
    if (cudaEventElapsedTime(&t0, ref, r.e0) != cudaSuccess) return DPP_ECUDA;
    if (cudaEventElapsedTime(&t1, ref, r.e1) != cudaSuccess) return DPP_ECUDA;
    out->launches[r.stage] += 1;
    out->ms[r.stage] += ms;
    out->flops[r.stage] += r.flops;
    if (r.flops > out->top_flops[r.stage]) { out->top_flops[r.stage] = r.flops; out->top_ms[r.stage] = ms; }
    iv[r.stage].push_back({(double)t0, (double)t1});
    const int64_t i = (int64_t)(&r - g_prof.recs.data());
    if (i < max_records) {  // (stage, start ms, end ms, flops) in issue order
      records[4 * i + 0] = r.stage; records[4 * i + 1] = t0; records[4 * i + 2] = t1; records[4 * i + 3] = r.flops;
    }
  }
  for (int st = 0; st < 5; ++st) {  // length of the union of the stage's launch intervals
    // offsets are from the first record ISSUED, so intervals on other streams may start before
    // it (negative offsets): the sweep starts from the earliest interval, not from 0
    std::sort(iv[st].begin(), iv[st].end());
    double u = 0.0;
    if (!iv[st].empty()) {
      double lo = iv[st][0].first, hi = iv[st][0].second;
      for (auto& p : iv[st]) {
        if (p.first > hi) { u += hi - lo; lo = p.first; hi = p.second; }
        else if (p.second > hi) hi = p.second;
      }
      u += hi - lo;
    }
    out->ms_union[st] = u;
  }
  g_prof.recs.clear();
  g_prof.used = 0;
  return DPP_OK;
}

const char* dpp_strerror(int code) {
  switch (code) {
    case DPP_OK: return "ok";
    case DPP_EINVAL: return "invalid argument";
    case DPP_EWORKSPACE: return "workspace missing, too small or misaligned";
    case DPP_ECUDA: return "CUDA error";
    case DPP_ENCCL: return "NCCL error";
    case DPP_EUNSUPPORTED: return "unsupported device (needs sm_100)";
  }
  return "unknown error";
}

const char* dpp_version(void) { return "dpp-b200 0.2.0 (sm_100a)"; }

}  // extern "C"
