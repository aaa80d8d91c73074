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
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace dpp;

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x, size_t a = ALIGN) { return (x + a - 1) / a * a; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct Opts {
  int nb;
  int lookahead;
  double tie_tol, range_tol;
  const uint8_t* forced;
  int64_t batch_chunk;
};

int resolve_opts(Kind kind, const dpp_opts_t* o, Opts* r) {
  r->nb = (o && o->nb) ? o->nb : (kind_cplx(kind) ? 64 : 128);
  r->lookahead = o ? o->lookahead : 1;
  r->tie_tol = (o && o->tie_tol > 0) ? o->tie_tol : 1e-9;
  r->range_tol = (o && o->range_tol > 0) ? o->range_tol : 1e-8;
  r->forced = o ? o->forced : nullptr;
  r->batch_chunk = o ? o->batch_chunk : 0;
  if (r->nb != 32 && r->nb != 64 && r->nb != 128) return DPP_EINVAL;
  if (kind_cplx(kind) && r->nb > 64) return DPP_EINVAL;  // complex tile must fit the diag kernel
  if (r->lookahead < 0 || r->lookahead > 1) return DPP_EINVAL;
  if (r->batch_chunk < 0) return DPP_EINVAL;
  return DPP_OK;
}

size_t esize(Kind k) { return kind_esize(k); }

int group_size();

// Workspace layout (all regions 256-byte aligned):
//   [SampleState x chunk]
//   [panel operators: Bm (and Am for LU), nb x nb per sample]
//   [D1 double buffer (Hermitian): 2 x chunk x nb doubles]
//   [U12^T double buffer (LU): 2 x chunk x ldk x nb complex -- the row panel in K-major form]
//   [W21 double buffer (Hermitian): 2 x chunk x ldk x nb -- the pre-scaled panel L21 D1]
//   [K copies: chunk x ldk x n (batched / host)][host staging: mask, loglik, info (host)]
struct WsLayout {
  size_t state_off, bm_off, am_off, d_off, ut_off, dh_off, k_off, mask_off, ll_off, info_off, total;
  int64_t ldk, strideK, strideM, strideU;
};

WsLayout layout(Kind kind, int64_t chunk, int64_t n, int nb, bool copies, bool host) {
  WsLayout L{};
  const size_t es = esize(kind);
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
  L.ut_off = off;  // W21 (Hermitian) or U12^T (LU): two group buffers of max(G, 2) panels each
  off = align_up(off + 2 * (size_t)std::max(group_size(), 2) * chunk * (size_t)L.strideU * es);
  L.dh_off = off;  // Hermitian: D of every pivot so far (chunk x n), the column-chunked schedule
  if (kind_herm(kind)) off = align_up(off + (size_t)chunk * (size_t)std::max<int64_t>(n, 1) * 8);
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
constexpr int MAX_CHUNKS = 64;
struct DeviceStreams {
  cudaStream_t s1 = nullptr, s2 = nullptr, s3 = nullptr;  // s3: host->device copies of the _host path
  cudaEvent_t ev_start, ev_panel, ev_rest, ev_done1, ev_done2, ev_delay, ev_copy_start;
  cudaEvent_t ev_chunk[MAX_CHUNKS];
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
    if (cudaStreamCreateWithPriority(&d.s3, cudaStreamNonBlocking, lo) != cudaSuccess) return DPP_ECUDA;
    for (cudaEvent_t* e : {&d.ev_start, &d.ev_panel, &d.ev_rest, &d.ev_done1, &d.ev_done2, &d.ev_delay, &d.ev_copy_start})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return DPP_ECUDA;
    for (cudaEvent_t& e : d.ev_chunk)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return DPP_ECUDA;
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
// persistently on the rest: minimise max(T1, T2) with T1 = diag latency + (tiles of the next
// block column's update + next panel) / R, T2 = tiles of (b) / (SMs - R), in units of one tile.
// g = G for the last step of a group: its trailing update has K = G nb (G times the tile time) and
// the chain beside it holds the next group's G diag tiles and G panels.
int reserve_sms(int64_t m2, int jn, int sms, int batch, int tile, bool herm, int g = 1) {
  // the diag tile in update-tile times (DPP_DIAG_TILES; 5 measured ~100 us vs ~20 us; after the
  // diag kernel went to 63 us, 2.5 .. 5 give the same C4 / UST rates within noise)
  static double diag_tiles = -1.0;
  if (diag_tiles < 0) {
    const char* e = getenv("DPP_DIAG_TILES");
    diag_tiles = e ? atof(e) : 5.0;
  }
  const double side = (double)((m2 + tile - 1) / tile), side_b = (double)((m2 - jn + tile - 1) / tile);
  const double ta = (herm ? 1.0 : 2.0) * side * batch;     // (a): next block column (LU: + row)
  const double tp = (herm ? 1.0 : 2.0) * side_b * batch;   // next panel GEMM(s)
  const double tb = (herm ? side_b * (side_b + 1) / 2 : side_b * side_b) * batch;  // (b) tiles
  int best = 8;
  double best_t = 1e300;
  for (int R = 4; R <= sms / 2; R += 2) {
    const double t1 = g * diag_tiles + (ta + g * tp) / R;
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
// Factors `batch` matrices A + s*strideA (in place), samples b0 + s.
// Column-chunked schedule (Hermitian kinds, lookahead on): the factorization proceeds over column
// chunks of cw columns; inside a chunk it is the right-looking loop below with its trailing
// updates restricted to the chunk's columns, and each new chunk first receives every earlier
// panel at once (one DMMA GEMM with K = c0, B scaled by the saved pivots) -- Prop. 5's exactness
// does not depend on the update order.  A chunk can start as soon as its columns are resident:
// the _host path copies chunk by chunk on a third stream and the chunk events gate the compute.
struct Chunking {
  int64_t cw = 0;               // 0: off
  const cudaEvent_t* ev = nullptr;  // per chunk: its columns are resident (nullable)
  // copy-gated mode (the _host path's default): the factorization is NOT restricted; the copy
  // arrives in chunks of copy_cw columns (events ev), each step's diag/panel/lookahead waits for
  // the chunk holding its next block column, and the trailing updates of the first split_steps
  // steps are launched per copy chunk, each waiting only for its own chunk
  int64_t copy_cw = 0;
  int split_steps = 0;
};

// DPP_CHUNK_COLS > 0 selects the column-chunked factorization (both paths; measured slower: 19.9
// vs 25.8 TF/s at n = 16384 with 2048-column chunks -- the restricted trailing updates leave the
// sequential chain exposed in every chunk).
int chunk_cols(bool host, int64_t n) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("DPP_CHUNK_COLS");
    v = e ? atoi(e) : 0;
  }
  (void)host;
  (void)n;
  return v;
}

// DPP_COPY_GATED=1: the _host path's copy-gated mode.  Off by default: measured slower (e2e 18.3
// vs 19.3 TF/s at n = 16384) -- the right-looking order needs every column before the first
// trailing update completes, and the work a left-looking order could do on the first columns is
// small, so little of the copy can hide behind compute.
// Grouped trailing updates (lookahead on): the trailing updates of G consecutive steps are applied
// by the group's last step as ONE DMMA pass with K = G nb (the G panels are adjacent columns of the
// factor; their operand copies -- W21 = L21 D1, or U12^T -- are stacked in one buffer), so the
// update kernel's per-tile epilogue and the C read/write are amortized over G times the work.
// G = 2 ("paired updates") by default; DPP_GROUP=g sets G, DPP_PAIR=0 turns grouping off.
int group_size() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPP_PAIR");
    const char* g = getenv("DPP_GROUP");
    v = (e && e[0] == '0') ? 1 : (g ? std::max(1, std::min(8, atoi(g))) : 2);
  }
  return v;
}

// rows below which the real Hermitian sampler switches to half-width blocks (DPP_TAIL_ROWS, 0 = off)
int64_t tail_rows() {
  static long long v = -1;
  if (v < 0) {
    const char* e = getenv("DPP_TAIL_ROWS");
    v = e ? atoll(e) : 0;
  }
  return (int64_t)v;
}

// trailing size below which updates are no longer paired (DPP_PAIR_MIN_ROWS; defaults: 6144 rows
// for 128-wide Hermitian blocks, where the 63..86-us diag tile makes the chain the bound near the end --
// measured C4 25.8 -> 26.1 TF/s -- 0 for 64-wide Hermitian blocks, whose chain is short (complex
// Hermitian n = 8192: 27.0 vs 26.6 TF/s with 6144), 8192 for LU)
int64_t pair_min_rows(int nb, bool herm, int batch) {
  static long long v = -2;
  if (v == -2) {
    const char* e = getenv("DPP_PAIR_MIN_ROWS");
    v = e ? atoll(e) : -1;
  }
  if (v >= 0) return (int64_t)v;
  if (batch >= 8) return 0;  // batched: the chain is shared by the batch, the updates dominate throughout
                             // (UST 40x40, 256 per launch: 2373 paired vs 2275 samples/s)
  if (!herm) return 8192;  // LU: two panel GEMMs and two lookahead updates per step (n = 8192: 27.6
                           // TF/s unpaired vs 26.1 paired; Aztec n = 25600: 33.3 paired vs 32.0)
  return nb >= 128 ? 6144 : 0;
}

bool head_block() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPP_HEAD_BLOCK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool copy_gated() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPP_COPY_GATED");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int run_blocked(Kind kind, const Opts& o, int64_t n, void* A, int64_t ld, int64_t strideA, int batch,
                uint64_t seed, uint64_t b0, uint8_t* mask, const uint8_t* forced, double* loglik,
                dpp_info_t* info, char* work, const WsLayout& L, cudaStream_t caller, bool map = false,
                Chunking ch = Chunking{}) {
  void* state = work + L.state_off;
  if (n == 0) { CK(launch_zero_state(state, loglik, info, batch, caller)); return DPP_OK; }
  DeviceStreams* ds = nullptr;
  int rc = get_streams(&ds, caller);
  if (rc) return rc;
  std::lock_guard<std::recursive_mutex> lk(ds->mu);
  const int nb = o.nb;
  const bool la = o.lookahead > 0;
  cudaStream_t s1 = la ? ds->s1 : caller, s2 = la ? ds->s2 : caller;
  if (la) {
    CK(cudaEventRecord(ds->ev_start, caller));
    CK(cudaStreamWaitEvent(s1, ds->ev_start, 0));
    CK(cudaStreamWaitEvent(s2, ds->ev_start, 0));
  }
  const size_t es = esize(kind);
  const bool herm = kind_herm(kind);
  char* Ab = reinterpret_cast<char*>(A);
  // 16-byte aligned columns: the TMA / cp.async 16-byte operand paths
  const bool vec = ((size_t)ld * es) % 16 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
                   ((size_t)strideA * es) % 16 == 0;
  void* Bm = work + L.bm_off;
  void* Am = work + L.am_off;
  int step = 0;
  bool have_rest = false;
  int gpos = -1;            // position of the previous step in its group (-1: none)
  bool prev_glast = false;  // the previous step was the last of a group
  const int sms = device_sms();
  if (!herm || !la || ch.cw < nb || ch.cw % nb) ch.cw = 0;
  if (ch.cw && (n + ch.cw - 1) / ch.cw > MAX_CHUNKS) ch.cw = (n + MAX_CHUNKS - 1) / MAX_CHUNKS / nb * nb + nb;
  double* dhist = herm ? reinterpret_cast<double*>(work + L.dh_off) : nullptr;
  // Tail blocks: once at most `thr` rows remain, the blocks are nb/2 wide -- the sequential chain
  // (diag tile, panel, lookahead column) is what bounds those steps, and a half-width diag tile
  // costs far less than half of a full one.  Pivot draws are by global index (R2): the blocking
  // does not change the sample.
  const int64_t thr = (nb == 128 && herm && la && !ch.cw && !ch.copy_cw) ? tail_rows() : 0;
  auto bs_of = [&](int64_t j) -> int { return (thr > 0 && n - j <= thr) ? nb / 2 : nb; };
  // Head block: when nb does not divide n, the FIRST block takes the remainder (n mod nb) so that
  // every trailing region is a whole number of 128-row tiles (a ragged last block would leave a
  // partly empty tile row and column in every trailing update).  Only when the remainder keeps every
  // block origin 16-byte aligned (the TMA operand copies): a multiple of 16 / element-size rows.
  // DPP_HEAD_BLOCK=0: ragged last block.
  const int64_t rem = n % nb;
  const int64_t head = (head_block() && !ch.cw && !ch.copy_cw && thr == 0 && n > nb && rem &&
                        rem % (int64_t)(16 / es) == 0) ? rem : 0;
  const int gbase = head ? 1 : 0;  // groups are aligned after the head block
  auto blk = [&](int64_t j) -> int64_t { return (head && j == 0) ? head : std::min<int64_t>(bs_of(j), n - j); };
  for (int64_t j0 = 0; j0 < n; j0 += blk(j0), ++step) {
    const int jb = (int)blk(j0);
    const int64_t j1 = j0 + jb, m2 = n - j1;
    const int64_t c0 = ch.cw ? (j0 / ch.cw) * ch.cw : 0;
    const int64_t ce = ch.cw ? std::min<int64_t>(n, c0 + ch.cw) : n;  // the chunk's columns: [c0, ce)
    if (ch.copy_cw && ch.ev) {
      // copy-gated: this step's tile, panel and lookahead column need the chunk of block column
      // j0 + 1 (and all before it -- the copies are issued in order on one stream)
      const int64_t need = std::min<int64_t>(n - 1, j1 + nb - 1);
      CK(cudaStreamWaitEvent(s1, ch.ev[need / ch.copy_cw], 0));
      // past the split steps the trailing updates are single launches: the whole copy must be in
      if (step == ch.split_steps) CK(cudaStreamWaitEvent(s2, ch.ev[(n - 1) / ch.copy_cw], 0));
    }
    if (ch.cw && j0 == c0) {
      if (ch.ev) {
        CK(cudaStreamWaitEvent(s1, ch.ev[j0 / ch.cw], 0));
        CK(cudaStreamWaitEvent(s2, ch.ev[j0 / ch.cw], 0));
      }
      if (c0 > 0) {
        // every earlier panel into the new chunk: A(c0:n, c0:ce) -= L(c0:n, 0:c0) D L(c0:ce, 0:c0)^H
        CK(cudaEventRecord(ds->ev_panel, s1));
        CK(cudaStreamWaitEvent(s2, ds->ev_panel, 0));
        UpdateArgs dl = base_update(kind, batch, vec);
        dl.Aop = Ab + (size_t)c0 * es; dl.lda = ld; dl.strideA = strideA;
        dl.Bop = Ab + (size_t)c0 * es; dl.ldb = ld; dl.strideB = strideA;
        dl.dscale = dhist; dl.dstride = n; dl.mask = 1; dl.conj = (kind == HERM_Z);
        dl.C = Ab + (size_t)(c0 + c0 * ld) * es; dl.ldc = ld; dl.strideC = strideA;
        dl.a_rows = (int)(n - c0); dl.b_rows = (int)(ce - c0); dl.K = (int)c0;
        dl.row0 = 0; dl.col0 = 0; dl.rows = (int)(n - c0); dl.cols = (int)(ce - c0); dl.tri = 0;
        {
          ProfScope ps(3, region_flops(kind, c0, c0, n - c0, ce - c0, (int)c0) * batch, s2);
          CK(launch_update(kind, dl, s2));
        }
        CK(cudaEventRecord(ds->ev_delay, s2));
        CK(cudaStreamWaitEvent(s1, ds->ev_delay, 0));
      }
    }
    double* dvec = herm ? reinterpret_cast<double*>(work + L.d_off) + (size_t)(step & 1) * batch * nb : nullptr;
    // LU: U12^T (m2 x jb, ld = ldk, K-major GEMM operand); Hermitian: W21 = L21 D1 (same shape);
    // double-buffered like D1
    const int64_t strideU = L.strideU;
    char* UT = work + L.ut_off + (size_t)(step & 1) * batch * strideU * es;
    // grouping: steps (G g .. G g + G-1) share the group buffer (g & 1) of G panels per sample
    const int G = group_size();
    const bool grouping = la && !ch.cw && !ch.copy_cw && G > 1 && nb == (int)std::min<int64_t>(nb, n);
    const int64_t strideW = (int64_t)std::max(G, 2) * strideU;
    const int gstep = step - gbase;  // (-1 for the head block: group buffer 1, unused by group 0)
    char* WP = work + L.ut_off + (size_t)((gstep < 0 ? 1 : gstep / G) & 1) * batch * strideW * es;
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
      } else if (gstep >= 0 && gstep % G == 0 && m2 - (int64_t)(G - 1) * nb > 0 &&
                 m2 > pair_min_rows(nb, herm, batch)) {
        bool full = true;
        for (int g = 0; g < G; ++g) full = full && bs_of(j0 + (int64_t)g * nb) == nb;
        if (full) gp = 0;
      }
    }
    const bool glast = gp == G - 1, gnonlast = gp >= 0 && !glast;
    char* const PH = WP + (size_t)(gp >= 0 ? gp * (strideU + nb) : (step % G) * strideU) * es;  // my slot
    char* const WG = WP + (size_t)(gp > 0 ? gp * nb : 0) * es;  // the stacked operand of panels 0..gp
    const int64_t jg0 = gp > 0 ? j0 - (int64_t)gp * nb : j0;  // the group's first column
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
    {
      const double fl = (herm ? 1.0 : 2.0) * jb * (double)jb * jb / 3.0 * cplx_mult(kind) * batch;
      ProfScope ps(0, fl, s1);
      CK(launch_diag(kind, bs_of(j0), d, s1));
    }
    if (m2 <= 0) break;
    if (ch.cw && herm)  // this block's pivots, for the later chunks' catch-up updates
      CK(cudaMemcpy2DAsync(dhist + j0, (size_t)n * 8, dvec, (size_t)nb * 8, (size_t)jb * 8, (size_t)batch,
                           cudaMemcpyDeviceToDevice, s1));
    // ---- stage 2: panel GEMMs with the tile operators (in place)
    {
      const double fl = (herm ? 1.0 : 2.0) * (double)m2 * jb * jb * cplx_mult(kind) * batch;  // TRSM count
      ProfScope ps(1, fl, s1);
      UpdateArgs p = base_update(kind, batch, vec);
      p.Aop = Ab + (size_t)(j1 + j0 * ld) * es; p.lda = ld; p.strideA = strideA;   // A21
      p.Bop = Bm; p.ldb = nb; p.strideB = L.strideM;
      p.C = Ab + (size_t)(j1 + j0 * ld) * es; p.ldc = ld; p.strideC = strideA;    // L21 in place
      p.a_rows = (int)m2; p.b_rows = jb; p.K = jb;
      p.row0 = 0; p.col0 = 0; p.rows = (int)m2; p.cols = jb;
      if (herm) {
        // and the pre-scaled copy W21 = L21 D1 (the trailing-update operand) into its panel slot
        // (written by the panel kernel's epilogue when it is the warp-specialized one)
        p.wout = grouping ? PH : UT; p.ldw = L.ldk; p.strideWo = grouping ? strideW : strideU;
        p.wscale = dvec; p.wsstride = nb;
      }
      CK(launch_update(kind, p, s1));
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
        q.a_rows = (int)m2; q.b_rows = jb; q.K = jb;
        q.row0 = 0; q.col0 = 0; q.rows = (int)m2; q.cols = jb;
        CK(launch_update(kind, q, s1));
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
    u.a_rows = (int)m2; u.b_rows = (int)m2; u.K = (gp > 0 ? gp * nb : 0) + jb;
    // width of the lookahead region: the next block -- or, at the last step of a group, the next
    // group's G blocks, so the next group's whole diag/panel chain runs under this group's update
    const int jn = (int)std::min<int64_t>(glast ? (int64_t)G * nb : bs_of(j1), m2);
    if (!la) {
      u.row0 = 0; u.col0 = 0; u.rows = (int)m2; u.cols = (int)m2; u.tri = herm;
      ProfScope ps(3, region_flops(kind, 0, 0, m2, m2, jb) * batch, s1);
      CK(launch_update(kind, u, s1));
      continue;
    }
    CK(cudaEventRecord(ds->ev_panel, s1));
    if (copyback) {
      CK(cudaStreamWaitEvent(s2, ds->ev_panel, 0));
      ProfScope pa(4, 0.0, s2);
      CK(launch_transpose(es, cb_src, L.ldk, cb_stride, cb_dst, ld, strideA, (int)m2, jb, batch, s2));  // U12 -> K
      copyback = false;
    }
    // (a) next block column [0, jn) x rows [0, m2)  (+ LU: next block row [0, jn) x cols [jn, m2));
    // chunked: only while the next block is in this chunk (else the catch-up update covers it)
    // (a non-last step of a group needs no wait: its lookahead block was covered by the previous
    // group's lookahead update and is not part of the previous trailing update)
    if (have_rest && !(gnonlast && (gp > 0 || prev_glast))) CK(cudaStreamWaitEvent(s1, ds->ev_rest, 0));
    prev_glast = glast;
    if (j1 < ce) {
      UpdateArgs ua = u;
      ua.row0 = 0; ua.col0 = 0; ua.rows = (int)m2; ua.cols = jn; ua.tri = 0;
      double fl = region_flops(kind, 0, 0, m2, jn, ua.K);
      if (!herm && m2 > jn) fl += region_flops(kind, 0, jn, jn, m2 - jn, jb);
      ProfScope ps(2, fl * batch, s1);
      CK(launch_update(kind, ua, s1));
      if (!herm && m2 > jn) {
        UpdateArgs ur = u;
        ur.row0 = 0; ur.col0 = jn; ur.rows = jn; ur.cols = (int)(m2 - jn); ur.tri = 0;
        CK(launch_update(kind, ur, s1));
      }
    }
    // (b) the rest [jn, m2)^2 on S2 (chunked: its columns restricted to the chunk)
    const int64_t colsb = std::min<int64_t>(m2, ce - j1) - jn;
    gpos = gp;  // a non-last position: the group's last step applies this step's trailing update
    if (m2 > jn && colsb > 0 && !gnonlast) {
      CK(cudaStreamWaitEvent(s2, ds->ev_panel, 0));
      UpdateArgs ub = u;
      ub.row0 = jn; ub.col0 = jn; ub.rows = (int)(m2 - jn); ub.cols = (int)colsb;
      ub.tri = herm && colsb == m2 - jn;
      if (vec)
        ub.grid_limit = sms - reserve_sms(m2, jn, sms, batch, kind_cplx(kind) ? 64 : 128, herm, glast ? G : 1);
      if (ch.copy_cw && ch.ev && step < ch.split_steps) {
        // one launch per copy chunk of the trailing columns, each gated by its own chunk
        for (int64_t g0 = j1 + jn; g0 < j1 + jn + colsb;) {
          const int64_t g1 = std::min<int64_t>(j1 + jn + colsb, (g0 / ch.copy_cw + 1) * ch.copy_cw);
          CK(cudaStreamWaitEvent(s2, ch.ev[(g1 - 1) / ch.copy_cw], 0));
          UpdateArgs up = ub;
          up.col0 = (int)(g0 - j1); up.cols = (int)(g1 - g0); up.tri = 0;
          ProfScope ps(3, region_flops(kind, jn, g0 - j1, m2 - jn, g1 - g0, jb) * batch, s2);
          CK(launch_update(kind, up, s2));
          g0 = g1;
        }
      } else {
        ProfScope ps(3, region_flops(kind, jn, jn, m2 - jn, colsb, ub.K) * batch, s2);
        CK(launch_update(kind, ub, s2));
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
  WsLayout L = layout(kind, 1, n, o.nb, false, false);
  if (!work || work_bytes < L.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  if (reinterpret_cast<uintptr_t>(K) % esize(kind)) return DPP_EINVAL;
  Chunking chk;
  chk.cw = kind_herm(kind) ? chunk_cols(false, n) : 0;
  return run_blocked(kind, o, n, K, ld, 0, 1, seed, 0, mask, o.forced, loglik, info, reinterpret_cast<char*>(work),
                     L, st, map, chk);
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
  WsLayout L = layout(kind, chunk, n, o.nb, true, host);
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
    const int64_t cw = (lower && cb == 1 && o.lookahead > 0) ? chunk_cols(host, n) : 0;
    const bool gated = host && lower && cb == 1 && o.lookahead > 0 && n >= 4096 && copy_gated();
    if (host && (cw > 0 || gated) && n > 0) {
      // pipelined: the copy of column chunk c (on s3) gates only chunk c of the factorization
      DeviceStreams* ds = nullptr;
      if ((rc = get_streams(&ds, st))) return rc;
      std::lock_guard<std::recursive_mutex> lk(ds->mu);
      CK(cudaEventRecord(ds->ev_copy_start, st));
      CK(cudaStreamWaitEvent(ds->s3, ds->ev_copy_start, 0));
      const char* src = reinterpret_cast<const char*>(K) + (size_t)(strideK * c0) * es;
      int64_t cwe = cw > 0 ? cw : 2048;
      if ((n + cwe - 1) / cwe > MAX_CHUNKS) cwe = (n + MAX_CHUNKS - 1) / MAX_CHUNKS / o.nb * o.nb + o.nb;
      for (int64_t q0 = 0, ci = 0; q0 < n; q0 += cwe, ++ci) {
        for (int64_t c = q0; c < std::min<int64_t>(n, q0 + cwe); c += 128) {
          const int64_t w_ = std::min<int64_t>({(int64_t)128, n - c, q0 + cwe - c});
          CK(cudaMemcpy2DAsync(Kc + (size_t)(c + c * L.ldk) * es, (size_t)L.ldk * es, src + (size_t)(c + c * ld) * es,
                               (size_t)ld * es, (size_t)(n - c) * es, (size_t)w_, ck, ds->s3));
        }
        CK(cudaEventRecord(ds->ev_chunk[ci], ds->s3));
      }
      uint8_t* mk = reinterpret_cast<uint8_t*>(w + L.mask_off);
      double* llk = reinterpret_cast<double*>(w + L.ll_off);
      dpp_info_t* ifo = info ? reinterpret_cast<dpp_info_t*>(w + L.info_off) : nullptr;
      const uint8_t* fz = o.forced ? o.forced + c0 * n : nullptr;
      Chunking chk;
      chk.ev = ds->ev_chunk;
      if (cw > 0) {
        chk.cw = cwe;
      } else {
        // copy-gated: split the trailing updates of the steps that can start before the copy is
        // over (estimate: copy at ~50 GB/s, trailing updates at ~25 TF/s)
        chk.copy_cw = cwe;
        double t_copy = 0.0;
        for (int64_t c = 0; c < n; c += 128) t_copy += (double)(n - c) * std::min<int64_t>(128, n - c) * es / 50e9;
        double t = 0.0;
        int k = 0;
        for (int64_t j = 0; j < n && t < t_copy; j += o.nb, ++k) {
          const double m = (double)(n - j - o.nb);
          t += m > 0 ? m * m * o.nb * cplx_mult(kind) / 25e12 : 0.0;
        }
        chk.split_steps = k + 1;
      }
      rc = run_blocked(kind, o, n, Kc, L.ldk, L.strideK, cb, seed, b0 + (uint64_t)c0, mk, fz, llk, ifo, w, L, st,
                       false, chk);
      if (rc) return rc;
      CK(cudaMemcpyAsync(mask + c0 * n, mk, (size_t)cb * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(loglik + c0, llk, 8 * (size_t)cb, cudaMemcpyDeviceToHost, st));
      if (info) CK(cudaMemcpyAsync(info + c0, ifo, sizeof(dpp_info_t) * (size_t)cb, cudaMemcpyDeviceToHost, st));
      continue;
    }
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
      } else {
        ProfScope pa(4, 0.0, st);
        CK(launch_copy_matrix(es, reinterpret_cast<const char*>(K) + (size_t)(strideK * c0) * es, ld,
                              strideK, Kc, L.ldk, L.strideK, (int)n, cb, lower, st));
      }
    }
    uint8_t* mk = host ? reinterpret_cast<uint8_t*>(w + L.mask_off) : mask + c0 * n;
    double* llk = host ? reinterpret_cast<double*>(w + L.ll_off) : loglik + c0;
    dpp_info_t* ifo = host ? (info ? reinterpret_cast<dpp_info_t*>(w + L.info_off) : nullptr) : (info ? info + c0 : nullptr);
    const uint8_t* fz = o.forced ? o.forced + c0 * n : nullptr;
    Chunking chk;
    chk.cw = cw;
    rc = run_blocked(kind, o, n, Kc, L.ldk, L.strideK, cb, seed, b0 + (uint64_t)c0, mk, fz, llk, ifo, w, L, st, false,
                     chk);
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
  return layout(kind, chunk, n, o.nb, batched, host).total;
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

int dpp_profile_begin_stages(unsigned stage_mask) {
  if (!(stage_mask & 0x1fu)) return DPP_EINVAL;
  g_prof.recs.clear();
  g_prof.used = 0;
  g_prof.mask = stage_mask & 0x1fu;
  g_prof.on = true;
  return DPP_OK;
}

int dpp_profile_begin(void) { return dpp_profile_begin_stages(0x1fu); }

int dpp_profile_end(dpp_profile_t* out) {
  g_prof.on = false;
  if (!out) return DPP_EINVAL;
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
    iv[r.stage].push_back({(double)t0, (double)t1});
  }
  for (int st = 0; st < 5; ++st) {  // length of the union of the stage's launch intervals
    std::sort(iv[st].begin(), iv[st].end());
    double lo = 0.0, hi = -1.0, u = 0.0;
    for (auto& p : iv[st]) {
      if (p.first > hi) { if (hi > lo) u += hi - lo; lo = p.first; hi = p.second; }
      else if (p.second > hi) hi = p.second;
    }
    if (hi > lo) u += hi - lo;
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
