// dist.cu -- 1D block-column-cyclic distributed sampler (mode 2).
//
// One sample of DPP(K) for a Hermitian K (real fp64 or complex128) too large (or too slow) for one
// GPU.  Rank r of P owns block columns c = r, r+P, ... (width nb: 128 real, 64 complex) of the
// lower triangle, stored contiguously.  Block step k of Listing 3/4:
//   owner(k) = k mod P:  stage 1 diag tile (decisions + D1 + tile operator), stage 2 panel GEMM
//                        (L21 = A21 L11^{-H} D1^{-1}, in place), pack [state | D1 | mask | L21];
//   all ranks:           broadcast the message from owner(k)   -- the one exchange per step;
//   receivers:           unpack state + decisions;
//   all ranks:           stage 3 on their local trailing block columns (C -= L21 D1 L21^H) with the
//                        DMMA update kernel in block-cyclic addressing mode.
// Because the decisions, pivots and the running log-likelihood ride in the message, every rank
// ends with the full mask and the same pivot-ordered loglik; no further collective is needed.
// The message carries only the live rows: L21 of step k is (n - j1) x jb at pitch
// round_up(n - j1, 16), so a receiver gets ~4 n^2 bytes (real) over the whole sample.
//
// Depth-1 lookahead (the distributed form of the paper's dependency scheduling):
// while every rank runs the trailing update of step k on the low-priority stream S2 (on all but a
// few SMs), the high-priority stream S1 of owner(k+1) first updates block column k+1 with step k's
// panel, then factors tile k+1 and its panel and packs message k+1, and every rank's S1 runs the
// broadcast of message k+1.  Messages are double-buffered: message k+1 is written only after the
// trailing update of step k-1 (the last reader of that buffer) has finished.  The broadcasts are
// issued in block order on S1 of every rank, so all ranks post the same sequence.
//
// Two transports drive the SAME per-step code (run_dist below):
//  * NCCL (dpp_comm_init): one process per GPU, ncclBroadcast(root = owner) on S1;
//  * in-process (dpp_comm_init_local): P virtual ranks on the calling thread's device, each with its
//    own streams, workspace and K_local; the broadcast is one device-to-device cudaMemcpyAsync per
//    receiver on the receiver's S1 after the owner's "packed" event, and an owner waits for every
//    receiver's copy before it reuses that message buffer.  The host issues each block step's
//    phases for all virtual ranks in order (pre-exchange, exchange, trailing update), so every
//    stream wait refers to work already enqueued: no kernel ever waits for another rank's kernel,
//    only stream-ordered events (PAPER.md:645-653's dependencies, on one GPU's streams).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace dpp;

namespace {

constexpr size_t ALIGN = 256;

#ifndef DPP_DIST_GROUP
#define DPP_DIST_GROUP 3           // default G of the grouped block steps
#endif
#ifndef DPP_DIST_GROUP_ROWS
#define DPP_DIST_GROUP_ROWS 6144    // real: groups while the group's last step keeps more trailing rows
#endif
#ifndef DPP_DIST_GROUP_ROWS_Z
#define DPP_DIST_GROUP_ROWS_Z 2048  // complex
#endif
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct RankStreams {
  cudaStream_t s1 = nullptr, s2 = nullptr;
  cudaEvent_t ev_start, ev_msg, ev_rest, ev_done1, ev_done2, ev_pack, ev_recv;
};

int make_rank_streams(RankStreams* rs) {
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return DPP_ECUDA;
  if (cudaStreamCreateWithPriority(&rs->s1, cudaStreamNonBlocking, hi) != cudaSuccess) return DPP_ECUDA;
  if (cudaStreamCreateWithPriority(&rs->s2, cudaStreamNonBlocking, lo) != cudaSuccess) return DPP_ECUDA;
  for (cudaEvent_t* ev : {&rs->ev_start, &rs->ev_msg, &rs->ev_rest, &rs->ev_done1, &rs->ev_done2, &rs->ev_pack,
                          &rs->ev_recv})
    if (cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) return DPP_ECUDA;
  return DPP_OK;
}

void destroy_rank_streams(RankStreams* rs) {
  if (rs->s1) cudaStreamDestroy(rs->s1);
  if (rs->s2) cudaStreamDestroy(rs->s2);
  for (cudaEvent_t ev : {rs->ev_start, rs->ev_msg, rs->ev_rest, rs->ev_done1, rs->ev_done2, rs->ev_pack, rs->ev_recv})
    if (ev) cudaEventDestroy(ev);
}

}  // namespace

struct dpp_comm_s {
  ncclComm_t nccl = nullptr;  // null: in-process virtual ranks
  int nranks = 1, rank = 0, device = 0, max_ctas = 8;
  bool local = false;
  std::vector<RankStreams> rs;  // one (NCCL) or nranks (local)
};

namespace {

// message = [SampleState 64 B][D1: nb doubles][mask: nb bytes -> 256-aligned][L21: m2 x jb at pitch
// round_up(m2, 16)]
struct MsgLayout {
  size_t d_off, mask_off, w_off, header_bytes;
};
MsgLayout msg_layout(int nb) {
  MsgLayout m;
  m.d_off = sizeof(SampleState);
  m.mask_off = m.d_off + 8 * (size_t)nb;
  m.w_off = align_up(m.mask_off + (size_t)nb);
  m.header_bytes = m.w_off;
  return m;
}
inline int64_t msg_pitch(int64_t m2) { return std::max<int64_t>(round_up(m2, 16), 16); }

// work = [state][panel operator Bm: nb x nb][D1: nb][message buffer 0][message buffer 1]
//        [W21 = L21 D1 of message 0][of message 1] (the pre-scaled A operand of the update)
struct DistWs {
  size_t state_off, bm_off, d_off, msg_off[2], w_off[2], gw_off[2], gl_off[2], total;
};
DistWs dist_ws(int64_t n, int nb, size_t es, int G) {
  DistWs w;
  const int64_t ldw = msg_pitch(n);  // the largest pitch (step 0 has m2 < n)
  MsgLayout m = msg_layout(nb);
  size_t off = 0;
  w.state_off = off; off = align_up(off + sizeof(SampleState));
  w.bm_off = off; off = align_up(off + (size_t)nb * nb * es);
  w.d_off = off; off = align_up(off + (size_t)nb * 8);
  for (int b = 0; b < 2; ++b) {
    w.msg_off[b] = off;
    off = align_up(off + m.header_bytes + (size_t)ldw * nb * es);
  }
  for (int b = 0; b < 2; ++b) {
    w.w_off[b] = off;
    off = align_up(off + (size_t)ldw * nb * es);
  }
  // grouped steps (see run_dist): the stacked operands of a group's K = G nb update, double-buffered
  // by group -- W = [W21_a | .. | W21_a+G-1] and (messages, P > 1) L = [L21_a | .. | L21_a+G-1]
  const int g = std::max(G, 1);
  for (int b = 0; b < 2; ++b) {
    w.gw_off[b] = off;
    off = align_up(off + (G > 1 ? (size_t)ldw * g * nb * es : 0));
  }
  for (int b = 0; b < 2; ++b) {
    w.gl_off[b] = off;
    off = align_up(off + (G > 1 ? (size_t)ldw * g * nb * es : 0));
  }
  w.total = off;
  return w;
}

// T11: the tile's first element; diagonal real parts at stride (ld + 1) elements of `dstride` doubles
__global__ void pack_header_kernel(const SampleState* st, const double* T11, int64_t dstep, int jb,
                                   const uint8_t* mask_j0, char* msg, MsgLayout m) {
  const int t = threadIdx.x;
  if (t == 0) *reinterpret_cast<SampleState*>(msg) = *st;
  for (int k = t; k < jb; k += blockDim.x) {
    reinterpret_cast<double*>(msg + m.d_off)[k] = T11[(int64_t)k * dstep];
    reinterpret_cast<uint8_t*>(msg + m.mask_off)[k] = mask_j0[k];
  }
}

__global__ void unpack_header_kernel(const char* msg, MsgLayout m, int jb, SampleState* st, uint8_t* mask_j0) {
  if (threadIdx.x == 0) *st = *reinterpret_cast<const SampleState*>(msg);
  for (int k = threadIdx.x; k < jb; k += blockDim.x) mask_j0[k] = reinterpret_cast<const uint8_t*>(msg + m.mask_off)[k];
}

__global__ void finalize_kernel(const SampleState* st, double* loglik, dpp_info_t* info) {
  if (threadIdx.x == 0) {
    *loglik = st->loglik;
    if (info) {
      info->n_kept = st->n_kept; info->n_ties = st->n_ties; info->first_tie = st->first_tie;
      info->n_out_of_range = st->n_out_of_range; info->min_abs_pivot = st->min_abs_pivot;
      info->max_abs_imag_pivot = st->max_abs_imag_pivot;
    }
  }
}

#define CK(x) do { if ((x) != cudaSuccess) return DPP_ECUDA; } while (0)
#define NK(x) do { if ((x) != ncclSuccess) return DPP_ENCCL; } while (0)

int dist_nb(Kind kind, const dpp_opts_t* opts) {
  const int def = kind == HERM_D ? 128 : 64;  // = the update kernel's tile width (bcc mode needs BN == nb)
  const int nb = (opts && opts->nb) ? opts->nb : def;
  return nb == def ? nb : -1;
}

// G: the trailing updates of G consecutive block steps applied as one K = G nb pass (dpp_opts_t.group:
// 0 = default 3, 1 = off, up to 4); -1 if out of range
int dist_group(const dpp_opts_t* opts) {
  const int g = (opts && opts->group) ? opts->group : DPP_DIST_GROUP;
  return (g >= 1 && g <= 4) ? g : -1;
}

int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// SMs to leave to S1 on owner(k+1) while the trailing update of step k runs persistently on the
// rest: minimise max(T1, T2), T1 = diag latency + (tiles of block column k+1 + of panel k+1) / R,
// T2 = this rank's share of the remaining lower-triangle tiles / (SMs - R), in tile times (the
// same model as the single-GPU driver, with the trailing tiles split over P ranks).
int reserve_sms(int64_t m2, int nb, int sms, int P) {
  const double diag_tiles = 5.0;
  const double side = (double)((m2 + nb - 1) / nb), side_b = (double)((m2 - nb + nb - 1) / nb);
  const double tb = side_b * (side_b + 1) / 2 / P;
  int best = 8;
  double best_t = 1e300;
  for (int R = 4; R <= sms / 2; R += 2) {
    const double t = std::max(diag_tiles + (side + side_b) / R, tb / (sms - R));
    if (t < best_t) { best_t = t; best = R; }
  }
  return best;
}

// One rank's view of a distributed call.
struct RankCtx {
  int r;
  char* K;           // K_local
  uint8_t* mask;     // n bytes (every rank ends with the full mask)
  double* loglik;
  dpp_info_t* info;
  char* w;           // workspace
  RankStreams* rs;
  cudaStream_t s1, s2;
  int64_t nloc;      // local blocks
};

int run_dist(Kind kind, dpp_comm_t comm, int64_t n, void* const* K_local, int64_t ld_local, uint64_t seed,
             uint8_t* const* mask, double* const* loglik, dpp_info_t* const* info, const dpp_opts_t* opts,
             void* const* work, size_t work_bytes, cudaStream_t st) {
  if (!comm || n < 0 || ld_local < std::max<int64_t>(n, 1)) return DPP_EINVAL;
  const int P = comm->nranks;
  const int nctx = comm->local ? P : 1;
  NvtxRange call_range("dpp dist %s n=%lld P=%d", kind == HERM_D ? "herm_d" : "herm_z", (long long)n, P);
  for (int i = 0; i < nctx; ++i)
    if (!loglik[i] || (n > 0 && (!mask[i] || !K_local[i]))) return DPP_EINVAL;
  const int nb = dist_nb(kind, opts);
  if (nb < 0) return DPP_EINVAL;
  const size_t es = kind == HERM_D ? 8 : 16;
  for (int i = 0; i < nctx; ++i)
    if (kind != HERM_D && reinterpret_cast<uintptr_t>(K_local[i]) % 16) return DPP_EINVAL;
  const double tie_tol = (opts && opts->tie_tol > 0) ? opts->tie_tol : 1e-9;
  const double range_tol = (opts && opts->range_tol > 0) ? opts->range_tol : 1e-8;
  const uint8_t* forced = opts ? opts->forced : nullptr;
  const bool la = !opts || opts->lookahead != 0;
  const int G = dist_group(opts);
  if (G < 0) return DPP_EINVAL;
  const DistWs W = dist_ws(n, nb, es, G);
  for (int i = 0; i < nctx; ++i)
    if (!work[i] || work_bytes < W.total || reinterpret_cast<uintptr_t>(work[i]) % ALIGN) return DPP_EWORKSPACE;
  if (n == 0) {
    for (int i = 0; i < nctx; ++i) CK(launch_zero_state(nullptr, loglik[i], info[i], 1, st));
    return DPP_OK;
  }
  const MsgLayout M = msg_layout(nb);
  const int64_t nblk = (n + nb - 1) / nb;
  const int sms = device_sms();
  std::vector<RankCtx> R(nctx);
  for (int i = 0; i < nctx; ++i) {
    RankCtx& c = R[i];
    c.r = comm->local ? i : comm->rank;
    c.K = reinterpret_cast<char*>(K_local[i]);
    c.mask = mask[i]; c.loglik = loglik[i]; c.info = info[i];
    c.w = reinterpret_cast<char*>(work[i]);
    c.rs = &comm->rs[i];
    c.s1 = la ? c.rs->s1 : st;
    c.s2 = la ? c.rs->s2 : st;
    c.nloc = (nblk - c.r + P - 1) / P;
    if (la) {
      CK(cudaEventRecord(c.rs->ev_start, st));
      CK(cudaStreamWaitEvent(c.s1, c.rs->ev_start, 0));
      CK(cudaStreamWaitEvent(c.s2, c.rs->ev_start, 0));
    }
  }
  const bool vec = kind != HERM_D || ((ld_local % 2 == 0) && [&] {
    for (int i = 0; i < nctx; ++i)
      if (reinterpret_cast<uintptr_t>(K_local[i]) % 16) return false;
    return true;
  }());
  // with one rank (NCCL transport) the panel is read straight from K_local: no message copy
  const bool self_only = P == 1;

  auto jb_of = [&](int64_t k) { return (int)std::min<int64_t>(nb, n - k * nb); };
  auto m2_of = [&](int64_t k) { return n - (k * nb + jb_of(k)); };
  auto msg_of = [&](const RankCtx& c, int64_t k) { return c.w + W.msg_off[k & 1]; };
  auto owner_ctx = [&](int64_t k) -> RankCtx* {
    const int o = (int)(k % P);
    for (auto& c : R)
      if (c.r == o) return &c;
    return nullptr;
  };
  // the L21 operand of step k on rank c: (pointer, leading dimension)
  auto l21_of = [&](const RankCtx& c, int64_t k) -> std::pair<const char*, int64_t> {
    if (self_only) return {c.K + (size_t)(k * nb + jb_of(k) + (k / P) * nb * ld_local) * es, ld_local};
    return {msg_of(c, k) + M.w_off, msg_pitch(m2_of(k))};
  };
  // Grouped steps (the distributed form of the single-GPU driver's grouped updates, G = 3 by
  // default): the trailing updates of steps a .. a+G-1 are deferred to the group's last step and
  // applied as ONE K = G nb pass over the stacked operands W = [W21_a | .. | W21_a+G-1],
  // L = [L21_a | .. | L21_a+G-1] (the slots of a group buffer, slot p shifted down by p nb rows so
  // that row r of the stacked operand is the same matrix row in every slot); step a+p's lookahead
  // update of block a+p+1 takes the panels a .. a+p (K = (p+1) nb), and the group's last step
  // updates the next group's G block columns, so the next group's steps run beside the group's
  // trailing update.  Groups form from the start while the group's last step keeps more than
  // group_rows trailing rows (near the end the chain bounds).
  // (dpp_opts_t: group = 1 turns groups off; group_min_rows > 0 sets the threshold, < 0 groups at
  // every size -- the tests' way to reach the grouped schedule at small n)
  const int64_t gmr = opts ? opts->group_min_rows : 0;
  const int64_t group_rows = std::max<int64_t>(
      (int64_t)G * nb, gmr < 0 ? 0 : gmr > 0 ? gmr : (kind == HERM_D ? DPP_DIST_GROUP_ROWS : DPP_DIST_GROUP_ROWS_Z));
  auto pos_of = [&](int64_t k) -> int {  // position of step k in its group, -1: ungrouped
    if (!la || G < 2) return -1;
    const int64_t a = k / G * G;
    if (a + G - 1 >= nblk || jb_of(a + G - 1) != nb || m2_of(a + G - 1) <= group_rows) return -1;
    return (int)(k - a);
  };
  const int64_t ldg = msg_pitch(n);
  auto gw_slot = [&](const RankCtx& c, int64_t k) {  // W21 of grouped step k in its group's W buffer
    const int64_t p = k % G;
    return c.w + W.gw_off[(k / G) & 1] + (size_t)(p * nb * ldg + p * nb) * es;
  };
  auto gl_slot = [&](const RankCtx& c, int64_t k) {  // L21 of grouped step k (messages only)
    const int64_t p = k % G;
    return c.w + W.gl_off[(k / G) & 1] + (size_t)(p * nb * ldg + p * nb) * es;
  };
  // owner(k): stage 1 + stage 2 of block k, packed into message k (stream s)
  auto factor_block = [&](RankCtx& c, int64_t k, cudaStream_t s) -> int {
    const int64_t j0 = k * nb;
    const int jb = jb_of(k);
    const int64_t j1 = j0 + jb, m2 = n - j1;
    const int64_t tcol = (k / P) * nb;  // storage column of block k on its owner
    char* msg = msg_of(c, k);
    SampleState* state = reinterpret_cast<SampleState*>(c.w + W.state_off);
    DiagArgs d{};
    d.A = c.K; d.ld = ld_local; d.strideA = 0; d.n = n; d.j0 = j0; d.tcol = tcol; d.jb = jb;
    d.seed = seed; d.b0 = 0; d.mask = c.mask; d.forced = forced; d.state = state; d.loglik = nullptr;
    d.info = nullptr; d.tie_tol = tie_tol; d.range_tol = range_tol; d.batch = 1;
    d.need_ops = m2 > 0; d.Bm = c.w + W.bm_off; d.dvec = reinterpret_cast<double*>(c.w + W.d_off); d.ldm = nb;
    d.strideM = 0;
    CK(launch_diag(kind, nb, d, s));
    if (m2 > 0) {
      // stage 2 in place: L21 = A21 L11^-H D1^-1, then into the message (live rows only)
      UpdateArgs p{};
      p.Aop = c.K + (size_t)(j1 + tcol * ld_local) * es; p.lda = ld_local;
      p.Bop = c.w + W.bm_off; p.ldb = nb;
      p.C = c.K + (size_t)(j1 + tcol * ld_local) * es; p.ldc = ld_local;
      p.a_rows = (int)m2; p.b_rows = jb; p.K = jb; p.rows = (int)m2; p.cols = jb; p.batch = 1; p.vec = vec ? 1 : 0;
      p.btri = 1;
      CK(launch_update(kind, p, s));
      if (!self_only)
        CK(cudaMemcpy2DAsync(msg + M.w_off, (size_t)msg_pitch(m2) * es, c.K + (size_t)(j1 + tcol * ld_local) * es,
                             (size_t)ld_local * es, (size_t)m2 * es, (size_t)jb, cudaMemcpyDeviceToDevice, s));
    }
    const double* T11 = reinterpret_cast<const double*>(c.K + (size_t)(j0 + tcol * ld_local) * es);
    pack_header_kernel<<<1, 128, 0, s>>>(state, T11, (ld_local + 1) * (int64_t)(es / 8), jb, c.mask + j0, msg, M);
    CK(cudaGetLastError());
    return DPP_OK;
  };
  auto msg_bytes = [&](int64_t k) {
    const int64_t m2 = m2_of(k);
    return M.header_bytes + (m2 > 0 && !self_only ? (size_t)msg_pitch(m2) * (size_t)jb_of(k) * es : 0);
  };
  // receivers of step k: unpack state + decisions; every rank: W21 = L21 D1 (the update's A
  // operand; the DMMA loop then needs no scaling)
  auto after_exchange = [&](RankCtx& c, int64_t k, cudaStream_t s) -> int {
    const int jb = jb_of(k);
    const int64_t m2 = m2_of(k);
    char* msg = msg_of(c, k);
    if (c.r != (int)(k % P)) {
      unpack_header_kernel<<<1, 128, 0, s>>>(msg, M, jb, reinterpret_cast<SampleState*>(c.w + W.state_off),
                                             c.mask + k * nb);
      CK(cudaGetLastError());
    }
    if (m2 > 0) {
      auto l = l21_of(c, k);
      const double* d1 = reinterpret_cast<const double*>(msg + M.d_off);
      if (pos_of(k) >= 0) {
        CK(launch_scale_cols(kind, l.first, l.second, 0, gw_slot(c, k), ldg, 0, d1, 0, (int)m2, jb, 1, s));
        if (!self_only)
          CK(cudaMemcpy2DAsync(gl_slot(c, k), (size_t)ldg * es, l.first, (size_t)l.second * es, (size_t)m2 * es,
                               (size_t)jb, cudaMemcpyDeviceToDevice, s));
      } else {
        CK(launch_scale_cols(kind, l.first, l.second, 0, c.w + W.w_off[k & 1], msg_pitch(m2), 0, d1, 0, (int)m2,
                             jb, 1, s));
      }
    }
    return DPP_OK;
  };
  // the broadcast of message k from owner(k), on every rank's S1 (phase run for all contexts)
  auto exchange = [&](int64_t k, bool lookahead_phase) -> int {
    const int owner = (int)(k % P);
    if (!comm->local) {
      RankCtx& c = R[0];
      cudaStream_t s = lookahead_phase ? c.s1 : st;
      char* msg = msg_of(c, k);
      if (P > 1) NK(ncclBroadcast(msg, msg, msg_bytes(k), ncclChar, owner, comm->nccl, s));
      return after_exchange(c, k, s);
    }
    RankCtx* oc = owner_ctx(k);
    CK(cudaEventRecord(oc->rs->ev_pack, oc->s1));
    for (auto& c : R) {
      if (c.r == owner) continue;
      CK(cudaStreamWaitEvent(c.s1, oc->rs->ev_pack, 0));
      CK(cudaMemcpyAsync(msg_of(c, k), msg_of(*oc, k), msg_bytes(k), cudaMemcpyDeviceToDevice, c.s1));
      CK(cudaEventRecord(c.rs->ev_recv, c.s1));
    }
    for (auto& c : R)
      if (int rc = after_exchange(c, k, c.s1)) return rc;
    return DPP_OK;
  };
  // in-process transport: before an owner rewrites a message buffer, every receiver's copy out of
  // it has completed (each rank's last ev_recv is at or after that copy)
  auto wait_receivers = [&](RankCtx& c) -> int {
    if (!comm->local) return DPP_OK;
    for (auto& o : R)
      if (o.r != c.r) CK(cudaStreamWaitEvent(c.s1, o.rs->ev_recv, 0));
    return DPP_OK;
  };
  // stage 3 of step k on local blocks q >= q_lo, up to `count` blocks (count < 0: all)
  auto update = [&](RankCtx& c, int64_t k, int64_t q_lo, int64_t count, int grid_limit, cudaStream_t s) -> int {
    const int jb = jb_of(k);
    const int64_t j1 = k * nb + jb, m2 = n - j1;
    const int64_t q_hi = count < 0 ? c.nloc : std::min<int64_t>(c.nloc, q_lo + count);
    if (m2 <= 0 || q_lo >= q_hi) return DPP_OK;
    auto l = l21_of(c, k);
    UpdateArgs u{};
    const int pk = pos_of(k);
    int K = jb;
    if (pk >= 1) {
      // the group's steps k-pk .. k: K = (pk+1) nb over the stacked operands from row j1 of step k
      // (the slots' common row: slot 0 shifted by pk nb rows)
      u.Aop = c.w + W.gw_off[(k / G) & 1] + (size_t)pk * nb * es; u.lda = ldg;
      if (self_only) {  // one rank: the group's blocks are adjacent local columns
        u.Bop = c.K + (size_t)(j1 + (k - pk) * nb * ld_local) * es; u.ldb = ld_local;
      } else {
        u.Bop = c.w + W.gl_off[(k / G) & 1] + (size_t)pk * nb * es; u.ldb = ldg;
      }
      K = (pk + 1) * nb;
    } else if (pk == 0) {
      u.Aop = gw_slot(c, k); u.lda = ldg;                  // W21 of step k alone
      u.Bop = l.first; u.ldb = l.second;
    } else {
      u.Aop = c.w + W.w_off[k & 1]; u.lda = msg_pitch(m2);  // W21 = L21 D1
      u.Bop = l.first; u.ldb = l.second;                    // L21 (conjugated on load for complex)
    }
    u.mask = 1;
    u.conj = kind == HERM_Z;
    u.C = c.K + (size_t)j1 * es;  // local column 0, A22 row 0
    u.ldc = ld_local;
    u.a_rows = (int)m2; u.b_rows = (int)m2; u.K = K; u.batch = 1; u.vec = vec ? 1 : 0;
    u.row0 = 0; u.rows = (int)m2; u.col0 = 0; u.cols = (int)m2; u.tri = 0;
    u.bcc_P = P; u.bcc_r = c.r; u.bcc_nb = nb; u.bcc_q0 = (int)q_lo; u.bcc_j1 = j1;
    u.tiles_n = (int)(q_hi - q_lo);
    u.grid_limit = grid_limit;
    CK(launch_update(kind, u, s));
    return DPP_OK;
  };
  int rc;
  // first local block strictly after block k on rank r
  auto first_after = [&](const RankCtx& c, int64_t k) { return (k + 1 - c.r + P - 1) / P; };

  if (!la) {
    for (int64_t k = 0; k < nblk; ++k) {
      NvtxRange step_range("dist step %lld", (long long)k);
      if (RankCtx* oc = owner_ctx(k)) {
        if ((rc = wait_receivers(*oc))) return rc;
        if ((rc = factor_block(*oc, k, st))) return rc;
      }
      if ((rc = exchange(k, false))) return rc;
      for (auto& c : R)
        if ((rc = update(c, k, first_after(c, k), -1, 0, st))) return rc;
    }
  } else {
    if (RankCtx* oc = owner_ctx(0))
      if ((rc = factor_block(*oc, 0, oc->s1))) return rc;
    if ((rc = exchange(0, true))) return rc;
    for (auto& c : R) CK(cudaEventRecord(c.rs->ev_msg, c.s1));
    for (int64_t k = 0; k < nblk; ++k) {
      const int64_t m2 = m2_of(k);
      if (m2 <= 0) break;
      NvtxRange step_range("dist step %lld", (long long)k);
      const int64_t kn = k + 1;  // the lookahead block
      const int pk = pos_of(k);
      // phase 1 (every rank's S1): message buffer kn&1 was last read by the trailing update of
      // step k-1; the owner of kn updates block column kn with step k's panel(s) and factors it.
      // A group's non-last steps need no wait: their lookahead blocks were covered by the previous
      // group's lookahead update and are not part of its trailing update (which reads group
      // buffers only); a group's last step also brings the next group's other blocks up to date.
      const bool glast = pk == G - 1;
      for (auto& c : R) {
        if (k > 0 && !(pk >= 0 && !glast && (pk > 0 || pos_of(k - 1) == G - 1)))
          CK(cudaStreamWaitEvent(c.s1, c.rs->ev_rest, 0));
        if (c.r == (int)(kn % P)) {
          if ((rc = update(c, k, kn / P, 1, 0, c.s1))) return rc;  // block column kn with step k's panel(s)
          if ((rc = wait_receivers(c))) return rc;
          if ((rc = factor_block(c, kn, c.s1))) return rc;
        }
        if (glast)
          for (int64_t b = kn + 1; b < kn + G && b < nblk; ++b)
            if (c.r == (int)(b % P))
              if ((rc = update(c, k, b / P, 1, 0, c.s1))) return rc;  // the next group's block columns
      }
      // phase 2: the exchange of message kn
      if ((rc = exchange(kn, true))) return rc;
      // phase 3 (S2): the rest of step k's trailing update (message k: ev_msg of the last step)
      for (auto& c : R) {
        if (pk >= 0 && !glast) {  // deferred to the group's last step
          CK(cudaEventRecord(c.rs->ev_msg, c.s1));  // message kn (exchange issued above)
          continue;
        }
        const bool own_next = c.r == (int)(kn % P);
        CK(cudaStreamWaitEvent(c.s2, c.rs->ev_msg, 0));
        const int64_t q_lo = glast ? first_after(c, k + G) : own_next ? kn / P + 1 : first_after(c, k);
        int reserve = 0;
        if (!comm->local) {
          if (own_next) {
            reserve = reserve_sms(m2, nb, sms, P);
            if (P > 1) reserve = std::min(sms / 2, reserve + comm->max_ctas);
          } else if (P > 1) {
            reserve = comm->max_ctas;  // the broadcast's CTAs
          }
        } else {
          // P virtual ranks share one GPU: each trailing update takes its share of the SMs
          reserve = sms - std::max(8, (sms - reserve_sms(m2, nb, sms, P)) / P);
        }
        if ((rc = update(c, k, q_lo, -1, vec ? sms - reserve : 0, c.s2))) return rc;
        CK(cudaEventRecord(c.rs->ev_rest, c.s2));
        CK(cudaEventRecord(c.rs->ev_msg, c.s1));  // message kn (exchange issued above)
      }
    }
  }
  // the final state: written by the diag kernel on the last block's owner, unpacked elsewhere
  for (auto& c : R) {
    cudaStream_t s = la ? c.s1 : st;
    finalize_kernel<<<1, 32, 0, s>>>(reinterpret_cast<SampleState*>(c.w + W.state_off), c.loglik, c.info);
    CK(cudaGetLastError());
    if (la) {
      CK(cudaEventRecord(c.rs->ev_done1, c.s1));
      CK(cudaEventRecord(c.rs->ev_done2, c.s2));
      CK(cudaStreamWaitEvent(st, c.rs->ev_done1, 0));
      CK(cudaStreamWaitEvent(st, c.rs->ev_done2, 0));
    }
  }
  return DPP_OK;
}

int run_dist_one(Kind kind, dpp_comm_t comm, int64_t n, void* K_local, int64_t ld_local, uint64_t seed,
                 uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                 size_t work_bytes, cudaStream_t st) {
  if (!comm || comm->local) return DPP_EINVAL;
  void* K[1] = {K_local};
  uint8_t* m[1] = {mask};
  double* l[1] = {loglik};
  dpp_info_t* i[1] = {info};
  void* w[1] = {work};
  return run_dist(kind, comm, n, K, ld_local, seed, m, l, i, opts, w, work_bytes, st);
}

int run_dist_local(Kind kind, dpp_comm_t comm, int64_t n, void* const* K_local, int64_t ld_local, uint64_t seed,
                   uint8_t* const* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts,
                   void* const* work, size_t work_bytes, cudaStream_t st) {
  if (!comm || !comm->local || !K_local || !mask || !loglik || !work) return DPP_EINVAL;
  const int P = comm->nranks;
  std::vector<double*> l(P);
  std::vector<dpp_info_t*> in(P);
  for (int r = 0; r < P; ++r) {
    l[r] = loglik + r;
    in[r] = info ? info + r : nullptr;
  }
  return run_dist(kind, comm, n, K_local, ld_local, seed, mask, l.data(), in.data(), opts, work, work_bytes, st);
}

}  // namespace

extern "C" {

int dpp_comm_init(const void* id, int nranks, int rank, dpp_comm_t* comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return DPP_EINVAL;
  ncclUniqueId uid;
  static_assert(sizeof(ncclUniqueId) == 128, "unique id size");
  std::memcpy(&uid, id, sizeof(uid));
  dpp_comm_s* c = new dpp_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  // cap the broadcast's CTAs so it fits in the SMs the trailing update leaves free
  c->max_ctas = 8;
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.maxCTAs = c->max_ctas;
  if (ncclCommInitRankConfig(&c->nccl, nranks, uid, rank, &cfg) != ncclSuccess) { delete c; return DPP_ENCCL; }
  c->rs.resize(1);
  if (make_rank_streams(&c->rs[0]) != DPP_OK) {
    destroy_rank_streams(&c->rs[0]);
    ncclCommDestroy(c->nccl);
    delete c;
    return DPP_ECUDA;
  }
  *comm = c;
  return DPP_OK;
}

int dpp_comm_init_local(int nranks, dpp_comm_t* comm) {
  if (!comm || nranks < 1 || nranks > 64) return DPP_EINVAL;
  dpp_comm_s* c = new dpp_comm_s();
  c->nranks = nranks;
  c->rank = -1;
  c->local = true;
  cudaGetDevice(&c->device);
  c->rs.resize(nranks);
  for (auto& rs : c->rs)
    if (make_rank_streams(&rs) != DPP_OK) {
      for (auto& x : c->rs) destroy_rank_streams(&x);
      delete c;
      return DPP_ECUDA;
    }
  *comm = c;
  return DPP_OK;
}

int dpp_comm_destroy(dpp_comm_t comm) {
  if (!comm) return DPP_EINVAL;
  ncclResult_t r = comm->nccl ? ncclCommDestroy(comm->nccl) : ncclSuccess;
  for (auto& rs : comm->rs) destroy_rank_streams(&rs);
  delete comm;
  return r == ncclSuccess ? DPP_OK : DPP_ENCCL;
}

int64_t dpp_bcc_local_cols(int64_t n, int32_t nb, int nranks, int rank) {
  if (n < 0 || nb <= 0 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
  const int64_t nblk = (n + nb - 1) / nb;
  int64_t cols = 0;
  for (int64_t c = rank; c < nblk; c += nranks) cols += std::min<int64_t>(nb, n - c * nb);
  return cols;
}

size_t dpp_dist_workspace_bytes(int op, int64_t n, int nranks, const dpp_opts_t* opts) {
  const int k = op & 0x7;
  if ((k != DPP_OP_HERM_D && k != DPP_OP_HERM_Z) || n < 0 || nranks < 1) return 0;
  const Kind kind = k == DPP_OP_HERM_D ? HERM_D : HERM_Z;
  const int nb = dist_nb(kind, opts);
  if (nb < 0) return 0;
  const int G = dist_group(opts);
  if (G < 0) return 0;
  return dist_ws(n, nb, kind == HERM_D ? 8 : 16, G).total;
}

int64_t dpp_dist_message_bytes(int op, int64_t n, int nranks, int64_t k) {
  const int kk = op & 0x7;
  if ((kk != DPP_OP_HERM_D && kk != DPP_OP_HERM_Z) || n < 0 || nranks < 1 || k < 0) return -1;
  const int nb = kk == DPP_OP_HERM_D ? 128 : 64;
  const size_t es = kk == DPP_OP_HERM_D ? 8 : 16;
  if (k * nb >= n) return -1;
  const int64_t jb = std::min<int64_t>(nb, n - k * nb), m2 = n - (k * nb + jb);
  if (nranks == 1) return (int64_t)msg_layout(nb).header_bytes;
  return (int64_t)(msg_layout(nb).header_bytes + (m2 > 0 ? (size_t)msg_pitch(m2) * (size_t)jb * es : 0));
}

int dpp_sample_herm_d_dist(dpp_comm_t comm, int64_t n, double* K_local, int64_t ld_local, uint64_t seed,
                           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream) {
  return run_dist_one(HERM_D, comm, n, K_local, ld_local, seed, mask, loglik, info, opts, work, work_bytes,
                      (cudaStream_t)stream);
}

int dpp_sample_herm_z_dist(dpp_comm_t comm, int64_t n, dpp_complex_t* K_local, int64_t ld_local, uint64_t seed,
                           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream) {
  return run_dist_one(HERM_Z, comm, n, K_local, ld_local, seed, mask, loglik, info, opts, work, work_bytes,
                      (cudaStream_t)stream);
}

int dpp_sample_herm_d_dist_local(dpp_comm_t comm, int64_t n, double* const* K_local, int64_t ld_local,
                                 uint64_t seed, uint8_t* const* mask, double* loglik, dpp_info_t* info,
                                 const dpp_opts_t* opts, void* const* work, size_t work_bytes, dpp_stream_t stream) {
  return run_dist_local(HERM_D, comm, n, reinterpret_cast<void* const*>(K_local), ld_local, seed, mask, loglik, info,
                        opts, work, work_bytes, (cudaStream_t)stream);
}

int dpp_sample_herm_z_dist_local(dpp_comm_t comm, int64_t n, dpp_complex_t* const* K_local, int64_t ld_local,
                                 uint64_t seed, uint8_t* const* mask, double* loglik, dpp_info_t* info,
                                 const dpp_opts_t* opts, void* const* work, size_t work_bytes, dpp_stream_t stream) {
  return run_dist_local(HERM_Z, comm, n, reinterpret_cast<void* const*>(K_local), ld_local, seed, mask, loglik, info,
                        opts, work, work_bytes, (cudaStream_t)stream);
}

}  // extern "C"
