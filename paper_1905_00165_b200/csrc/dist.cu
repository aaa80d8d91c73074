// dist.cu -- 1D block-column-cyclic distributed sampler over NCCL (mode 2).
//
// One sample of DPP(K) for a Hermitian K (real fp64 or complex128) too large (or too slow) for one
// GPU.  Rank r of P owns block columns c = r, r+P, ... (width nb: 128 real, 64 complex) of the
// lower triangle, stored contiguously.  Block step k of Listing 3/4:
//   owner(k) = k mod P:  stage 1 diag tile (decisions + D1 + tile operator), stage 2 panel GEMM
//                        (L21 = A21 L11^{-H} D1^{-1}, in place), pack [state | D1 | mask | L21];
//   all ranks:           ncclBroadcast(message, root = owner(k))   -- the one exchange per step;
//   receivers:           unpack state + decisions;
//   all ranks:           stage 3 on their local trailing block columns (C -= L21 D1 L21^H) with the
//                        DMMA update kernel in block-cyclic addressing mode.
// Because the decisions, pivots and the running log-likelihood ride in the message, every rank
// ends with the full mask and the same pivot-ordered loglik; no further collective is needed.
//
// Depth-1 lookahead (the distributed form of the paper's dependency scheduling):
// while every rank runs the trailing update of step k on the low-priority stream S2 (on all but a
// few SMs), the high-priority stream S1 of owner(k+1) first updates block column k+1 with step k's
// panel, then factors tile k+1 and its panel and packs message k+1, and every rank's S1 runs the
// broadcast of message k+1.  Messages are double-buffered: message k+1 is written only after the
// trailing update of step k-1 (the last reader of that buffer) has finished.  The broadcasts are
// issued in block order on S1 of every rank, so all ranks post the same NCCL sequence.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

using namespace dpp;

struct dpp_comm_s {
  ncclComm_t nccl;
  int nranks, rank, device, max_ctas;
  cudaStream_t s1, s2;
  cudaEvent_t ev_start, ev_msg, ev_rest, ev_done1, ev_done2;
};

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// message = [SampleState 64 B][D1: nb doubles][mask: nb bytes -> 256-aligned][L21: ldw x nb elems]
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

// work = [state][panel operator Bm: nb x nb][D1: nb][message buffer 0][message buffer 1]
//        [W21 = L21 D1 of message 0][of message 1] (the pre-scaled A operand of the update)
struct DistWs {
  size_t state_off, bm_off, d_off, msg_off[2], w_off[2], total;
  int64_t ldw;
};
DistWs dist_ws(int64_t n, int nb, size_t es) {
  DistWs w;
  w.ldw = std::max<int64_t>(round_up(n, 16), 16);
  MsgLayout m = msg_layout(nb);
  size_t off = 0;
  w.state_off = off; off = align_up(off + sizeof(SampleState));
  w.bm_off = off; off = align_up(off + (size_t)nb * nb * es);
  w.d_off = off; off = align_up(off + (size_t)nb * 8);
  for (int b = 0; b < 2; ++b) {
    w.msg_off[b] = off;
    off = align_up(off + m.header_bytes + (size_t)w.ldw * nb * es);
  }
  for (int b = 0; b < 2; ++b) {
    w.w_off[b] = off;
    off = align_up(off + (size_t)w.ldw * nb * es);
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

int run_dist(Kind kind, dpp_comm_t comm, int64_t n, void* K_local, int64_t ld_local, uint64_t seed, uint8_t* mask,
             double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work, size_t work_bytes,
             cudaStream_t st) {
  if (!comm || n < 0 || !loglik || (n > 0 && (!mask || !K_local)) || ld_local < std::max<int64_t>(n, 1))
    return DPP_EINVAL;
  const int nb = dist_nb(kind, opts);
  if (nb < 0) return DPP_EINVAL;
  const size_t es = kind == HERM_D ? 8 : 16;
  if (kind != HERM_D && reinterpret_cast<uintptr_t>(K_local) % 16) return DPP_EINVAL;
  const double tie_tol = (opts && opts->tie_tol > 0) ? opts->tie_tol : 1e-9;
  const double range_tol = (opts && opts->range_tol > 0) ? opts->range_tol : 1e-8;
  const uint8_t* forced = opts ? opts->forced : nullptr;
  const bool la = !opts || opts->lookahead != 0;
  const DistWs W = dist_ws(n, nb, es);
  if (!work || work_bytes < W.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  if (n == 0) { CK(launch_zero_state(nullptr, loglik, info, 1, st)); return DPP_OK; }
  const int P = comm->nranks, r = comm->rank;
  char* w = reinterpret_cast<char*>(work);
  SampleState* state = reinterpret_cast<SampleState*>(w + W.state_off);
  void* Bm = w + W.bm_off;
  double* dvec = reinterpret_cast<double*>(w + W.d_off);
  const MsgLayout M = msg_layout(nb);
  const int64_t nblk = (n + nb - 1) / nb;
  const int64_t nloc = (nblk - r + P - 1) / P;  // local blocks on r
  char* Kb = reinterpret_cast<char*>(K_local);
  const bool vec = kind != HERM_D || ((ld_local % 2 == 0) && (reinterpret_cast<uintptr_t>(K_local) % 16 == 0));
  const int sms = device_sms();
  cudaStream_t s1 = la ? comm->s1 : st, s2 = la ? comm->s2 : st;
  if (la) {
    CK(cudaEventRecord(comm->ev_start, st));
    CK(cudaStreamWaitEvent(s1, comm->ev_start, 0));
    CK(cudaStreamWaitEvent(s2, comm->ev_start, 0));
  }

  auto jb_of = [&](int64_t k) { return (int)std::min<int64_t>(nb, n - k * nb); };
  auto msg_of = [&](int64_t k) { return w + W.msg_off[k & 1]; };
  // owner(k): stage 1 + stage 2 of block k, packed into message k (stream s)
  auto factor_block = [&](int64_t k, cudaStream_t s) -> int {
    const int64_t j0 = k * nb;
    const int jb = jb_of(k);
    const int64_t j1 = j0 + jb, m2 = n - j1;
    const int64_t tcol = (k / P) * nb;  // storage column of block k on its owner
    char* msg = msg_of(k);
    DiagArgs d{};
    d.A = K_local; d.ld = ld_local; d.strideA = 0; d.n = n; d.j0 = j0; d.tcol = tcol; d.jb = jb;
    d.seed = seed; d.b0 = 0; d.mask = mask; d.forced = forced; d.state = state; d.loglik = nullptr;
    d.info = nullptr; d.tie_tol = tie_tol; d.range_tol = range_tol; d.batch = 1;
    d.need_ops = m2 > 0; d.Bm = Bm; d.dvec = dvec; d.ldm = nb; d.strideM = 0;
    CK(launch_diag(kind, nb, d, s));
    if (m2 > 0) {
      // stage 2 in place: L21 = A21 L11^-H D1^-1, then into the message
      UpdateArgs p{};
      p.Aop = Kb + (size_t)(j1 + tcol * ld_local) * es; p.lda = ld_local;
      p.Bop = Bm; p.ldb = nb;
      p.C = Kb + (size_t)(j1 + tcol * ld_local) * es; p.ldc = ld_local;
      p.a_rows = (int)m2; p.b_rows = jb; p.K = jb; p.rows = (int)m2; p.cols = jb; p.batch = 1; p.vec = vec ? 1 : 0;
      CK(launch_update(kind, p, s));
      CK(cudaMemcpy2DAsync(msg + M.w_off, (size_t)W.ldw * es, Kb + (size_t)(j1 + tcol * ld_local) * es,
                           (size_t)ld_local * es, (size_t)m2 * es, (size_t)jb, cudaMemcpyDeviceToDevice, s));
    }
    const double* T11 = reinterpret_cast<const double*>(Kb + (size_t)(j0 + tcol * ld_local) * es);
    pack_header_kernel<<<1, 128, 0, s>>>(state, T11, (ld_local + 1) * (int64_t)(es / 8), jb, mask + j0, msg, M);
    CK(cudaGetLastError());
    return DPP_OK;
  };
  // every rank: broadcast message k from its owner; receivers take the state and decisions
  auto exchange = [&](int64_t k, cudaStream_t s) -> int {
    const int owner = (int)(k % P);
    const int jb = jb_of(k);
    const int64_t m2 = n - (k * nb + jb);
    char* msg = msg_of(k);
    const size_t bytes = M.header_bytes + (m2 > 0 ? (size_t)W.ldw * (size_t)jb * es : 0);
    if (P > 1) NK(ncclBroadcast(msg, msg, bytes, ncclChar, owner, comm->nccl, s));
    if (r != owner) {
      unpack_header_kernel<<<1, 128, 0, s>>>(msg, M, jb, state, mask + k * nb);
      CK(cudaGetLastError());
    }
    // every rank: W21 = L21 D1 (the update's A operand; the DMMA loop then needs no scaling)
    if (m2 > 0)
      CK(launch_scale_cols(kind, msg + M.w_off, W.ldw, 0, w + W.w_off[k & 1], W.ldw, 0,
                           reinterpret_cast<const double*>(msg + M.d_off), 0, (int)m2, jb, 1, s));
    return DPP_OK;
  };
  // stage 3 of step k on local blocks q >= q_lo, up to `count` blocks (count < 0: all)
  auto update = [&](int64_t k, int64_t q_lo, int64_t count, int grid_limit, cudaStream_t s) -> int {
    const int jb = jb_of(k);
    const int64_t j1 = k * nb + jb, m2 = n - j1;
    const int64_t q_hi = count < 0 ? nloc : std::min<int64_t>(nloc, q_lo + count);
    if (m2 <= 0 || q_lo >= q_hi) return DPP_OK;
    char* msg = msg_of(k);
    UpdateArgs u{};
    u.Aop = w + W.w_off[k & 1]; u.lda = W.ldw;   // W21 = L21 D1
    u.Bop = msg + M.w_off; u.ldb = W.ldw; u.mask = 1;  // L21 (conjugated on load for complex)
    u.conj = kind == HERM_Z;
    u.C = Kb + (size_t)j1 * es;  // local column 0, A22 row 0
    u.ldc = ld_local;
    u.a_rows = (int)m2; u.b_rows = (int)m2; u.K = jb; u.batch = 1; u.vec = vec ? 1 : 0;
    u.row0 = 0; u.rows = (int)m2; u.col0 = 0; u.cols = (int)m2; u.tri = 0;
    u.bcc_P = P; u.bcc_r = r; u.bcc_nb = nb; u.bcc_q0 = (int)q_lo; u.bcc_j1 = j1;
    u.tiles_n = (int)(q_hi - q_lo);
    u.grid_limit = grid_limit;
    CK(launch_update(kind, u, s));
    return DPP_OK;
  };
  int rc;
  // first local block strictly after block k on this rank
  auto first_after = [&](int64_t k) { return (k + 1 - r + P - 1) / P; };

  if (!la) {
    for (int64_t k = 0; k < nblk; ++k) {
      if (r == (int)(k % P) && (rc = factor_block(k, st))) return rc;
      if ((rc = exchange(k, st))) return rc;
      if ((rc = update(k, first_after(k), -1, 0, st))) return rc;
    }
  } else {
    if (r == 0 && (rc = factor_block(0, s1))) return rc;
    if ((rc = exchange(0, s1))) return rc;
    CK(cudaEventRecord(comm->ev_msg, s1));
    for (int64_t k = 0; k < nblk; ++k) {
      const int64_t m2 = n - (k * nb + jb_of(k));
      if (m2 <= 0) break;
      const int64_t kn = k + 1;                 // the lookahead block
      const bool own_next = r == (int)(kn % P);
      // S1: message buffer kn&1 was last read by the trailing update of step k-1
      if (k > 0) CK(cudaStreamWaitEvent(s1, comm->ev_rest, 0));
      if (own_next) {
        if ((rc = update(k, kn / P, 1, 0, s1))) return rc;  // block column kn with step k's panel
        if ((rc = factor_block(kn, s1))) return rc;
      }
      if ((rc = exchange(kn, s1))) return rc;
      // S2: the rest of step k's trailing update (message k is ready: ev_msg recorded last step)
      CK(cudaStreamWaitEvent(s2, comm->ev_msg, 0));
      {
        const int64_t q_lo = own_next ? kn / P + 1 : first_after(k);
        int reserve = 0;
        if (own_next) {
          reserve = reserve_sms(m2, nb, sms, P);
          if (P > 1) reserve = std::min(sms / 2, reserve + comm->max_ctas);
        } else if (P > 1) {
          reserve = comm->max_ctas;  // the broadcast's CTAs
        }
        if ((rc = update(k, q_lo, -1, vec ? sms - reserve : 0, s2))) return rc;
      }
      CK(cudaEventRecord(comm->ev_rest, s2));
      CK(cudaEventRecord(comm->ev_msg, s1));  // message kn (exchange issued above)
    }
  }
  // the final state: written by the diag kernel on the last block's owner, unpacked elsewhere
  finalize_kernel<<<1, 32, 0, s1>>>(state, loglik, info);
  CK(cudaGetLastError());
  if (la) {
    CK(cudaEventRecord(comm->ev_done1, s1));
    CK(cudaEventRecord(comm->ev_done2, s2));
    CK(cudaStreamWaitEvent(st, comm->ev_done1, 0));
    CK(cudaStreamWaitEvent(st, comm->ev_done2, 0));
  }
  return DPP_OK;
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
  const char* e = getenv("DPP_NCCL_MAX_CTAS");
  c->max_ctas = (e && atoi(e) > 0) ? atoi(e) : 8;
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.maxCTAs = c->max_ctas;
  if (ncclCommInitRankConfig(&c->nccl, nranks, uid, rank, &cfg) != ncclSuccess) { delete c; return DPP_ENCCL; }
  int lo = 0, hi = 0;
  bool ok = cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess &&
            cudaStreamCreateWithPriority(&c->s1, cudaStreamNonBlocking, hi) == cudaSuccess &&
            cudaStreamCreateWithPriority(&c->s2, cudaStreamNonBlocking, lo) == cudaSuccess;
  for (cudaEvent_t* ev : {&c->ev_start, &c->ev_msg, &c->ev_rest, &c->ev_done1, &c->ev_done2})
    ok = ok && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) { ncclCommDestroy(c->nccl); delete c; return DPP_ECUDA; }
  *comm = c;
  return DPP_OK;
}

int dpp_comm_destroy(dpp_comm_t comm) {
  if (!comm) return DPP_EINVAL;
  ncclResult_t r = ncclCommDestroy(comm->nccl);
  cudaStreamDestroy(comm->s1);
  cudaStreamDestroy(comm->s2);
  for (cudaEvent_t ev : {comm->ev_start, comm->ev_msg, comm->ev_rest, comm->ev_done1, comm->ev_done2})
    cudaEventDestroy(ev);
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
  const int k = op & 3;
  if ((k != DPP_OP_HERM_D && k != DPP_OP_HERM_Z) || n < 0 || nranks < 1) return 0;
  const Kind kind = k == DPP_OP_HERM_D ? HERM_D : HERM_Z;
  const int nb = dist_nb(kind, opts);
  if (nb < 0) return 0;
  return dist_ws(n, nb, kind == HERM_D ? 8 : 16).total;
}

int dpp_sample_herm_d_dist(dpp_comm_t comm, int64_t n, double* K_local, int64_t ld_local, uint64_t seed,
                           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream) {
  return run_dist(HERM_D, comm, n, K_local, ld_local, seed, mask, loglik, info, opts, work, work_bytes,
                  (cudaStream_t)stream);
}

int dpp_sample_herm_z_dist(dpp_comm_t comm, int64_t n, dpp_complex_t* K_local, int64_t ld_local, uint64_t seed,
                           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream) {
  return run_dist(HERM_Z, comm, n, K_local, ld_local, seed, mask, loglik, info, opts, work, work_bytes,
                  (cudaStream_t)stream);
}

}  // extern "C"
