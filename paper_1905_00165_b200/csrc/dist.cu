// dist.cu -- 1D block-column-cyclic distributed sampler over NCCL (mode 2).
//
// One sample of DPP(K) for a Hermitian real K too large (or too slow) for one GPU.  Rank r of P
// owns block columns c = r, r+P, ... (width nb) of the lower triangle, stored contiguously.  Block
// step k of Listing 3/4:
//   owner(k) = k mod P:  stage 1 diag tile (decisions + D1 + tile operator), stage 2 panel GEMM
//                        (L21 = A21 L11^{-T} D1^{-1}, in place), pack [state | D1 | mask | L21];
//   all ranks:           ncclBroadcast(message, root = owner(k))   -- the one exchange per step;
//   receivers:           unpack state + decisions;
//   all ranks:           stage 3 on their local trailing block columns (C -= L21 D1 L21^T) with the
//                        DMMA update kernel in block-cyclic addressing mode.
// Because the decisions, pivots and the running log-likelihood ride in the message, every rank
// ends with the full mask and the same pivot-ordered loglik; no further collective is needed.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

using namespace dpp;

struct dpp_comm_s {
  ncclComm_t nccl;
  int nranks, rank;
};

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// message = [SampleState 64 B][D1: nb doubles][mask: nb bytes -> 256-aligned][L21: ldw x nb]
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

// work = [state][panel operator Bm: nb x nb][D1: nb][message buffer]
struct DistWs {
  size_t state_off, bm_off, d_off, msg_off, total;
  int64_t ldw;
};
DistWs dist_ws(int64_t n, int nb) {
  DistWs w;
  w.ldw = std::max<int64_t>(round_up(n, 16), 16);
  MsgLayout m = msg_layout(nb);
  size_t off = 0;
  w.state_off = off; off = align_up(off + sizeof(SampleState));
  w.bm_off = off; off = align_up(off + (size_t)nb * nb * 8);
  w.d_off = off; off = align_up(off + (size_t)nb * 8);
  w.msg_off = off; off = align_up(off + m.header_bytes + (size_t)w.ldw * nb * 8);
  w.total = off;
  return w;
}

__global__ void pack_header_kernel(const SampleState* st, const double* T11, int64_t ld, int jb,
                                   const uint8_t* mask_j0, char* msg, MsgLayout m) {
  const int t = threadIdx.x;
  if (t == 0) *reinterpret_cast<SampleState*>(msg) = *st;
  for (int k = t; k < jb; k += blockDim.x) {
    reinterpret_cast<double*>(msg + m.d_off)[k] = T11[(int64_t)k * ld + k];
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
  if (ncclCommInitRank(&c->nccl, nranks, uid, rank) != ncclSuccess) { delete c; return DPP_ENCCL; }
  *comm = c;
  return DPP_OK;
}

int dpp_comm_destroy(dpp_comm_t comm) {
  if (!comm) return DPP_EINVAL;
  ncclResult_t r = ncclCommDestroy(comm->nccl);
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
  if ((op & 3) != DPP_OP_HERM_D || n < 0 || nranks < 1) return 0;
  const int nb = (opts && opts->nb) ? opts->nb : 128;
  if (nb != 128) return 0;
  return dist_ws(n, nb).total;
}

int dpp_sample_herm_d_dist(dpp_comm_t comm, int64_t n, double* K_local, int64_t ld_local, uint64_t seed,
                           uint8_t* mask, double* loglik, dpp_info_t* info, const dpp_opts_t* opts, void* work,
                           size_t work_bytes, dpp_stream_t stream_) {
  if (!comm || n < 0 || !loglik || (n > 0 && (!mask || !K_local)) || ld_local < std::max<int64_t>(n, 1))
    return DPP_EINVAL;
  const int nb = (opts && opts->nb) ? opts->nb : 128;
  if (nb != 128) return DPP_EINVAL;  // the update kernel's tile width equals the block width
  const double tie_tol = (opts && opts->tie_tol > 0) ? opts->tie_tol : 1e-9;
  const double range_tol = (opts && opts->range_tol > 0) ? opts->range_tol : 1e-8;
  const uint8_t* forced = opts ? opts->forced : nullptr;
  cudaStream_t st = (cudaStream_t)stream_;
  DistWs W = dist_ws(n, nb);
  if (!work || work_bytes < W.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  if (n == 0) { CK(launch_zero_state(nullptr, loglik, info, 1, st)); return DPP_OK; }
  const int P = comm->nranks, r = comm->rank;
  char* w = reinterpret_cast<char*>(work);
  SampleState* state = reinterpret_cast<SampleState*>(w + W.state_off);
  double* Bm = reinterpret_cast<double*>(w + W.bm_off);
  double* dvec = reinterpret_cast<double*>(w + W.d_off);
  char* msg = w + W.msg_off;
  const MsgLayout M = msg_layout(nb);
  double* Lmsg = reinterpret_cast<double*>(msg + M.w_off);          // L21 rows j1.., ld = ldw
  const double* Dmsg = reinterpret_cast<const double*>(msg + M.d_off);
  const int64_t nblk = (n + nb - 1) / nb;
  const bool vec = (ld_local % 2 == 0) && (reinterpret_cast<uintptr_t>(K_local) % 16 == 0);

  for (int64_t k = 0; k < nblk; ++k) {
    const int owner = (int)(k % P);
    const int64_t j0 = k * nb;
    const int jb = (int)std::min<int64_t>(nb, n - j0);
    const int64_t j1 = j0 + jb, m2 = n - j1;
    const int64_t lq = k / P;                 // local block index of block k on its owner
    const int64_t tcol = lq * nb;             // storage column on the owner
    if (r == owner) {
      DiagArgs d{};
      d.A = K_local; d.ld = ld_local; d.strideA = 0; d.n = n; d.j0 = j0; d.tcol = tcol; d.jb = jb;
      d.seed = seed; d.b0 = 0; d.mask = mask; d.forced = forced; d.state = state; d.loglik = nullptr;
      d.info = nullptr; d.tie_tol = tie_tol; d.range_tol = range_tol; d.batch = 1;
      d.need_ops = m2 > 0; d.Bm = Bm; d.dvec = dvec; d.ldm = nb; d.strideM = 0;
      CK(launch_diag(HERM_D, nb, d, st));
      if (m2 > 0) {
        // stage 2 in place: L21 = A21 L11^-T D1^-1, then into the message
        UpdateArgs p{};
        p.Aop = K_local + j1 + tcol * ld_local; p.lda = ld_local;
        p.Bop = Bm; p.ldb = nb;
        p.C = K_local + j1 + tcol * ld_local; p.ldc = ld_local;
        p.a_rows = (int)m2; p.b_rows = jb; p.K = jb; p.rows = (int)m2; p.cols = jb; p.batch = 1; p.vec = vec ? 1 : 0;
        CK(launch_update(HERM_D, p, st));
        CK(cudaMemcpy2DAsync(Lmsg, (size_t)W.ldw * 8, K_local + j1 + tcol * ld_local, (size_t)ld_local * 8,
                             (size_t)m2 * 8, (size_t)jb, cudaMemcpyDeviceToDevice, st));
      }
      pack_header_kernel<<<1, 128, 0, st>>>(state, K_local + j0 + tcol * ld_local, ld_local, jb, mask + j0, msg, M);
      CK(cudaGetLastError());
    }
    // one exchange per block step: header (+ L21 when a trailing matrix remains)
    const size_t bytes = M.header_bytes + (m2 > 0 ? (size_t)W.ldw * (size_t)jb * 8 : 0);
    if (P > 1) NK(ncclBroadcast(msg, msg, bytes, ncclChar, owner, comm->nccl, st));
    if (r != owner) {
      unpack_header_kernel<<<1, 128, 0, st>>>(msg, M, jb, state, mask + j0);
      CK(cudaGetLastError());
    }
    if (m2 <= 0) break;
    // stage 3 on the local trailing block columns: blocks c > k with c = r + q P
    const int64_t q0 = (k + 1 - r + P - 1) / P;  // first q with r + qP > k
    const int64_t nloc = (nblk - r + P - 1) / P;  // local blocks on r
    if (q0 < nloc) {
      UpdateArgs u{};
      u.Aop = Lmsg; u.lda = W.ldw;
      u.Bop = Lmsg; u.ldb = W.ldw; u.dscale = Dmsg; u.mask = 1;
      u.C = K_local + j1;  // local column 0, A22 row 0
      u.ldc = ld_local;
      u.a_rows = (int)m2; u.b_rows = (int)m2; u.K = jb; u.batch = 1; u.vec = vec ? 1 : 0;
      u.row0 = 0; u.rows = (int)m2; u.col0 = 0; u.cols = (int)m2; u.tri = 0;
      u.bcc_P = P; u.bcc_r = r; u.bcc_nb = nb; u.bcc_q0 = (int)q0; u.bcc_j1 = j1;
      u.tiles_n = (int)(nloc - q0);
      CK(launch_update(HERM_D, u, st));
    }
  }
  // the final state lives on the owner of the last block; its header went out in the last step
  finalize_kernel<<<1, 32, 0, st>>>(state, loglik, info);
  CK(cudaGetLastError());
  return DPP_OK;
}

}  // extern "C"
