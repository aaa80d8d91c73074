// elementary.cu -- elementary (projection) DPP sampler: Listing 2
// (PAPER.md:514-537), Theorem "Factorization-based elementary DPP sampling".
//
// For a rank-k orthogonal projection K, k steps of a left-looking, diagonally pivoted Cholesky
// factorization whose pivot j is DRAWN from the current diagonal d with probability d_t / (k - j):
//   t_j ~ d / (k - j);  A_j = sqrt(d_t);  L(:, j) = (K(:, t) - L(:, 0:j) L(t, 0:j)^T) / A_j;
//   d -= L(:, j)^2;     loglik = sum_j ln d_{t_j} = ln det(K_Y).
// Reading R20: no physical swap; the candidates are the unchosen items in original
// index order and t_j is the first whose running sum of d exceeds u_j * sum(d), u_j the Philox
// uniform of pivot j and sample b (R2).
//
// B200 mapping (a batch of independent samples; the work is a sequence of k GEMVs, HBM/L2-bound):
//   * elem_select_kernel: one 1024-thread CTA per sample -- block-wide scan of d over the n items
//     (each thread a contiguous segment), the draw, the pivot bookkeeping, and a copy of the
//     pivot's factor row L(t, 0:j) next to the state;
//   * elem_column_kernel: one thread per (row, sample): the new column as a dot product over j
//     factor columns (coalesced column-major reads, 4 independent partial sums), divided by A_j,
//     and the diagonal update.
// Both are launched once per step on the caller's stream (2k launches per call) -- or, when the
// batch has at least one sample per SM, elem_fused_kernel runs all k steps of a sample in one CTA
// (one launch per call).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace dpp {

struct ElemState {
  int64_t t;        // pivot of the current step
  double Aj;        // sqrt(d_t)
  double loglik;
  int32_t n_ties, first_tie;
};

struct ElemArgs {
  const double* K;
  int64_t ld;
  int64_t n, k;
  uint64_t seed, b0;
  double tie_tol;
  double* L;        // per sample: n x k, leading dimension ldL
  int64_t ldL, strideL;
  double* d;        // per sample: n
  uint8_t* chosen;  // per sample: n
  double* lt;       // per sample: k (the pivot's factor row)
  ElemState* st;    // per sample
  int64_t* order;   // batch x k
  double* loglik;   // batch
  int32_t* ties;    // batch x 2 (n_ties, first_tie) or null
};

__global__ void elem_init_kernel(ElemArgs a) {
  const int64_t s = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.n) {
    a.d[s * a.n + i] = a.K[i + i * a.ld];  // d := diag(K)
    a.chosen[s * a.n + i] = 0;
  }
  if (i == 0) {
    ElemState& st = a.st[s];
    st.t = -1; st.Aj = 0.0; st.loglik = 0.0; st.n_ties = 0; st.first_tie = -1;
  }
}

constexpr int SEL_T = 1024;

struct SelShared {
  double wsum[SEL_T / 32];
  double S, target;
  long long t, last;
};

// Draw of pivot j for sample s by one CTA of SEL_T threads (block-wide scan of d over the items,
// each thread a contiguous segment), the pivot bookkeeping, and the pivot's factor row L(t, 0:j)
// copied next to the state.  Ends with the CTA synchronised.
__device__ __forceinline__ void elem_select(const ElemArgs& a, int64_t s, int64_t j, SelShared& sh) {
  const double* d = a.d + s * a.n;
  uint8_t* ch = a.chosen + s * a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* wsum = sh.wsum;
  double& sh_S = sh.S;
  double& sh_target = sh.target;
  long long& sh_t = sh.t;
  long long& sh_last = sh.last;
  // contiguous segment of this thread
  const int64_t per = (a.n + SEL_T - 1) / SEL_T;
  const int64_t i0 = min((int64_t)a.n, (int64_t)tid * per), i1 = min((int64_t)a.n, i0 + per);
  double seg = 0.0;
  int64_t seg_last = -1;
  for (int64_t i = i0; i < i1; ++i)
    if (!ch[i]) {
      seg += d[i];
      if (d[i] > 0.0) seg_last = i;
    }
  // exclusive scan of the segment sums (warp shuffles, then across warps)
  double incl = seg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  if (tid == 0) { sh_t = LLONG_MAX; sh_last = -1; }
  __syncthreads();
  if (warp == 0) {
    double w = wsum[lane];
    double wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    wsum[lane] = wi - w;  // exclusive prefix of the warps
    if (lane == 31) {
      sh_S = wi;
      sh_target = uniform_u(a.seed, (uint64_t)j, a.b0 + (uint64_t)s) * wi;
    }
  }
  __syncthreads();
  const double base = wsum[warp] + incl - seg;  // running sum before my segment
  const double S = sh_S, target = sh_target;
  if (seg_last >= 0) atomicMax(&sh_last, (long long)seg_last);
  // the thread whose segment crosses the target finds t sequentially (same rule as R20); if
  // rounding puts the crossing at a segment boundary, the earliest claim wins (atomicMin)
  bool tie = false;
  if (seg > 0.0 && base <= target && base + seg > target) {
    double run = base;
    long long found = seg_last;  // rounding inside the segment: its last candidate
    for (int64_t i = i0; i < i1; ++i) {
      if (ch[i]) continue;
      const double before = run;
      run += d[i];
      if (run > target) {
        found = i;
        tie = fabs(target - before) <= a.tie_tol * S || fabs(run - target) <= a.tie_tol * S;
        break;
      }
    }
    atomicMin(&sh_t, found);
  }
  __syncthreads();
  int64_t t = sh_t;
  if (t == LLONG_MAX) t = sh_last;  // rounding left no crossing: the last candidate with d > 0
  if (tie && t >= i0 && t < i1) {
    ElemState& st = a.st[s];
    if (st.n_ties == 0) st.first_tie = (int32_t)j;
    st.n_ties += 1;
  }
  // pivot bookkeeping and the factor row L(t, 0:j)
  double* L = a.L + s * a.strideL;
  for (int64_t m = tid; m < j; m += SEL_T) a.lt[s * a.k + m] = L[t + m * a.ldL];
  if (tid == 0) {
    const double dt = d[t];
    ElemState& st = a.st[s];
    st.t = t;
    st.Aj = sqrt(dt);
    st.loglik += log(dt);
    L[t + j * a.ldL] = st.Aj;
    ch[t] = 1;
    a.order[s * a.k + j] = t;
    if (j == a.k - 1) {
      a.loglik[s] = st.loglik;
      if (a.ties) { a.ties[2 * s] = st.n_ties; a.ties[2 * s + 1] = st.first_tie; }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(SEL_T) elem_select_kernel(ElemArgs a, int64_t j) {
  __shared__ SelShared sh;
  elem_select(a, blockIdx.x, j, sh);
}

// The whole sampler for one sample per CTA (all k steps in one launch): the draw, then the new
// factor column, rows strided over the CTA's threads (for batches large enough to fill the GPU with
// one CTA per sample; removes the 2k launches per call).
__global__ void __launch_bounds__(SEL_T) elem_fused_kernel(ElemArgs a) {
  __shared__ SelShared sh;
  extern __shared__ double lt_s[];
  const int64_t s = blockIdx.x;
  double* L = a.L + s * a.strideL;
  const uint8_t* ch = a.chosen + s * a.n;
  double* d = a.d + s * a.n;
  for (int64_t i = threadIdx.x; i < a.n; i += SEL_T) {
    d[i] = a.K[i + i * a.ld];
    a.chosen[s * a.n + i] = 0;
  }
  if (threadIdx.x == 0) {
    ElemState& st = a.st[s];
    st.t = -1; st.Aj = 0.0; st.loglik = 0.0; st.n_ties = 0; st.first_tie = -1;
  }
  __syncthreads();
  for (int64_t j = 0; j < a.k; ++j) {
    elem_select(a, s, j, sh);
    if (j + 1 == a.k) break;
    for (int64_t m = threadIdx.x; m < j; m += SEL_T) lt_s[m] = a.lt[s * a.k + m];
    __syncthreads();
    const int64_t t = a.st[s].t;
    const double Aj = a.st[s].Aj;
    for (int64_t i = threadIdx.x; i < a.n; i += SEL_T) {
      if (ch[i]) {
        if (i != t) L[i + j * a.ldL] = 0.0;
        continue;
      }
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      int64_t m = 0;
      for (; m + 4 <= j; m += 4) {
        c0 = fma(L[i + m * a.ldL], lt_s[m], c0);
        c1 = fma(L[i + (m + 1) * a.ldL], lt_s[m + 1], c1);
        c2 = fma(L[i + (m + 2) * a.ldL], lt_s[m + 2], c2);
        c3 = fma(L[i + (m + 3) * a.ldL], lt_s[m + 3], c3);
      }
      for (; m < j; ++m) c0 = fma(L[i + m * a.ldL], lt_s[m], c0);
      const double c = (a.K[i + t * a.ld] - ((c0 + c1) + (c2 + c3))) / Aj;
      L[i + j * a.ldL] = c;
      d[i] -= c * c;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) elem_column_kernel(ElemArgs a, int64_t j) {
  const int64_t s = blockIdx.y;
  extern __shared__ double lt_s[];
  for (int64_t m = threadIdx.x; m < j; m += blockDim.x) lt_s[m] = a.lt[s * a.k + m];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  double* L = a.L + s * a.strideL;
  if (a.chosen[s * a.n + i]) {
    if (a.st[s].t != i) L[i + j * a.ldL] = 0.0;
    return;
  }
  const int64_t t = a.st[s].t;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
  int64_t m = 0;
  for (; m + 4 <= j; m += 4) {
    c0 = fma(L[i + m * a.ldL], lt_s[m], c0);
    c1 = fma(L[i + (m + 1) * a.ldL], lt_s[m + 1], c1);
    c2 = fma(L[i + (m + 2) * a.ldL], lt_s[m + 2], c2);
    c3 = fma(L[i + (m + 3) * a.ldL], lt_s[m + 3], c3);
  }
  for (; m < j; ++m) c0 = fma(L[i + m * a.ldL], lt_s[m], c0);
  const double c = (a.K[i + t * a.ld] - ((c0 + c1) + (c2 + c3))) / a.st[s].Aj;
  L[i + j * a.ldL] = c;
  a.d[s * a.n + i] -= c * c;
}

}  // namespace dpp

namespace {
constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }
struct ElemWs {
  size_t L_off, d_off, ch_off, lt_off, st_off, total;
  int64_t ldL;
};
ElemWs elem_ws(int64_t batch, int64_t n, int64_t k) {
  ElemWs w;
  w.ldL = std::max<int64_t>((n + 31) / 32 * 32, 32);
  size_t off = 0;
  w.L_off = off; off = align_up(off + (size_t)batch * w.ldL * std::max<int64_t>(k, 1) * 8);
  w.d_off = off; off = align_up(off + (size_t)batch * std::max<int64_t>(n, 1) * 8);
  w.ch_off = off; off = align_up(off + (size_t)batch * std::max<int64_t>(n, 1));
  w.lt_off = off; off = align_up(off + (size_t)batch * std::max<int64_t>(k, 1) * 8);
  w.st_off = off; off = align_up(off + (size_t)batch * sizeof(dpp::ElemState));
  w.total = off;
  return w;
}
}  // namespace

extern "C" {

size_t dpp_elementary_workspace_bytes(int64_t batch, int64_t n, int64_t k) {
  if (batch < 0 || n < 0 || k < 0 || k > n) return 0;
  return elem_ws(std::max<int64_t>(batch, 1), n, k).total;
}

int dpp_elementary_herm_d(int64_t batch, int64_t n, int64_t k, const double* K, int64_t ld, uint64_t seed,
                          uint64_t b0, int64_t* order, double* loglik, int32_t* ties, void* work, size_t work_bytes,
                          dpp_stream_t stream_) {
  using namespace dpp;
  if (batch < 0 || n < 0 || k < 0 || k > n || ld < std::max<int64_t>(1, n)) return DPP_EINVAL;
  if (batch == 0) return DPP_OK;
  if (batch > 65535 || (k > 0 && (!K || !order || !loglik)) || (k == 0 && !loglik)) return DPP_EINVAL;
  if ((size_t)k * 8 > 200 * 1024) return DPP_EINVAL;  // the factor row lives in shared memory
  const ElemWs W = elem_ws(batch, n, k);
  if (!work || work_bytes < W.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream_;
  char* w = reinterpret_cast<char*>(work);
  if (k == 0) {
    if (cudaMemsetAsync(loglik, 0, 8 * (size_t)batch, st) != cudaSuccess) return DPP_ECUDA;
    if (ties && cudaMemsetAsync(ties, 0, 8 * (size_t)batch, st) != cudaSuccess) return DPP_ECUDA;
    return DPP_OK;
  }
  ElemArgs a{};
  a.K = K; a.ld = ld; a.n = n; a.k = k; a.seed = seed; a.b0 = b0; a.tie_tol = 1e-12;
  a.L = reinterpret_cast<double*>(w + W.L_off); a.ldL = W.ldL; a.strideL = W.ldL * k;
  a.d = reinterpret_cast<double*>(w + W.d_off);
  a.chosen = reinterpret_cast<uint8_t*>(w + W.ch_off);
  a.lt = reinterpret_cast<double*>(w + W.lt_off);
  a.st = reinterpret_cast<ElemState*>(w + W.st_off);
  a.order = order; a.loglik = loglik; a.ties = ties;
  const size_t smem = (size_t)k * 8;
  // one CTA per sample for the whole draw when the batch fills the GPU (one launch per call: 3.7x
  // at rank 10); otherwise per-step kernels that spread each sample's column update over the SMs
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool fused = batch >= sms;
  if (fused) {
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(elem_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return DPP_ECUDA;
    elem_fused_kernel<<<(unsigned)batch, SEL_T, smem, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? DPP_OK : DPP_ECUDA;
  }
  const dim3 rows((unsigned)((n + 255) / 256), (unsigned)batch);
  elem_init_kernel<<<rows, 256, 0, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return DPP_ECUDA;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(elem_column_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return DPP_ECUDA;
  for (int64_t j = 0; j < k; ++j) {
    elem_select_kernel<<<(unsigned)batch, SEL_T, 0, st>>>(a, j);
    if (j + 1 < k) elem_column_kernel<<<rows, 256, smem, st>>>(a, j);
    if (cudaGetLastError() != cudaSuccess) return DPP_ECUDA;
  }
  return DPP_OK;
}

}  // extern "C"
