// lensemble.cu -- L-ensemble -> marginal kernel conversion K = I - (L + I)^{-1} (
// "the incorporation of a tiled extension of [Bientinesi et al. 2008] for
// converting a Hermitian L-ensemble kernel into a marginal kernel via K = I - (L + I)^{-1} ... could be
// expected to require the equivalent of 3 samples worth of time").
//
// Real symmetric (fp64, tiles of 128) and complex Hermitian (complex128, tiles of 64).  Three n^3/3
// phases, every one on the kernels of the sampler:
//   1. M = L + I = Lf D Lf^T: the sampler itself with every decision forced to "keep" (no pivot is
//      modified, so the modified factorization IS the plain LDL^T; its log-likelihood is ln det M);
//   2. Y = Lf^{-T} (upper triangular, the transpose of the unit-lower inverse X = Lf^{-1}) by block
//      forward substitution over block rows of X, right-looking: with the diagonal-tile inverses
//      Lkk^{-1} (tile_inverse_kernel) every step is two DMMA GEMMs on column panels of Y --
//        Y(:, k)  <- Y(:, k) Lkk^{-T}           (in place, as Y - Y (I - Lkk^{-1})^T)
//        Y(:, >k) -= Y(:, k) L(>k, k)^T
//   3. K = I - M^{-1} = I - Y D^{-1} Y^T on the lower triangle: one HERK-shaped DMMA pass (K = n, B
//      scaled by D^{-1} on load, each tile's K loop starting at its first row since Y is upper
//      triangular), written over L.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "tri_inverse.cuh"

namespace dpp {

template <typename T>
__global__ void lens_add_diag_kernel(T* A, int64_t ld, int64_t n, double v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[i + i * ld] = make_real(re(A[i + i * ld]) + v, zero<T>());  // Im of a diagonal is 0 (R5)
}

// D^{-1} from the factored diagonal; Y := I (full n x n, column-major, ld = ldy)
template <typename T>
__global__ void lens_prepare_kernel(const T* A, int64_t ld, int64_t n, double* dinv, T* Y, int64_t ldy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    dinv[i] = 1.0 / re(A[i + i * ld]);
    Y[i + i * ldy] = make_real(1.0, zero<T>());
  }
}

// K's lower triangle := I (the output of the final pass accumulates -Y D^{-1} Y^H into it)
template <typename T>
__global__ void lens_identity_lower_kernel(T* A, int64_t ld, int64_t n) {
  const int64_t j = blockIdx.x;
  for (int64_t i = j + threadIdx.x; i < n; i += blockDim.x)
    A[i + j * ld] = (i == j) ? make_real(1.0, zero<T>()) : zero<T>();
}

// Am_k(j, kk) = -Linv_kk(j, kk) (j > kk), else 0, for the unit-lower diagonal tile k of the factor
// (strict lower part of A); nb x nb per tile, column-major, ld = nb.
template <typename T, int NB>
__global__ void __launch_bounds__(256) lens_tile_inverse_kernel(const T* A, int64_t ld, int64_t n, T* Am) {
  constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;
  extern __shared__ __align__(16) unsigned char dsm[];
  T* Lb = reinterpret_cast<T*>(dsm);
  T* Xb = Lb + NPB * BLK_SZ;
  T* Tb = Xb + NPB * BLK_SZ;
  const int64_t k = blockIdx.x, j0 = k * NB;
  const int jb = (int)min((int64_t)NB, n - j0);
  const T* Tl = A + j0 + j0 * ld;
  const T one = make_real(1.0, zero<T>());
  for (int idx = threadIdx.x; idx < NB * NB; idx += 256) {
    const int l = idx / NB, i = idx % NB;
    if (i >= l) Lb[bp(i, l)] = (i == l) ? one : ((i < jb && l < jb) ? Tl[i + (int64_t)l * ld] : zero<T>());
  }
  __syncthreads();
  tri_inverse_lower<T, true, 256>(Lb, Xb, Tb, (jb + 15) >> 4);
  T* M = Am + k * (int64_t)NB * NB;
  for (int l = threadIdx.x >> 5; l < jb; l += 8)
    for (int i = threadIdx.x & 31; i < jb; i += 32) M[i + (int64_t)l * NB] = (i > l) ? neg(Xb[bp(i, l)]) : zero<T>();
}

}  // namespace dpp

namespace {
constexpr size_t ALIGN = 256;
inline size_t align_up(size_t x) { return (x + ALIGN - 1) / ALIGN * ALIGN; }
struct LensWs {
  size_t samp_off, samp_bytes, forced_off, mask_off, ll_off, am_off, dinv_off, y_off, total;
  int64_t ldy;
  int nb;
};
LensWs lens_ws(dpp::Kind kind, int64_t n) {
  LensWs w;
  w.nb = kind == dpp::HERM_D ? 128 : 64;  // the sampler's tile for the kind
  const size_t es = kind == dpp::HERM_D ? 8 : 16;
  dpp_opts_t o{};
  o.nb = w.nb;
  o.lookahead = 1;
  w.samp_bytes = dpp_workspace_bytes(kind == dpp::HERM_D ? DPP_OP_HERM_D : DPP_OP_HERM_Z, 1, n, &o);
  w.ldy = std::max<int64_t>((n + 15) / 16 * 16, 16);
  const int64_t nblk = (n + w.nb - 1) / w.nb;
  size_t off = 0;
  w.samp_off = off; off = align_up(off + w.samp_bytes);
  w.forced_off = off; off = align_up(off + (size_t)std::max<int64_t>(n, 1));
  w.mask_off = off; off = align_up(off + (size_t)std::max<int64_t>(n, 1));
  w.ll_off = off; off = align_up(off + 8);
  w.am_off = off; off = align_up(off + (size_t)nblk * w.nb * w.nb * es);
  w.dinv_off = off; off = align_up(off + (size_t)std::max<int64_t>(n, 1) * 8);
  w.y_off = off; off = align_up(off + (size_t)w.ldy * std::max<int64_t>(n, 1) * es);
  w.total = off;
  return w;
}

template <typename T, int NB>
int lens_run(dpp::Kind kind, int64_t n, T* A, int64_t ld, double* logdet, void* work, size_t work_bytes,
             dpp_stream_t stream_) {
  using namespace dpp;
  const bool cplx = kind == HERM_Z;
  if (n < 0 || ld < std::max<int64_t>(1, n) || (n > 0 && !A)) return DPP_EINVAL;
  if (n > (int64_t)1 << 30) return DPP_EINVAL;
  if (cplx && reinterpret_cast<uintptr_t>(A) % 16) return DPP_EINVAL;
  const LensWs W = lens_ws(kind, n);
  if (!work || work_bytes < W.total || reinterpret_cast<uintptr_t>(work) % ALIGN) return DPP_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream_;
  char* w = reinterpret_cast<char*>(work);
  double* ll = reinterpret_cast<double*>(w + W.ll_off);
  if (n == 0) {
    if (logdet && cudaMemsetAsync(logdet, 0, 8, st) != cudaSuccess) return DPP_ECUDA;
    return DPP_OK;
  }
  // 16-byte aligned columns of L take the TMA-fed kernel, others the cp.async fallback (Y always aligned)
  const int avec = (((size_t)ld * sizeof(T)) % 16 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0) ? 1 : 0;
  const unsigned g1 = (unsigned)((n + 255) / 256);
  // ---- 1. M = L + I = Lf D Lf^H: the sampler with every decision forced to "keep"
  lens_add_diag_kernel<T><<<g1, 256, 0, st>>>(A, ld, n, 1.0);
  uint8_t* forced = reinterpret_cast<uint8_t*>(w + W.forced_off);
  if (cudaMemsetAsync(forced, 1, (size_t)n, st) != cudaSuccess) return DPP_ECUDA;
  dpp_opts_t o{};
  o.nb = NB;
  o.lookahead = 1;
  o.forced = forced;
  int rc = cplx ? dpp_sample_herm_z(n, reinterpret_cast<dpp_complex_t*>(A), ld, 0, reinterpret_cast<uint8_t*>(w + W.mask_off),
                                    ll, nullptr, &o, w + W.samp_off, W.samp_bytes, stream_)
                : dpp_sample_herm_d(n, reinterpret_cast<double*>(A), ld, 0, reinterpret_cast<uint8_t*>(w + W.mask_off),
                                    ll, nullptr, &o, w + W.samp_off, W.samp_bytes, stream_);
  if (rc) return rc;
  if (logdet && cudaMemcpyAsync(logdet, ll, 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return DPP_ECUDA;
  // ---- 2. Y = Lf^{-H}
  const int64_t nblk = (n + NB - 1) / NB;
  T* Am = reinterpret_cast<T*>(w + W.am_off);
  double* dinv = reinterpret_cast<double*>(w + W.dinv_off);
  T* Y = reinterpret_cast<T*>(w + W.y_off);
  {
    constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;
    const size_t smem = (size_t)(2 * NPB + NBLK - 1) * BLK_SZ * sizeof(T);
    if (cudaFuncSetAttribute(lens_tile_inverse_kernel<T, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return DPP_ECUDA;
    lens_tile_inverse_kernel<T, NB><<<(unsigned)nblk, 256, smem, st>>>(A, ld, n, Am);
  }
  if (cudaMemsetAsync(Y, 0, (size_t)W.ldy * n * sizeof(T), st) != cudaSuccess) return DPP_ECUDA;
  lens_prepare_kernel<T><<<g1, 256, 0, st>>>(A, ld, n, dinv, Y, W.ldy);
  if (cudaGetLastError() != cudaSuccess) return DPP_ECUDA;
  for (int64_t k = 0; k < nblk; ++k) {
    const int64_t j0 = k * NB;
    const int jb = (int)std::min<int64_t>(NB, n - j0);
    const int64_t r = j0 + jb;  // rows of Y's block column k that can be nonzero
    UpdateArgs u{};
    u.batch = 1; u.vec = 1; u.conj = cplx;
    // Y(:, k) <- Y(:, k) - Y(:, k) (I - Lkk^{-1})^H   (in place; one column tile; op(B) = conj(Am))
    u.Aop = Y + j0 * W.ldy; u.lda = W.ldy;
    u.Bop = Am + k * (int64_t)NB * NB; u.ldb = NB;
    u.C = Y + j0 * W.ldy; u.ldc = W.ldy;
    u.a_rows = (int)r; u.b_rows = jb; u.K = jb;
    u.rows = (int)r; u.cols = jb;
    if (launch_update(kind, u, st) != cudaSuccess) return DPP_ECUDA;
    if (r < n) {
      // Y(0:r, r:n) -= Y(0:r, k) L(r:n, k)^H
      UpdateArgs v{};
      v.batch = 1; v.vec = avec; v.conj = cplx;
      v.Aop = Y + j0 * W.ldy; v.lda = W.ldy;
      v.Bop = A + r + j0 * ld; v.ldb = ld;
      v.C = Y + r * W.ldy; v.ldc = W.ldy;
      v.a_rows = (int)r; v.b_rows = (int)(n - r); v.K = jb;
      v.rows = (int)r; v.cols = (int)(n - r);
      if (launch_update(kind, v, st) != cudaSuccess) return DPP_ECUDA;
    }
  }
  // ---- 3. K = I - Y D^{-1} Y^H on the lower triangle, over L
  lens_identity_lower_kernel<T><<<(unsigned)n, 256, 0, st>>>(A, ld, n);
  UpdateArgs s{};
  s.batch = 1; s.vec = avec; s.conj = cplx;
  s.Aop = Y; s.lda = W.ldy;
  s.Bop = Y; s.ldb = W.ldy; s.dscale = dinv; s.dstride = 0;
  s.C = A; s.ldc = ld;
  s.a_rows = (int)n; s.b_rows = (int)n; s.K = (int)n;
  s.rows = (int)n; s.cols = (int)n; s.tri = 1; s.mask = 1; s.ktri = 1;
  if (launch_update(kind, s, st) != cudaSuccess) return DPP_ECUDA;
  return cudaGetLastError() == cudaSuccess ? DPP_OK : DPP_ECUDA;
}
}  // namespace

extern "C" {

size_t dpp_lensemble_workspace_bytes(int op, int64_t n) {
  if (n < 0 || (op != DPP_OP_HERM_D && op != DPP_OP_HERM_Z)) return 0;
  return lens_ws(op == DPP_OP_HERM_D ? dpp::HERM_D : dpp::HERM_Z, n).total;
}

int dpp_lensemble_to_marginal_d(int64_t n, double* A, int64_t ld, double* logdet, void* work, size_t work_bytes,
                                dpp_stream_t stream) {
  return lens_run<double, 128>(dpp::HERM_D, n, A, ld, logdet, work, work_bytes, stream);
}

int dpp_lensemble_to_marginal_z(int64_t n, dpp_complex_t* A, int64_t ld, double* logdet, void* work,
                                size_t work_bytes, dpp_stream_t stream) {
  return lens_run<double2, 64>(dpp::HERM_Z, n, reinterpret_cast<double2*>(A), ld, logdet, work, work_bytes, stream);
}

}  // extern "C"
