// diag.cu -- Stage 1: sequential sample-and-factor of one diagonal tile.
//
// Listing 4 replaces the diagonal-block LU of Listing 3 (line 583) by the
// unblocked sampler of Listing 1 applied to A_J1:
//   for k in J1:  keep iff u_k <= Re A(k,k)  else A(k,k) -= 1          (line 437)
//                 A(k+1:, k) /= A(k,k)                                  (line 438)
//                 A(k+1:, k+1:) -= A(k+1:, k) A(k, k+1:)                (line 439)
// Prop. 5 ("the subtraction of 1 from each eliminated pivot commutes with the
// outer product updates") makes taking these decisions tile-locally exact.
//
// Design (B200): one CTA per (tile, sample); the whole jb x jb tile lives in shared memory
// (real nb=128: 128 KB); 8 warps; warps own trailing columns round-robin, lanes own rows.
// One __syncthreads per pivot: the scaled column k (and pivot) are written back at the start
// of step k+1 (nobody reads column k during step k+1), so the pivot step needs no second barrier.
// The Hermitian path reads/writes the lower triangle only.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace dpp {

template <typename T, bool HERM, int NB, int NT>
__global__ void __launch_bounds__(NT) diag_kernel(const DiagArgs a) {
  constexpr int NW = NT / 32;
  constexpr int RC = (NB + 31) / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* S = reinterpret_cast<T*>(smem_raw);               // S(i,l) at l*NB + i
  double* U = reinterpret_cast<double*>(S + NB * NB);  // uniforms of the tile's pivots
  uint8_t* keepv = reinterpret_cast<uint8_t*>(U + NB);

  const int s = blockIdx.y;
  const int jb = a.jb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA + a.j0 + a.tcol * a.ld;
  SampleState* st = reinterpret_cast<SampleState*>(a.state) + s;
  const uint64_t b = a.b0 + (uint64_t)s;

  // ---- stage the tile (Hermitian: lower triangle only) and this tile's uniforms
  for (int l = warp; l < jb; l += NW)
    for (int i = lane; i < jb; i += 32)
      if (!HERM || i >= l) S[l * NB + i] = A[(int64_t)l * a.ld + i];
  for (int k = tid; k < jb; k += NT) {
    U[k] = uniform_u(a.seed, (uint64_t)(a.j0 + k), b);
    if (a.forced) keepv[k] = a.forced[(int64_t)s * a.n + a.j0 + k] != 0;
  }

  // thread 0 carries the running per-sample state in pivot order
  double ll = 0.0, minabs = INFINITY, maximag = 0.0;
  int nkept = 0, nties = 0, firsttie = -1, noor = 0;
  if (tid == 0 && a.j0 > 0) {
    ll = st->loglik; minabs = st->min_abs_pivot; maximag = st->max_abs_imag_pivot;
    nkept = st->n_kept; nties = st->n_ties; firsttie = st->first_tie; noor = st->n_out_of_range;
  }
  __syncthreads();

  T Lprev[RC];
  T pprev = zero<T>();
#pragma unroll
  for (int c = 0; c < RC; ++c) Lprev[c] = zero<T>();

  for (int k = 0; k < jb; ++k) {
    // deferred write-back of step k-1: scaled column k-1 and its final pivot
    if (k > 0 && warp == (k - 1) % NW) {
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        const int i = lane + 32 * c;
        if (i > k - 1 && i < jb) S[(k - 1) * NB + i] = Lprev[c];
      }
      if (lane == 0) S[(k - 1) * NB + (k - 1)] = pprev;
    }
    T p = S[k * NB + k];
    if (HERM) p = make_real(re(p), p);
    const double d = re(p);
    const double u = U[k];
    const bool keep = a.forced ? (keepv[k] != 0) : (u <= d);
    if (!keep) p = sub_one(p);  // Listing 1: A_j -= 1
    if (tid == 0) {
      if (fabs(u - d) <= a.tie_tol) { if (nties == 0) firsttie = (int)(a.j0 + k); ++nties; }
      if (d < -a.range_tol || d > 1.0 + a.range_tol) ++noor;
      if (!HERM) maximag = fmax(maximag, fabs(im(S[k * NB + k])));
      const double ap = absval(p);
      ll += log(ap);
      minabs = fmin(minabs, ap);
      nkept += keep ? 1 : 0;
      if (!a.forced) keepv[k] = keep ? 1 : 0;
    }
    const T r = recip(p);
    // line 438: L(i,k) = A(i,k) / p for this lane's rows
    T Lk[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      const int i = lane + 32 * c;
      Lk[c] = (i > k && i < jb) ? mul(S[k * NB + i], r) : zero<T>();
    }
    // line 439: rank-1 update of the trailing part of the tile
    for (int l = k + 1 + warp; l < jb; l += NW) {
      const T bl = HERM ? cj(S[k * NB + l]) : S[l * NB + k];  // conj(w_l) or U(k,l)
      T* col = S + l * NB;
#pragma unroll
      for (int c = 0; c < RC; ++c) {
        const int i = lane + 32 * c;
        if ((HERM ? (i >= l) : (i > k)) && i < jb) col[i] = fms(col[i], Lk[c], bl);
      }
    }
#pragma unroll
    for (int c = 0; c < RC; ++c) Lprev[c] = Lk[c];
    pprev = p;
    __syncthreads();
  }
  if (jb > 0 && warp == (jb - 1) % NW) {
    if (lane == 0) S[(jb - 1) * NB + (jb - 1)] = pprev;
  }
  __syncthreads();

  // ---- write the factored tile, decisions and state back
  for (int l = warp; l < jb; l += NW)
    for (int i = lane; i < jb; i += 32)
      if (!HERM || i >= l) A[(int64_t)l * a.ld + i] = S[l * NB + i];
  for (int k = tid; k < jb; k += NT) a.mask[(int64_t)s * a.n + a.j0 + k] = keepv[k];
  if (tid == 0) {
    st->loglik = ll; st->min_abs_pivot = minabs; st->max_abs_imag_pivot = maximag;
    st->n_kept = nkept; st->n_ties = nties; st->first_tie = firsttie; st->n_out_of_range = noor;
    if (a.j0 + jb == a.n && a.loglik) {
      a.loglik[s] = ll;
      if (a.info) {
        dpp_info_t* inf = reinterpret_cast<dpp_info_t*>(a.info) + s;
        inf->n_kept = nkept; inf->n_ties = nties; inf->first_tie = firsttie; inf->n_out_of_range = noor;
        inf->min_abs_pivot = minabs; inf->max_abs_imag_pivot = maximag;
      }
    }
  }
}

template <typename T, bool HERM, int NB>
static cudaError_t launch_diag_t(const DiagArgs& a, cudaStream_t s) {
  constexpr int NT = 256;
  const size_t smem = (size_t)NB * NB * sizeof(T) + NB * sizeof(double) + NB;
  auto* fn = diag_kernel<T, HERM, NB, NT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(1, a.batch);
  fn<<<grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

size_t diag_smem_bytes(Kind kind, int nb) {
  return (size_t)nb * nb * (kind == HERM_D ? 8 : 16) + nb * 9;
}

cudaError_t launch_diag(Kind kind, int nb, const DiagArgs& a, cudaStream_t s) {
  switch (kind) {
    case HERM_D:
      if (nb <= 32) return launch_diag_t<double, true, 32>(a, s);
      if (nb <= 64) return launch_diag_t<double, true, 64>(a, s);
      return launch_diag_t<double, true, 128>(a, s);
    case HERM_Z:
      if (nb <= 32) return launch_diag_t<double2, true, 32>(a, s);
      return launch_diag_t<double2, true, 64>(a, s);
    case LU_Z:
      if (nb <= 32) return launch_diag_t<double2, false, 32>(a, s);
      return launch_diag_t<double2, false, 64>(a, s);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- small helpers
__global__ void uniforms_kernel(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) u[i] = uniform_u(seed, j0 + (uint64_t)i, b);
}

cudaError_t launch_uniforms(uint64_t seed, uint64_t j0, uint64_t b, int64_t count, double* u, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  uniforms_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(seed, j0, b, count, u);
  return cudaGetLastError();
}

__global__ void zero_state_kernel(double* loglik, dpp_info_t* info, int batch) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) {
    loglik[i] = 0.0;
    if (info) {
      info[i].n_kept = 0; info[i].n_ties = 0; info[i].first_tie = -1; info[i].n_out_of_range = 0;
      info[i].min_abs_pivot = INFINITY; info[i].max_abs_imag_pivot = 0.0;
    }
  }
}

cudaError_t launch_zero_state(void*, double* loglik, void* info, int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  zero_state_kernel<<<(batch + 127) / 128, 128, 0, s>>>(loglik, reinterpret_cast<dpp_info_t*>(info), batch);
  return cudaGetLastError();
}

}  // namespace dpp
