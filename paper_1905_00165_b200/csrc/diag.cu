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
// Design (B200, latency-bound: jb dependent pivot steps):
//  * one CTA of 256 threads per (tile, sample); the tile lives in REGISTERS, distributed 2-D
//    cyclically over a 16 x 16 thread grid (thread (tr, tc) owns rows tr + 16a, cols tc + 16b);
//  * per pivot only the pivot column (and, for LU, the pivot row) goes through shared memory,
//    double-buffered, so each pivot step costs exactly one __syncthreads;
//  * the rank-1 update is branch-free (eliminated rows/columns carry zero multipliers; Hermitian
//    blocks strictly above the diagonal are skipped at compile time);
//  * column k keeps its unscaled values after step k; the scaling L = w * (1/p) and the final
//    pivots are applied once at the end (reading R17), and the log-likelihood / tie / range
//    bookkeeping is done in parallel after the loop and summed by one thread IN PIVOT ORDER.
// The Hermitian path reads/writes the lower triangle only.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace dpp {

template <typename T, bool HERM, int NB>
__global__ void __launch_bounds__(256, 1) diag_kernel(const DiagArgs a) {
  constexpr int TR = 16, TC = 16, RA = NB / TR, CB = NB / TC;
  __shared__ T colbuf[2][NB];
  __shared__ T rowbuf[HERM ? 1 : 2][HERM ? 1 : NB];
  __shared__ T pv[NB], rv[NB];
  __shared__ double U[NB], dv[NB], imv[NB], lg[NB];
  __shared__ uint8_t keepv[NB];

  const int s = blockIdx.y;
  const int jb = a.jb;
  const int tid = threadIdx.x;
  const int tr = tid % TR, tc = tid / TR;
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA + a.j0 + a.tcol * a.ld;
  SampleState* st = reinterpret_cast<SampleState*>(a.state) + s;
  const uint64_t b = a.b0 + (uint64_t)s;

  // ---- stage: registers (Hermitian: lower triangle only), uniforms, forced decisions
  T R[RA][CB];
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int i = tr + TR * ia, l = tc + TC * ib;
      R[ia][ib] = (i < jb && l < jb && (!HERM || i >= l)) ? A[(int64_t)l * a.ld + i] : zero<T>();
    }
  for (int k = tid; k < jb; k += 256) {
    U[k] = uniform_u(a.seed, (uint64_t)(a.j0 + k), b);
    if (a.forced) keepv[k] = a.forced[(int64_t)s * a.n + a.j0 + k] != 0;
  }
  // publish pivot column 0 (and row 0)
  if (tc == 0) {
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) colbuf[0][tr + TR * ia] = R[ia][0];
  }
  if (!HERM && tr == 0) {
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) rowbuf[0][tc + TC * ib] = R[0][ib];
  }
  __syncthreads();

  for (int k = 0; k < jb; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    T p = colbuf[cur][k];
    if (HERM) p = make_real(re(p), p);
    const double d = re(p);
    const bool keep = a.forced ? (keepv[k] != 0) : (U[k] <= d);
    if (!keep) p = sub_one(p);  // Listing 1
    const T r = recip(p);
    if (tid == 0) {
      pv[k] = p; rv[k] = r; dv[k] = d; imv[k] = im(colbuf[cur][k]);
      if (!a.forced) keepv[k] = keep ? 1 : 0;
    }
    // multipliers: L(i,k) = w_i / p (line 438) for my rows, conj(w_l) or U(k,l) for my columns
    T Li[RA], Wl[CB];
#pragma unroll
    for (int ia = 0; ia < RA; ++ia) {
      const int i = tr + TR * ia;
      Li[ia] = (i > k && i < jb) ? mul(colbuf[cur][i], r) : zero<T>();
    }
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int l = tc + TC * ib;
      Wl[ib] = (l > k && l < jb) ? (HERM ? cj(colbuf[cur][l]) : rowbuf[HERM ? 0 : cur][l]) : zero<T>();
    }
    // rank-1 update (line 439); eliminated rows/columns have zero multipliers, so the update is
    // branch-free (Hermitian: blocks strictly above the diagonal are skipped statically)
#pragma unroll
    for (int ia = 0; ia < RA; ++ia)
#pragma unroll
      for (int ib = 0; ib < CB; ++ib)
        if (!HERM || ib <= ia) R[ia][ib] = fms(R[ia][ib], Li[ia], Wl[ib]);
    // publish pivot column k+1 (and row k+1) for the next step
    // (the owning register is selected with compile-time indices only: a runtime index into R
    //  would demote the tile to local memory)
    const int kn = k + 1;
    if (kn < jb) {
#pragma unroll
      for (int ib = 0; ib < CB; ++ib) {
        if (tc + TC * ib == kn) {
#pragma unroll
          for (int ia = 0; ia < RA; ++ia) {
            const int i = tr + TR * ia;
            if (i >= kn) colbuf[nxt][i] = R[ia][ib];
          }
        }
      }
      if (!HERM) {
#pragma unroll
        for (int ia = 0; ia < RA; ++ia) {
          if (tr + TR * ia == kn) {
#pragma unroll
            for (int ib = 0; ib < CB; ++ib) {
              const int l = tc + TC * ib;
              if (l > kn) rowbuf[HERM ? 0 : nxt][l] = R[ia][ib];
            }
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- finalize the factor: L = (unscaled column) * (1/p), diagonal = final pivot
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int i = tr + TR * ia, l = tc + TC * ib;
      if (i < jb && l < jb && (!HERM || i >= l)) {
        T v = R[ia][ib];
        if (i > l) v = mul(v, rv[l]);
        else if (i == l) v = pv[l];
        A[(int64_t)l * a.ld + i] = v;
      }
    }
  // ---- decisions, likelihood terms and diagnostics, in parallel; summed in pivot order
  for (int k = tid; k < jb; k += 256) {
    a.mask[(int64_t)s * a.n + a.j0 + k] = keepv[k];
    lg[k] = log(absval(pv[k]));
  }
  __syncthreads();
  if (tid == 0) {
    double ll = 0.0, minabs = INFINITY, maximag = 0.0;
    int nkept = 0, nties = 0, firsttie = -1, noor = 0;
    if (a.j0 > 0) {
      ll = st->loglik; minabs = st->min_abs_pivot; maximag = st->max_abs_imag_pivot;
      nkept = st->n_kept; nties = st->n_ties; firsttie = st->first_tie; noor = st->n_out_of_range;
    }
    for (int k = 0; k < jb; ++k) {
      const double d = dv[k], u = U[k];
      if (fabs(u - d) <= a.tie_tol) { if (nties == 0) firsttie = (int)(a.j0 + k); ++nties; }
      if (d < -a.range_tol || d > 1.0 + a.range_tol) ++noor;
      if (!HERM) maximag = fmax(maximag, fabs(imv[k]));
      ll += lg[k];
      minabs = fmin(minabs, absval(pv[k]));
      nkept += keepv[k];
    }
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
  dim3 grid(1, a.batch);
  diag_kernel<T, HERM, NB><<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

size_t diag_smem_bytes(Kind kind, int nb) {
  return (size_t)nb * (kind == HERM_D ? 8 : 16) * 6 + nb * 33;
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
