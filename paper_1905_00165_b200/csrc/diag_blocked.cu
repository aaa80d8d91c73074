// diag_blocked.cu -- Stage 1 for HERMITIAN tiles (real and complex), sub-blocked by 32 columns:
// the same sample-and-factor of the diagonal tile as diag.cu (Listing 4 -> Listing 1 on the tile,
// keep iff u_k <= Re A(k,k), else A(k,k) -= 1, then the Schur
// update of the tile), reorganised so that the sequential pivot chain runs inside ONE warp:
//   for each 32-column block c0 of the tile:
//     (a) warp 0 factors the 32 x 32 diagonal block warp-synchronously -- lane i holds row i in
//         registers, the pivot and the unscaled column are broadcast with shuffles (no block
//         barrier per pivot);
//     (b) the rows below the block are finished against it (forward substitution, one thread per
//         row: L(r, c0+p) = x_p / p_p, later columns -= L(r, c0+p) conj(w_q));
//     (c) the rest of the tile is updated with the block: A22 -= L21 D1 L21^H (lower, all threads).
// Prop. 5 makes the blocked order exact; the arithmetic differs from the
// unblocked order only by rounding (reading R17).  Outputs, diagnostics and the stage-2 operators
// are those of diag_kernel (the triangular inverse read straight from the factored tile).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"
#include "tri_inverse.cuh"

namespace dpp {

// block-packed 16x16 blocks with a column pitch of 16 (see tri_inverse.cuh's bp)
__device__ __forceinline__ int bp16(int i, int k) {
  const int I = i >> 4, J = k >> 4;
  return ((I * (I + 1) / 2 + J) << 8) + (i & 15) + ((k & 15) << 4);
}


__device__ __forceinline__ double shfl_idx(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double2 shfl_idx(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <typename T, int NB>
__global__ void __launch_bounds__(256, 1) diag_herm_blocked_kernel(const DiagArgs a) {
  constexpr int NT = 256;
  constexpr int LDS = NB + 1;                                   // smem tile column stride
  constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;
  constexpr int MB = (NB > 32) ? (NB - 32) / 16 : 1;            // 16-row groups below one block
  extern __shared__ __align__(16) unsigned char dsm[];
  T* S = reinterpret_cast<T*>(dsm);                             // S[i + l*LDS] = tile(i, l), lower
  T* Xb = S + NB * LDS;                                         // packed inverse of L11
  T* Tb = Xb + NPB * 256;                                       // scratch for the inverse
  __shared__ double U[NB], dv[NB], pf[NB], pr[NB], lg[NB];
  __shared__ uint8_t keepv[NB];

  const int s = blockIdx.y, jb = a.jb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* A = reinterpret_cast<T*>(a.A) + (int64_t)s * a.strideA + a.j0 + a.tcol * a.ld;
  SampleState* st = reinterpret_cast<SampleState*>(a.state) + s;
  const uint64_t b = a.b0 + (uint64_t)s;

  // ---- stage the lower triangle (zero above the diagonal and beyond jb), uniforms, forced
  for (int l = warp; l < NB; l += NT / 32)
    for (int i = lane; i < NB; i += 32)
      S[i + l * LDS] = (i < jb && l < jb && i >= l) ? A[i + (int64_t)l * a.ld] : zero<T>();
  for (int k = tid; k < jb; k += NT) {
    U[k] = a.map ? 0.5 : uniform_u(a.seed, (uint64_t)(a.j0 + k), b);  // MAP: reading R18
    if (a.forced) keepv[k] = a.forced[(int64_t)s * a.n + a.j0 + k] != 0;
  }
  __syncthreads();

  for (int c0 = 0; c0 < jb; c0 += 32) {
    const int nbj = min(32, jb - c0);
    // ---- (a) the 32 x 32 diagonal block, one warp, lane = row
    if (warp == 0) {
      T r[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) r[q] = (c0 + lane < NB) ? S[(c0 + lane) + (c0 + q) * LDS] : zero<T>();
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        if (p < nbj) {
          const double d = re(shfl_idx(r[p], p));                    // Im of a pivot is 0 (R5)
          const bool keep = a.forced ? (keepv[c0 + p] != 0) : (U[c0 + p] <= d);   // line 437
          const double f = keep ? d : d - 1.0;
          const double rp = recip(f);
          if (lane == 0) {
            dv[c0 + p] = d; pf[c0 + p] = f; pr[c0 + p] = rp;
            if (!a.forced) keepv[c0 + p] = keep ? 1 : 0;
          }
          const T l = (lane > p) ? scal(r[p], rp) : zero<T>();       // line 438 (multiplier)
#pragma unroll
          for (int q = p + 1; q < 32; ++q) r[q] = fms(r[q], l, cj(shfl_idx(r[p], q)));  // line 439
          if (lane > p) r[p] = l;
          else if (lane == p) r[p] = make_real(f, zero<T>());
        }
      }
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q <= lane && c0 + lane < NB) S[(c0 + lane) + (c0 + q) * LDS] = r[q];
    }
    __syncthreads();
    const int s0 = c0 + 32;
    if (s0 >= jb) break;
    // ---- (b) rows below the block: finish their block columns against it
    for (int row = s0 + tid; row < jb; row += NT) {
      T x[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) x[q] = S[row + (c0 + q) * LDS];
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        if (p < nbj) {
          const T l = scal(x[p], pr[c0 + p]);
          const double f = pf[c0 + p];
#pragma unroll
          for (int q = p + 1; q < 32; ++q) x[q] = fms(x[q], l, scal(cj(S[(c0 + q) + (c0 + p) * LDS]), f));
          x[p] = l;
        }
      }
#pragma unroll
      for (int q = 0; q < 32; ++q) S[row + (c0 + q) * LDS] = x[q];
    }
    __syncthreads();
    // ---- (c) the rest of the tile: A(i, l) -= sum_p L(i, c0+p) p_p conj(L(l, c0+p)), i >= l >= s0
    {
      const int tr = tid & 15, tc = tid >> 4;
      T acc[MB][MB];
#pragma unroll
      for (int u = 0; u < MB; ++u)
#pragma unroll
        for (int v = 0; v < MB; ++v) acc[u][v] = zero<T>();
      for (int p = 0; p < nbj; ++p) {
        const double f = pf[c0 + p];
        const T* col = S + (c0 + p) * LDS;
        T li[MB], wl[MB];
#pragma unroll
        for (int u = 0; u < MB; ++u) {
          const int i = s0 + tr + 16 * u;
          li[u] = (i < jb) ? col[i] : zero<T>();
        }
#pragma unroll
        for (int v = 0; v < MB; ++v) {
          const int l = s0 + tc + 16 * v;
          wl[v] = (l < jb) ? scal(cj(col[l]), f) : zero<T>();
        }
#pragma unroll
        for (int u = 0; u < MB; ++u)
#pragma unroll
          for (int v = 0; v <= u; ++v) acc[u][v] = madd(acc[u][v], li[u], wl[v]);
      }
#pragma unroll
      for (int u = 0; u < MB; ++u)
#pragma unroll
        for (int v = 0; v <= u; ++v) {
          const int i = s0 + tr + 16 * u, l = s0 + tc + 16 * v;
          if (i < jb && l < jb && i >= l) S[i + l * LDS] = add(S[i + l * LDS], neg(acc[u][v]));
        }
    }
    __syncthreads();
  }

  // ---- the factor back to the tile (lower): strict lower = L, diagonal = final pivots
  for (int l = warp; l < jb; l += NT / 32)
    for (int i = l + lane; i < jb; i += 32) A[i + (int64_t)l * a.ld] = S[i + l * LDS];
  // ---- decisions, likelihood terms and diagnostics (as diag_kernel)
  for (int k = tid; k < jb; k += NT) {
    a.mask[(int64_t)s * a.n + a.j0 + k] = keepv[k];
    lg[k] = log(fabs(pf[k]));
  }
  __syncthreads();
  if (tid < 32) {
    int nkept = 0, nties = 0, firsttie = -1, noor = 0;
    double minabs = INFINITY;
    for (int k0 = 0; k0 < jb; k0 += 32) {
      const int k = k0 + lane;
      const bool in = k < jb;
      const double d = in ? dv[k] : 0.0;
      const unsigned tb = __ballot_sync(0xffffffffu, in && fabs(U[k] - d) <= a.tie_tol);
      if (tb && firsttie < 0) firsttie = (int)(a.j0 + k0 + __ffs(tb) - 1);
      nties += __popc(tb);
      noor += __popc(__ballot_sync(0xffffffffu, in && (d < -a.range_tol || d > 1.0 + a.range_tol)));
      nkept += __popc(__ballot_sync(0xffffffffu, in && keepv[k]));
      if (in) minabs = fmin(minabs, fabs(pf[k]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) minabs = fmin(minabs, __shfl_xor_sync(0xffffffffu, minabs, o));
    if (lane == 0) {
      double ll = 0.0, maximag = 0.0;
      if (a.j0 > 0) {
        ll = st->loglik;
        minabs = fmin(minabs, st->min_abs_pivot);
        maximag = st->max_abs_imag_pivot;
        nkept += st->n_kept;
        if (st->n_ties > 0) firsttie = st->first_tie;
        nties += st->n_ties;
        noor += st->n_out_of_range;
      }
      for (int k = 0; k < jb; ++k) ll += lg[k];  // in pivot order
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
  if (!a.need_ops) return;
  // ---- stage-2 operator: Bm(j,k) = delta_jk - conj(Linv(j,k)) / D(j), from the factored tile
  const int nblk = (jb + 15) >> 4;
  // X blocks with a pitch of 16 here (this kernel's shared memory is full: no room for bp's padding)
  tri_inverse_lower_g<T, true, NT>([=](int I, int K) { return S + 16 * I + 16 * K * LDS; }, LDS, Xb, Tb, nblk, 16);
  double* dvec = a.dvec + (int64_t)s * a.ldm;
  for (int k = tid; k < jb; k += NT) dvec[k] = pf[k];
  T* Bm = reinterpret_cast<T*>(a.Bm) + (int64_t)s * a.strideM;
  for (int k = warp; k < jb; k += NT / 32)
    for (int j = lane; j < jb; j += 32) {
      T v = zero<T>();
      if (j >= k) {
        v = neg(scal(cj(Xb[bp16(j, k)]), pr[j]));
        if (j == k) v = make_real(re(v) + 1.0, v);
      }
      Bm[j + (int64_t)k * a.ldm] = v;
    }
}

template <typename T, int NB>
static cudaError_t launch_t(const DiagArgs& a, cudaStream_t s) {
  constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;
  const size_t smem = ((size_t)NB * (NB + 1) + (size_t)(NPB + NBLK - 1) * 256) * sizeof(T);
  auto* fn = diag_herm_blocked_kernel<T, NB>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<dim3(1, a.batch), 256, smem, s>>>(a);
  return cudaGetLastError();
}

// Blocked diag kernel for Hermitian double / double2 tiles of 64 and 128, selected with
// DPP_DIAG_BLOCKED=1.  Measured SLOWER than the register-tile kernel of diag.cu (118 vs 88 us per
// 128-tile: the per-row forward substitution of (b) and the per-pivot shuffles of (a) are latency
// chains on few threads), so it is not the default.  Returns cudaErrorNotSupported when off.
cudaError_t launch_diag_herm_blocked(Kind kind, int nb, const DiagArgs& a, cudaStream_t s) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("DPP_DIAG_BLOCKED");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  if (!on) return cudaErrorNotSupported;
  if (kind == HERM_D && nb == 128) return launch_t<double, 128>(a, s);
  if (kind == HERM_D && nb == 64) return launch_t<double, 64>(a, s);
  if (kind == HERM_Z && nb == 64) return launch_t<double2, 64>(a, s);
  return cudaErrorNotSupported;
}

}  // namespace dpp
