// diag.cu -- Stage 1: sequential sample-and-factor of one diagonal tile,
// plus the tile operators that turn stage 2 into tensor-core GEMMs.
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
//    bookkeeping is done in parallel after the loop and summed by one thread IN PIVOT ORDER;
//  * then (if a trailing matrix remains) the inverses of the unit-lower L11 (and, LU, of U11) are
//    formed by a 16x16-blocked triangular inversion in shared memory, and written as the small
//    right/left operators of the stage-2 GEMMs (L21 = A21 L11^-H D1^-1, U12 = L11^-1 A12,
//    L21 = A21 U11^-1) -- Listing 3 lines 584-585 as products with inverses.
// The Hermitian path reads/writes the lower triangle only.
#include <cuda_runtime.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

#include "tri_inverse.cuh"

namespace dpp {


template <typename T, bool HERM, int NB, int NT>
__global__ void __launch_bounds__(NT, 1) diag_kernel(const DiagArgs a) {
  constexpr int TC = 16, TR = NT / TC, RA = NB / TR, CB = NB / TC;
  static_assert(NB % TR == 0, "tile rows must be a multiple of the thread-grid rows");
  constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;  // packed 16x16 blocks
  __shared__ T colbuf[2][2][NB];                    // [buffer][pivot of the pair][row], 0 on/above the pivot
  __shared__ T rowbuf[HERM ? 1 : 2][2][HERM ? 1 : NB];  // LU: [buffer][pivot][column], 0 on/left of the pivot
  __shared__ T pivbuf[2][2];                         // the pair's diagonal entries
  __shared__ T pv[NB], rv[NB];
  __shared__ double U[NB], dv[NB], imv[NB], lg[NB];
  __shared__ uint8_t keepv[NB];
  extern __shared__ __align__(16) unsigned char dsm[];
  T* Lb = reinterpret_cast<T*>(dsm);          // block-packed L11 (unit lower)
  T* Ub = Lb + NPB * BLK_SZ;                   // LU: block-packed U11^T (lower, non-unit)
  T* Xb = Ub + (HERM ? 0 : NPB * BLK_SZ);      // inverse
  T* Tb = Xb + NPB * BLK_SZ;                   // scratch (NBLK - 1 blocks)

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
  for (int k = tid; k < jb; k += NT) {
    // greedy MAP: the decision u <= d with u = 1/2 is "keep iff Re p >= 1/2" (reading R18)
    U[k] = a.map ? 0.5 : uniform_u(a.seed, (uint64_t)(a.j0 + k), b);
    if (a.forced) keepv[k] = a.forced[(int64_t)s * a.n + a.j0 + k] != 0;
  }
  // publish pivot columns kn, kn+1 (strictly below their diagonal, zero elsewhere), their
  // diagonal entries and, LU, rows kn, kn+1 (strictly right of the diagonal).  Zero padding lets
  // the step below run without per-row predicates.  The owning register block is a compile-time
  // index (a runtime index into R would demote the tile to local memory): columns kn, kn+1 (kn even)
  // both lie in register column block IB = kn / TC, rows kn, kn+1 in row block IA = kn / TR, and
  // the caller passes the block it knows kn is in.
  auto publish_col = [&](auto IBC, int kn, int buf) {
    constexpr int IB = decltype(IBC)::value;
    const int l = tc + TC * IB;
    if (l == kn || l == kn + 1) {
#pragma unroll
      for (int ia = 0; ia < RA; ++ia) {
        const int i = tr + TR * ia;
        const T v = R[ia][IB];
        if (i == l) pivbuf[buf][l - kn] = v;
        colbuf[buf][l - kn][i] = (i > l) ? v : zero<T>();
      }
    }
  };
  auto publish_row = [&](auto IAC, int kn, int buf) {
    constexpr int IA = decltype(IAC)::value;
    const int i = tr + TR * IA;
    if (i == kn || i == kn + 1) {
#pragma unroll
      for (int ib = 0; ib < CB; ++ib) {
        const int l = tc + TC * ib;
        rowbuf[HERM ? 0 : buf][i - kn][l] = (l > i) ? R[IA][ib] : zero<T>();
      }
    }
  };
  // kn in [16P + 2, 16P + 16] (the pivot pair after one of phase P), or 0
  auto publish = [&](auto PC, int kn, int buf) {
    constexpr int P = decltype(PC)::value;
    constexpr int IBa = (16 * P) / TC, IBb = (16 * P + 16) / TC;
    if (kn / TC == IBa) publish_col(std::integral_constant<int, IBa>{}, kn, buf);
    else if constexpr (IBb < CB) publish_col(std::integral_constant<int, IBb>{}, kn, buf);
    if (!HERM) {
      constexpr int IAa = (16 * P) / TR, IAb = (16 * P + 16) / TR;
      if (kn / TR == IAa) publish_row(std::integral_constant<int, IAa>{}, kn, buf);
      else if constexpr (IAb < RA) publish_row(std::integral_constant<int, IAb>{}, kn, buf);
    }
  };
  publish(std::integral_constant<int, 0>{}, 0, 0);
  __syncthreads();

  // Two pivots per barrier: every thread redoes the 2x2 micro-step of pivots (k, k+1) from the two
  // published columns, derives both multiplier columns for its rows and both update rows for its
  // columns, and applies the two rank-1 updates (line 439) in pivot order -- the same arithmetic,
  // operation for operation, as two single-pivot steps.  Rows/columns at or above the pivot carry
  // zeros (tile entries beyond jb are zero too), so only row/column k+1 needs a predicate.
  // The pivot loop runs in phases of 16 pivots: in phase P (pivots 16P .. 16P+15) every row and
  // column of the tile below 16P is final, so register blocks holding only such rows (ia < IA0) or
  // columns (ib < IB0) are skipped at compile time -- each phase is its own instantiation of the
  // step, selected by a warp-uniform switch.
  auto step = [&](auto PC, int k) {
    constexpr int P = decltype(PC)::value;
    constexpr int IA0 = (16 * P) / TR, IB0 = (16 * P) / TC;
    const int cur = (k >> 1) & 1, nxt = cur ^ 1;
    const bool two = k + 1 < jb;
    const T* c0 = colbuf[cur][0];
    const T* c1 = colbuf[cur][1];
    // pivot k (line 437)
    T p0 = pivbuf[cur][0];
    if (HERM) p0 = make_real(re(p0), p0);
    const double d0 = re(p0);
    const bool keep0 = a.forced ? (keepv[k] != 0) : (U[k] <= d0);
    if (!keep0) p0 = sub_one(p0);
    const T r0 = recip(p0);
    // pivot k+1 after the rank-1 update of pivot k
    const T a10 = c0[k + 1];                                                     // A(k+1, k)
    const T u01 = HERM ? cj(a10) : rowbuf[HERM ? 0 : cur][0][k + 1];             // conj(w) / U(k,k+1)
    const T p1raw = fms(pivbuf[cur][1], mul(a10, r0), u01);
    T p1 = p1raw;
    if (HERM) p1 = make_real(re(p1), p1);
    const double d1 = re(p1);
    const bool keep1 = two && (a.forced ? (keepv[k + 1] != 0) : (U[k + 1] <= d1));
    if (two && !keep1) p1 = sub_one(p1);
    const T r1 = two ? recip(p1) : zero<T>();
    if (tid == 0) {
      pv[k] = p0; rv[k] = r0; dv[k] = d0; imv[k] = im(pivbuf[cur][0]);
      if (!a.forced) keepv[k] = keep0 ? 1 : 0;
      if (two) {
        pv[k + 1] = p1; rv[k + 1] = r1; dv[k + 1] = d1; imv[k + 1] = im(p1raw);
        if (!a.forced) keepv[k + 1] = keep1 ? 1 : 0;
      }
    }
    // multipliers L(i,k), L(i,k+1) (line 438) for my rows
    T L0[RA], L1[RA];
#pragma unroll
    for (int ia = IA0; ia < RA; ++ia) {
      const int i = tr + TR * ia;
      const T l0 = mul(c0[i], r0);
      L0[ia] = l0;
      L1[ia] = (i == k + 1) ? zero<T>() : mul(fms(c1[i], l0, u01), r1);
    }
    // update rows for my columns: conj(w_l) or U(k, l), U(k+1, l)
    T W0[CB], W1[CB];
#pragma unroll
    for (int ib = IB0; ib < CB; ++ib) {
      const int l = tc + TC * ib;
      if (HERM) {
        const T w0 = c0[l];
        W0[ib] = cj(w0);
        W1[ib] = (l == k + 1) ? zero<T>() : cj(fms(c1[l], mul(w0, r0), u01));
      } else {
        const T w0 = rowbuf[HERM ? 0 : cur][0][l];
        W0[ib] = w0;
        W1[ib] = (l == k + 1) ? zero<T>() : fms(rowbuf[HERM ? 0 : cur][1][l], mul(a10, r0), w0);
      }
    }
    // two rank-1 updates (line 439), branch-free within the live blocks, pivot order
#pragma unroll
    for (int ia = IA0; ia < RA; ++ia)
#pragma unroll
      for (int ib = IB0; ib < CB; ++ib)
        if (!HERM || TC * ib <= TR * ia + TR - 1) {  // skip register blocks entirely above the diagonal
          R[ia][ib] = fms(R[ia][ib], L0[ia], W0[ib]);
          R[ia][ib] = fms(R[ia][ib], L1[ia], W1[ib]);
        }
    if (k + 2 < jb) publish(PC, k + 2, nxt);
    __syncthreads();
  };
  using std::integral_constant;
  for (int k = 0; k < jb; k += 2) {
    switch (k >> 4) {
      case 0: step(integral_constant<int, 0>{}, k); break;
      case 1: if constexpr (NB > 16) step(integral_constant<int, 1>{}, k); break;
      case 2: if constexpr (NB > 32) step(integral_constant<int, 2>{}, k); break;
      case 3: if constexpr (NB > 48) step(integral_constant<int, 3>{}, k); break;
      case 4: if constexpr (NB > 64) step(integral_constant<int, 4>{}, k); break;
      case 5: if constexpr (NB > 80) step(integral_constant<int, 5>{}, k); break;
      case 6: if constexpr (NB > 96) step(integral_constant<int, 6>{}, k); break;
      default: if constexpr (NB > 112) step(integral_constant<int, 7>{}, k); break;
    }
  }

  // ---- finalize the factor: L = (unscaled column) * (1/p), diagonal = final pivot; also stage
  //      the triangular factors block-packed for the inversion (identity beyond jb).  The raw tile
  //      goes to shared memory first (one store per register) and a rolled loop does the rest:
  //      the unrolled per-register form was ~10 KB of straight-line code run once (instruction
  //      fetch stalls dominated it).
  const bool ops = a.need_ops != 0;
#pragma unroll
  for (int ia = 0; ia < RA; ++ia)
#pragma unroll
    for (int ib = 0; ib < CB; ++ib) {
      const int i = tr + TR * ia, l = tc + TC * ib;
      if (i >= l) Lb[bp(i, l)] = R[ia][ib];
      if (!HERM && i <= l) Ub[bp(l, i)] = R[ia][ib];  // U^T(l, i) = U(i, l)
    }
  __syncthreads();
  for (int e = tid; e < NB * NB; e += NT) {
    const int i = e % NB, l = e / NB;  // column-major: consecutive threads, consecutive rows
    const bool in = i < jb && l < jb;
    const T one = make_real(1.0, zero<T>());
    if (i > l) {
      const T v = mul(Lb[bp(i, l)], rv[l < jb ? l : 0]);
      if (in) A[(int64_t)l * a.ld + i] = v;
      Lb[bp(i, l)] = in ? v : zero<T>();
    } else if (i == l) {
      const T v = pv[i < jb ? i : 0];
      if (in) A[(int64_t)l * a.ld + i] = v;
      Lb[bp(i, l)] = one;
      if (!HERM) Ub[bp(l, i)] = in ? v : one;
    } else if (!HERM) {
      const T v = Ub[bp(l, i)];
      if (in) A[(int64_t)l * a.ld + i] = v;
      Ub[bp(l, i)] = in ? v : zero<T>();
    }
  }
  // ---- decisions, likelihood terms and diagnostics: warp 0 reduces the flags with ballots and
  //      shuffles; the log-likelihood terms are summed by one lane IN PIVOT ORDER
  for (int k = tid; k < jb; k += NT) {
    a.mask[(int64_t)s * a.n + a.j0 + k] = keepv[k];
    lg[k] = log((double)absval(pv[k]));
  }
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    int nkept = 0, nties = 0, firsttie = -1, noor = 0;
    double minabs = INFINITY, maximag = 0.0;
    for (int k0 = 0; k0 < jb; k0 += 32) {
      const int k = k0 + lane;
      const bool in = k < jb;
      const double d = in ? dv[k] : 0.0;
      const bool tie = in && fabs(U[k] - d) <= a.tie_tol;
      const unsigned tb = __ballot_sync(0xffffffffu, tie);
      if (tb && firsttie < 0) firsttie = (int)(a.j0 + k0 + __ffs(tb) - 1);
      nties += __popc(tb);
      noor += __popc(__ballot_sync(0xffffffffu, in && (d < -a.range_tol || d > 1.0 + a.range_tol)));
      nkept += __popc(__ballot_sync(0xffffffffu, in && keepv[k]));
      if (in) {
        minabs = fmin(minabs, (double)absval(pv[k]));
        if (!HERM) maximag = fmax(maximag, fabs(imv[k]));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      minabs = fmin(minabs, __shfl_xor_sync(0xffffffffu, minabs, o));
      maximag = fmax(maximag, __shfl_xor_sync(0xffffffffu, maximag, o));
    }
    if (lane == 0) {
      double ll = 0.0;
      if (a.j0 > 0) {
        ll = st->loglik;
        minabs = fmin(minabs, st->min_abs_pivot);
        maximag = fmax(maximag, st->max_abs_imag_pivot);
        nkept += st->n_kept;
        if (st->n_ties > 0) firsttie = st->first_tie;
        nties += st->n_ties;
        noor += st->n_out_of_range;
      }
      for (int k = 0; k < jb; ++k) ll += lg[k];
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
  if (!ops) return;

  // ---- stage-2 operators from the inverses of the tile's triangular factors
  const int nblk = (jb + 15) >> 4;
  T* Bm = reinterpret_cast<T*>(a.Bm) + (int64_t)s * a.strideM;
  tri_inverse_lower<T, true, NT>(Lb, Xb, Tb, nblk);  // Xb = L11^{-1}
  if (HERM) {
    double* dvec = a.dvec + (int64_t)s * a.ldm;  // D1 of sample s (stride nb)
    for (int k = tid; k < jb; k += NT) dvec[k] = re(pv[k]);
    // Bm(j,k) = delta_jk - conj(Linv(j,k)) / D(j)  (j >= k), 0 above  (column k per warp, coalesced)
    for (int k = tid >> 5; k < jb; k += NT / 32)
      for (int j = tid & 31; j < jb; j += 32) {
        T v = zero<T>();
        if (j >= k) {
          v = neg(mul(cj(Xb[bp(j, k)]), make_real(re(rv[j]), zero<T>())));
          if (j == k) v = make_real(re(v) + 1.0, v);
        }
        Bm[j + (int64_t)k * a.ldm] = v;
      }
  } else {
    // Am(i,k) = -Linv(i,k) (i > k), else 0
    T* Am = reinterpret_cast<T*>(a.Am) + (int64_t)s * a.strideM;
    for (int k = tid >> 5; k < jb; k += NT / 32)
      for (int i = tid & 31; i < jb; i += 32) Am[i + (int64_t)k * a.ldm] = (i > k) ? neg(Xb[bp(i, k)]) : zero<T>();
    __syncthreads();
    tri_inverse_lower<T, false, NT>(Ub, Xb, Tb, nblk);  // Xb = (U11^T)^{-1} = (U11^{-1})^T
    // Bm(j,k) = delta_jk - Uinv(k,j) = delta_jk - Xb(j,k)  (j >= k), 0 above
    for (int k = tid >> 5; k < jb; k += NT / 32)
      for (int j = tid & 31; j < jb; j += 32) {
        T v = zero<T>();
        if (j >= k) {
          v = neg(Xb[bp(j, k)]);
          if (j == k) v = make_real(re(v) + 1.0, v);
        }
        Bm[j + (int64_t)k * a.ldm] = v;
      }
  }
}

template <typename T, bool HERM, int NB, int NT>
static cudaError_t launch_diag_nt(const DiagArgs& a, cudaStream_t s) {
  constexpr int NBLK = NB / 16, NPB = NBLK * (NBLK + 1) / 2;
  // the packed factors are also the staging area of the finalize pass: always allocated
  const size_t smem = (size_t)((HERM ? 2 : 3) * NPB + NBLK - 1) * BLK_SZ * sizeof(T);
  auto* fn = diag_kernel<T, HERM, NB, NT>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(1, a.batch);
  fn<<<grid, NT, smem, s>>>(a);
  return cudaGetLastError();
}

// 256 threads per tile CTA (8 x 8 register blocks per thread at nb = 128; a 512-thread grid was
// slower, 107 vs 101 us per tile at the time: the per-pivot chain, not the update FLOPs, bounds
// this kernel).
template <typename T, bool HERM, int NB>
static cudaError_t launch_diag_t(const DiagArgs& a, cudaStream_t s) {
  return launch_diag_nt<T, HERM, NB, 256>(a, s);
}

cudaError_t launch_diag_rl(int nb, const DiagArgs& a, cudaStream_t s, bool fp32);

cudaError_t launch_diag(Kind kind, int nb, const DiagArgs& a, cudaStream_t s) {
  // real symmetric 64- and 128-tiles: the blocked kernel of diag_rl.cu (warp sub-panels + DMMA)
  if (kind == HERM_D && (nb == 64 || nb == 128)) return launch_diag_rl(nb, a, s, false);
  if (kind == HERM_S && (nb == 64 || nb == 128)) return launch_diag_rl(nb, a, s, true);
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
    case HERM_S:
      if (nb <= 32) return launch_diag_t<float, true, 32>(a, s);
      if (nb <= 64) return launch_diag_t<float, true, 64>(a, s);
      return launch_diag_t<float, true, 128>(a, s);
    case LU_C:
      if (nb <= 32) return launch_diag_t<float2, false, 32>(a, s);
      return launch_diag_t<float2, false, 64>(a, s);
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
