/*
 * dpp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the factorization-based DPP
 * sampler of arXiv 1905.00165 ("High-performance sampling of generic
 * Determinantal Point Processes").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_1905_00165_b200/) never includes, links or calls it, and
 * this file shares no code, header, table or constant generator with it.
 *
 * Everything here follows the paper's Listing 1 ("Unblocked,
 * right-looking, non-Hermitian DPP sampling") step by step, unblocked, in fp64:
 *
 *     sample := []; A := K
 *     for j in range(n):
 *       sample.append(j) if Bernoulli(A_j) else A_j -= 1      (line 437)
 *       A_[j+1:n], j /= A_j                                    (line 438)
 *       A_[j+1:n] -= A_[j+1:n], j  A_j, [j+1:n]                (line 439)
 *     return sample, A
 *
 * with the Hermitian (LDL^H) specialisation the theorem and the caption allow
 * ("the work can be roughly halved by exploiting symmetry";
 * PAPER.md:433-434 "Symmetry can be exploited in the outer products").
 * The log-likelihood is the sum of ln|final pivot| (PAPER.md:395-396,
 * PAPER.md:419-422).
 *
 * Readings of points the paper leaves open (all listed in DESIGN.md §Readings):
 *   R1  Bernoulli(A_j): draw u_j in (0,1) and keep iff u_j <= Re A_j.
 *   R2  u_j = Philox4x32-10(counter = (lo32 j, hi32 j, lo32 b, hi32 b),
 *       key = (lo32 seed, hi32 seed)); x = (r.y << 32) | r.x;
 *       u = (2*(x >> 12) + 1) * 2^-53   (exact in fp64, never 0 or 1).
 *       One draw per pivot whatever the pivot value.
 *   R3  Pivots are NOT clamped; out-of-range pivots are counted.
 *   R4  Non-Hermitian complex pivot p: decide on Re p, subtract 1 from p,
 *       likelihood uses |p| (complex modulus), max |Im p| is reported.
 *   R5  Hermitian kernels: only the lower triangle is read and written; the
 *       imaginary part of a diagonal entry is treated as 0.
 *   R6  Layout: column-major with leading dimension ld; complex numbers are
 *       interleaved (re, im) pairs of doubles.
 *   R8  Ties: a pivot with |u - d| <= tie_tol is counted and the first such
 *       pivot index recorded.  If `forced` is non-NULL the decision for pivot j
 *       is forced[j] != 0 instead of the draw (replay, SPEC log_likelihood_of).
 *   R18 Greedy MAP ("replacing the Bernoulli samples ... with
 *       the maximum-likelihood result for each index inclusion"): the more
 *       probable branch, keep iff Re p >= 1/2 (include at exactly 1/2); a tie
 *       is |Re p - 1/2| <= tie_tol.  No uniform is drawn.  oracle_map_* below
 *       are the same loops with this decision.
 *
 * Build: gcc -O2 -ffp-contract=off -std=c11 -shared -fPIC (single thread, no BLAS).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n_kept;          /* |Y| */
  int32_t n_ties;          /* pivots with |u - d| <= tie_tol */
  int32_t first_tie;       /* first such pivot index, -1 if none */
  int32_t n_out_of_range;  /* pivots with d < -range_tol or d > 1 + range_tol */
  double min_abs_pivot;    /* min_j |final pivot_j| (+inf for n = 0) */
  double max_abs_imag_pivot; /* LU only: max_j |Im p_j| before modification */
} oracle_info_t;

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11), written from the published round    */
/* function: 10 rounds, multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key bumps  */
/* 0x9E3779B9 / 0xBB67AE85.                                                  */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Reading R2: the uniform for pivot j of sample b under `seed`. */
double oracle_uniform(uint64_t seed, uint64_t j, uint64_t b) {
  uint32_t ctr[4] = {(uint32_t)j, (uint32_t)(j >> 32), (uint32_t)b, (uint32_t)(b >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  oracle_philox4x32_10(ctr, key, r);
  uint64_t x = ((uint64_t)r[1] << 32) | (uint64_t)r[0];
  uint64_t m = x >> 12;                          /* 52 random bits */
  return (double)(2 * m + 1) * 0x1.0p-53;        /* odd multiple of 2^-53 */
}

static void info_init(oracle_info_t* info) {
  info->n_kept = 0;
  info->n_ties = 0;
  info->first_tie = -1;
  info->n_out_of_range = 0;
  info->min_abs_pivot = INFINITY;
  info->max_abs_imag_pivot = 0.0;
}

/* Decision at pivot j with real pivot value d (Listing 1; R1, R3, R8);
   map != 0: the greedy maximum-likelihood decision of R18 instead of the draw. */
static int decide(double d, int64_t j, uint64_t seed, uint64_t b, const uint8_t* forced,
                  double tie_tol, double range_tol, oracle_info_t* info, int map) {
  double u = map ? 0.5 : oracle_uniform(seed, (uint64_t)j, b);
  if (fabs(u - d) <= tie_tol) {
    if (info->n_ties == 0) info->first_tie = (int32_t)j;
    info->n_ties++;
  }
  if (d < -range_tol || d > 1.0 + range_tol) info->n_out_of_range++;
  if (forced) return forced[j] != 0;
  return map ? d >= 0.5 : u <= d;
}

/*
 * Real symmetric kernel, LDL^T specialisation of Listing 1 (lower triangle).
 * On return A's strict lower triangle holds L (unit diagonal implicit), its
 * diagonal holds D, and L D L^T = K - 1_{Y^c}.  The upper triangle is untouched.
 */
static int run_herm_d(int map, int64_t n, double* A, int64_t ld, uint64_t seed, uint64_t b,
                         const uint8_t* forced, double tie_tol, double range_tol,
                         uint8_t* mask, double* loglik, oracle_info_t* info) {
  if (n < 0 || ld < (n > 1 ? n : 1)) return -1;
  oracle_info_t inf;
  info_init(&inf);
  double ll = 0.0;
  double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  if (!w) return -2;
#define A_(i, l) A[(size_t)(l) * (size_t)ld + (size_t)(i)]
  for (int64_t j = 0; j < n; ++j) {
    double d = A_(j, j);
    int keep = decide(d, j, seed, b, forced, tie_tol, range_tol, &inf, map);
    if (!keep) d -= 1.0;                      /* line 437: A_j -= 1 */
    A_(j, j) = d;
    mask[j] = (uint8_t)keep;
    inf.n_kept += keep;
    ll += log(fabs(d));
    if (fabs(d) < inf.min_abs_pivot) inf.min_abs_pivot = fabs(d);
    for (int64_t i = j + 1; i < n; ++i) {     /* line 438: column / pivot */
      w[i] = A_(i, j);
      A_(i, j) = w[i] / d;
    }
    for (int64_t l = j + 1; l < n; ++l)       /* line 439: rank-1, lower only */
      for (int64_t i = l; i < n; ++i)
        A_(i, l) -= A_(i, j) * w[l];
  }
#undef A_
  free(w);
  *loglik = ll;
  if (info) *info = inf;
  return 0;
}

/* Complex Hermitian kernel, LDL^H specialisation (lower triangle, R5). */
static int run_herm_z(int map, int64_t n, double* Araw, int64_t ld, uint64_t seed, uint64_t b,
                         const uint8_t* forced, double tie_tol, double range_tol,
                         uint8_t* mask, double* loglik, oracle_info_t* info) {
  if (n < 0 || ld < (n > 1 ? n : 1)) return -1;
  double complex* A = (double complex*)Araw;
  oracle_info_t inf;
  info_init(&inf);
  double ll = 0.0;
  double complex* w = (double complex*)malloc(sizeof(double complex) * (size_t)(n > 0 ? n : 1));
  if (!w) return -2;
#define A_(i, l) A[(size_t)(l) * (size_t)ld + (size_t)(i)]
  for (int64_t j = 0; j < n; ++j) {
    double d = creal(A_(j, j));               /* R5: Im of a diagonal entry is 0 */
    int keep = decide(d, j, seed, b, forced, tie_tol, range_tol, &inf, map);
    if (!keep) d -= 1.0;
    A_(j, j) = d;                             /* stored with zero imaginary part */
    mask[j] = (uint8_t)keep;
    inf.n_kept += keep;
    ll += log(fabs(d));
    if (fabs(d) < inf.min_abs_pivot) inf.min_abs_pivot = fabs(d);
    for (int64_t i = j + 1; i < n; ++i) {
      w[i] = A_(i, j);
      A_(i, j) = w[i] / d;
    }
    for (int64_t l = j + 1; l < n; ++l)       /* A(i,l) -= L(i,j) conj(w(l)), i >= l */
      for (int64_t i = l; i < n; ++i)
        A_(i, l) -= A_(i, j) * conj(w[l]);
  }
#undef A_
  free(w);
  *loglik = ll;
  if (info) *info = inf;
  return 0;
}

/* Complex non-Hermitian kernel: Listing 1 literally (unpivoted LU, R4). */
static int run_lu_z(int map, int64_t n, double* Araw, int64_t ld, uint64_t seed, uint64_t b,
                       const uint8_t* forced, double tie_tol, double range_tol,
                       uint8_t* mask, double* loglik, oracle_info_t* info) {
  if (n < 0 || ld < (n > 1 ? n : 1)) return -1;
  double complex* A = (double complex*)Araw;
  oracle_info_t inf;
  info_init(&inf);
  double ll = 0.0;
#define A_(i, l) A[(size_t)(l) * (size_t)ld + (size_t)(i)]
  for (int64_t j = 0; j < n; ++j) {
    double complex p = A_(j, j);
    if (fabs(cimag(p)) > inf.max_abs_imag_pivot) inf.max_abs_imag_pivot = fabs(cimag(p));
    int keep = decide(creal(p), j, seed, b, forced, tie_tol, range_tol, &inf, map);
    if (!keep) p -= 1.0;                      /* line 437 */
    A_(j, j) = p;
    mask[j] = (uint8_t)keep;
    inf.n_kept += keep;
    ll += log(cabs(p));
    if (cabs(p) < inf.min_abs_pivot) inf.min_abs_pivot = cabs(p);
    for (int64_t i = j + 1; i < n; ++i)       /* line 438 */
      A_(i, j) = A_(i, j) / p;
    for (int64_t l = j + 1; l < n; ++l)       /* line 439: full rank-1 update */
      for (int64_t i = j + 1; i < n; ++i)
        A_(i, l) -= A_(i, j) * A_(j, l);
  }
#undef A_
  *loglik = ll;
  if (info) *info = inf;
  return 0;
}

/* Exported entry points: sampling (Listing 1) and greedy MAP (R18). */
#define ORACLE_EXPORT(name)                                                                     \
  int oracle_sample_##name(int64_t n, double* A, int64_t ld, uint64_t seed, uint64_t b,         \
                           const uint8_t* forced, double tie_tol, double range_tol,             \
                           uint8_t* mask, double* loglik, oracle_info_t* info) {                \
    return run_##name(0, n, A, ld, seed, b, forced, tie_tol, range_tol, mask, loglik, info);    \
  }                                                                                             \
  int oracle_map_##name(int64_t n, double* A, int64_t ld, const uint8_t* forced,               \
                        double tie_tol, double range_tol, uint8_t* mask, double* loglik,        \
                        oracle_info_t* info) {                                                  \
    return run_##name(1, n, A, ld, 0, 0, forced, tie_tol, range_tol, mask, loglik, info);       \
  }
ORACLE_EXPORT(herm_d)
ORACLE_EXPORT(herm_z)
ORACLE_EXPORT(lu_z)


/* ------------------------------------------------------------------------ */
/* Single precision (the paper's single-precision runs, */
/* PAPER.md:1164-1169).  The same Listing 1 loops with every matrix entry,   */
/* pivot, multiplier and update in fp32 (float / float complex); the         */
/* decision compares the fp64 uniform with the fp32 pivot promoted to        */
/* double, and the log-likelihood is accumulated in fp64 from the fp32       */
/* pivots (reading R19).                                                     */
/* ------------------------------------------------------------------------ */
static int run_herm_s(int map, int64_t n, float* A, int64_t ld, uint64_t seed, uint64_t b,
                      const uint8_t* forced, double tie_tol, double range_tol,
                      uint8_t* mask, double* loglik, oracle_info_t* info) {
  if (n < 0 || ld < (n > 1 ? n : 1)) return -1;
  oracle_info_t inf;
  info_init(&inf);
  double ll = 0.0;
  float* w = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  if (!w) return -2;
#define A_(i, l) A[(size_t)(l) * (size_t)ld + (size_t)(i)]
  for (int64_t j = 0; j < n; ++j) {
    float d = A_(j, j);
    int keep = decide((double)d, j, seed, b, forced, tie_tol, range_tol, &inf, map);
    if (!keep) d -= 1.0f;                     /* line 437 */
    A_(j, j) = d;
    mask[j] = (uint8_t)keep;
    inf.n_kept += keep;
    ll += log(fabs((double)d));
    if (fabs((double)d) < inf.min_abs_pivot) inf.min_abs_pivot = fabs((double)d);
    for (int64_t i = j + 1; i < n; ++i) {     /* line 438 */
      w[i] = A_(i, j);
      A_(i, j) = w[i] / d;
    }
    for (int64_t l = j + 1; l < n; ++l)       /* line 439: rank-1, lower only */
      for (int64_t i = l; i < n; ++i)
        A_(i, l) -= A_(i, j) * w[l];
  }
#undef A_
  free(w);
  *loglik = ll;
  if (info) *info = inf;
  return 0;
}

static int run_lu_c(int map, int64_t n, float* Araw, int64_t ld, uint64_t seed, uint64_t b,
                    const uint8_t* forced, double tie_tol, double range_tol,
                    uint8_t* mask, double* loglik, oracle_info_t* info) {
  if (n < 0 || ld < (n > 1 ? n : 1)) return -1;
  float complex* A = (float complex*)Araw;
  oracle_info_t inf;
  info_init(&inf);
  double ll = 0.0;
#define A_(i, l) A[(size_t)(l) * (size_t)ld + (size_t)(i)]
  for (int64_t j = 0; j < n; ++j) {
    float complex p = A_(j, j);
    if (fabs((double)cimagf(p)) > inf.max_abs_imag_pivot) inf.max_abs_imag_pivot = fabs((double)cimagf(p));
    int keep = decide((double)crealf(p), j, seed, b, forced, tie_tol, range_tol, &inf, map);
    if (!keep) p -= 1.0f;                     /* line 437 */
    A_(j, j) = p;
    mask[j] = (uint8_t)keep;
    inf.n_kept += keep;
    double ap = hypot((double)crealf(p), (double)cimagf(p));
    ll += log(ap);
    if (ap < inf.min_abs_pivot) inf.min_abs_pivot = ap;
    for (int64_t i = j + 1; i < n; ++i)       /* line 438 */
      A_(i, j) = A_(i, j) / p;
    for (int64_t l = j + 1; l < n; ++l)       /* line 439 */
      for (int64_t i = j + 1; i < n; ++i)
        A_(i, l) -= A_(i, j) * A_(j, l);
  }
#undef A_
  *loglik = ll;
  if (info) *info = inf;
  return 0;
}

int oracle_sample_herm_s(int64_t n, float* A, int64_t ld, uint64_t seed, uint64_t b, const uint8_t* forced,
                         double tie_tol, double range_tol, uint8_t* mask, double* loglik, oracle_info_t* info) {
  return run_herm_s(0, n, A, ld, seed, b, forced, tie_tol, range_tol, mask, loglik, info);
}
int oracle_sample_lu_c(int64_t n, float* A, int64_t ld, uint64_t seed, uint64_t b, const uint8_t* forced,
                       double tie_tol, double range_tol, uint8_t* mask, double* loglik, oracle_info_t* info) {
  return run_lu_c(0, n, A, ld, seed, b, forced, tie_tol, range_tol, mask, loglik, info);
}


/* ------------------------------------------------------------------------ */
/* Elementary (projection) DPP sampler: Listing 2,        */
/* Theorem "Factorization-based elementary DPP sampling": */
/* k steps of a left-looking, diagonally pivoted Cholesky factorization of a */
/* rank-k orthogonal projection K, each pivot drawn from the current         */
/* diagonal with probability d_t / (k - j).                                  */
/*                                                                            */
/* Reading R20 (the listing permutes A and d after every draw; the law of    */
/* the draw does not depend on the order of the candidates): no physical    */
/* swap -- the candidates are the items not yet chosen, in ORIGINAL index    */
/* order; with u_j the Philox uniform of pivot j (R2) and S the sum of their */
/* d (= k - j in exact arithmetic), t is the first candidate whose running   */
/* sum of d exceeds u_j S (if rounding leaves none, the last candidate with  */
/* d > 0).  A draw is a tie when u_j S lies within tie_tol * S of the        */
/* running sum just before or at t.  L is stored by original row: column j   */
/* of the n x k array Lf holds the j-th factor column, L(t_j, j) = sqrt(d).  */
/* The likelihood is ln prod_j A_j^2 = sum_j ln d_{t_j}.  */
/* ------------------------------------------------------------------------ */
int oracle_elementary_herm_d(int64_t n, int64_t k, const double* K, int64_t ld, uint64_t seed, uint64_t b,
                             double tie_tol, int64_t* order, double* Lf, double* loglik, int32_t* n_ties,
                             int32_t* first_tie) {
  if (n < 0 || k < 0 || k > n || ld < (n > 1 ? n : 1)) return -1;
  double* d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  uint8_t* chosen = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!d || !chosen) { free(d); free(chosen); return -2; }
#define K_(i, l) K[(size_t)(l) * (size_t)ld + (size_t)(i)]
#define L_(i, j) Lf[(size_t)(j) * (size_t)n + (size_t)(i)]
  for (int64_t i = 0; i < n; ++i) d[i] = K_(i, i);            /* d := diag(K) */
  for (size_t e = 0; e < (size_t)n * (size_t)k; ++e) Lf[e] = 0.0;
  double ll = 0.0;
  int32_t ties = 0, ftie = -1;
  for (int64_t j = 0; j < k; ++j) {
    /* draw t with probability d_t / (k - j) among the candidates (R20) */
    double S = 0.0;
    for (int64_t i = 0; i < n; ++i)
      if (!chosen[i]) S += d[i];
    const double target = oracle_uniform(seed, (uint64_t)j, b) * S;
    int64_t t = -1, last = -1;
    double run = 0.0, before = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (chosen[i]) continue;
      if (d[i] > 0.0) last = i;
      before = run;
      run += d[i];
      if (run > target) { t = i; break; }
    }
    if (t < 0) { t = last; before = run; }
    if (fabs(target - before) <= tie_tol * S || fabs(run - target) <= tie_tol * S) {
      if (ties == 0) ftie = (int32_t)j;
      ties++;
    }
    order[j] = t;
    chosen[t] = 1;
    const double Aj = sqrt(d[t]);                              /* A_j := sqrt(d_j) */
    ll += log(d[t]);                                           /* ln A_j^2 */
    L_(t, j) = Aj;
    if (j == k - 1) break;
    /* new column: A_[j+1:n], j -= A_[j+1:n], [0:j] A_j, [0:j]^H ; then / A_j; d -= |.|^2 */
    for (int64_t i = 0; i < n; ++i) {
      if (chosen[i]) continue;
      double c = K_(i, t);
      for (int64_t m = 0; m < j; ++m) c -= L_(i, m) * L_(t, m);
      c /= Aj;
      L_(i, j) = c;
      d[i] -= c * c;
    }
  }
#undef K_
#undef L_
  free(d);
  free(chosen);
  *loglik = ll;
  if (n_ties) *n_ties = ties;
  if (first_tie) *first_tie = ftie;
  return 0;
}

/*
 * Many independent samples b = b0 .. b0+batch-1 of ONE kernel K (read-only),
 * each on a fresh copy of K.  A plain loop over the single-sample routines
 * above (kind 0 = herm_d, 1 = herm_z, 2 = lu_z); used by the brute-force
 * statistics tests to avoid per-call Python overhead.
 */
int oracle_sample_many(int kind, int64_t n, const double* K, int64_t ld, uint64_t seed,
                       uint64_t b0, int64_t batch, uint8_t* masks, double* logliks) {
  /* element bytes: herm_d 8, herm_z 16, lu_z 16, herm_s 4, lu_c 8 */
  static const size_t ebytes[5] = {8, 16, 16, 4, 8};
  if (kind < 0 || kind > 4) return -1;
  size_t bytes = (size_t)ld * (size_t)(n > 0 ? n : 1) * ebytes[kind];
  double* work = (double*)malloc(bytes);
  if (!work) return -2;
  for (int64_t s = 0; s < batch; ++s) {
    memcpy(work, K, bytes);
    int rc;
    if (kind == 3)
      rc = oracle_sample_herm_s(n, (float*)work, ld, seed, b0 + (uint64_t)s, NULL, 1e-9, 1e-8,
                                masks + (size_t)s * (size_t)n, logliks + s, NULL);
    else if (kind == 4)
      rc = oracle_sample_lu_c(n, (float*)work, ld, seed, b0 + (uint64_t)s, NULL, 1e-9, 1e-8,
                              masks + (size_t)s * (size_t)n, logliks + s, NULL);
    else if (kind == 0)
      rc = oracle_sample_herm_d(n, work, ld, seed, b0 + (uint64_t)s, NULL, 1e-9, 1e-8,
                                masks + (size_t)s * (size_t)n, logliks + s, NULL);
    else if (kind == 1)
      rc = oracle_sample_herm_z(n, work, ld, seed, b0 + (uint64_t)s, NULL, 1e-9, 1e-8,
                                masks + (size_t)s * (size_t)n, logliks + s, NULL);
    else
      rc = oracle_sample_lu_z(n, work, ld, seed, b0 + (uint64_t)s, NULL, 1e-9, 1e-8,
                              masks + (size_t)s * (size_t)n, logliks + s, NULL);
    if (rc) { free(work); return rc; }
  }
  free(work);
  return 0;
}
