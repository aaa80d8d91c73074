"""Statistical helpers for brute-force checks (test infrastructure).

Implements DESIGN.md reading #12 (north_star "within 3 sigma" for 2^n
simultaneous subset frequencies):
  (i)   #subsets outside 3 sigma <= the 99.9% quantile of Binomial(2^n, 0.0027),
  (ii)  no subset beyond the two-sided Bonferroni z for alpha = 1e-3,
  (iii) Pearson chi^2 with bins merged below 5 expected counts passes at 1e-3,
  (iv)  every p_S = 0 subset has zero count.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy import stats


def subset_probabilities(K: np.ndarray) -> np.ndarray:
    """P(Y = S) = |det(K - 1_{S^c})| for every S (bit i of the index <-> item i).

    PAPER.md:452-455 (proof of Prop. 1): det(K - 1_{Y^C}) = prod_{j in Y} p_j
    prod_{j in Y^C} (p_j - 1); its absolute value is the sample's probability.
    Uses numpy's LAPACK determinant (a library routine), not the sampler."""
    n = K.shape[0]
    out = np.zeros(1 << n)
    for s in range(1 << n):
        comp = np.array([0.0 if (s >> i) & 1 else 1.0 for i in range(n)])
        out[s] = abs(np.linalg.det(K - np.diag(comp)))
    return out


def masks_to_index(masks: np.ndarray) -> np.ndarray:
    n = masks.shape[1]
    w = (1 << np.arange(n)).astype(np.int64)
    return masks.astype(np.int64) @ w


def check_subset_frequencies(p: np.ndarray, counts: np.ndarray, alpha: float = 1e-3):
    """Returns (ok, report) under reading #12."""
    N = counts.sum()
    m = len(p)
    p = p / p.sum()
    expected = N * p
    sd = np.sqrt(np.maximum(N * p * (1 - p), 1e-300))
    z = np.where(p > 0, (counts - expected) / sd, 0.0)
    outside3 = int(np.sum((p > 0) & (np.abs(z) > 3)))
    q = int(stats.binom.ppf(0.999, m, 0.0027))
    zb = stats.norm.isf(alpha / (2 * m))
    zero_bad = int(np.sum((p <= 1e-14) & (counts > 0)))
    # Pearson chi^2 with merging of small bins
    order = np.argsort(expected)
    e_s, c_s = expected[order], counts[order]
    keep = e_s > 1e-12
    e_s, c_s = e_s[keep], c_s[keep]
    bins_e, bins_c, acc_e, acc_c = [], [], 0.0, 0.0
    for e, c in zip(e_s, c_s):
        acc_e += e
        acc_c += c
        if acc_e >= 5:
            bins_e.append(acc_e)
            bins_c.append(acc_c)
            acc_e, acc_c = 0.0, 0.0
    if acc_e > 0 and bins_e:
        bins_e[-1] += acc_e
        bins_c[-1] += acc_c
    bins_e, bins_c = np.array(bins_e), np.array(bins_c)
    chi2 = float(np.sum((bins_c - bins_e) ** 2 / bins_e))
    dof = max(len(bins_e) - 1, 1)
    pval = float(stats.chi2.sf(chi2, dof))
    ok = (outside3 <= q) and (np.max(np.abs(z)) <= zb) and zero_bad == 0 and pval >= alpha
    report = dict(outside3=outside3, quantile=q, max_z=float(np.max(np.abs(z))), bonferroni_z=zb,
                  zero_bad=zero_bad, chi2=chi2, dof=dof, pval=pval)
    return ok, report


def check_marginals(K: np.ndarray, masks: np.ndarray, alpha: float = 1e-3):
    """Inclusion frequencies vs diag(K) (Definition 1 with |Y| = 1)."""
    N, n = masks.shape
    p = np.real(np.diagonal(K))
    f = masks.mean(axis=0)
    sd = np.sqrt(np.maximum(p * (1 - p) / N, 1e-300))
    z = np.where((p > 1e-12) & (p < 1 - 1e-12), (f - p) / sd, 0.0)
    zb = stats.norm.isf(alpha / (2 * n))
    det_ok = bool(np.all(f[p <= 1e-12] == 0) and np.all(f[p >= 1 - 1e-12] == 1))
    return (np.max(np.abs(z)) <= zb) and det_ok, dict(max_z=float(np.max(np.abs(z))), bonferroni_z=zb)


def all_subsets(n):
    return itertools.product([0, 1], repeat=n)
