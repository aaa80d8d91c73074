"""Pins of the oracle's elementary (projection) DPP sampler -- Listing 2, Theorem
"Factorization-based elementary DPP sampling", reading R20.

Independent of the oracle's loop: cardinality k (the theorem), loglik = ln det(K_Y) (numpy slogdet,
the proof's P[Y = Y] = det(K_Y) = prod A_j^2), the returned factor is the Cholesky factor of K_Y,
brute-force subset frequencies vs det(K_S), inclusion frequencies vs diag(K), and UST spanning
trees with likelihood -ln tau(G).
"""
import itertools

import numpy as np
import pytest

import workloads as W
from tests.stats_util import check_marginals, check_subset_frequencies


@pytest.mark.parametrize("n,k,seed", [(40, 1, 0), (60, 12, 1), (120, 45, 2), (30, 30, 3)])
def test_elementary_cardinality_loglik_and_factor(oracle_mod, n, k, seed):
    K = W.projection_kernel(n, k, seed=seed)
    for b in range(4):
        r = oracle_mod.elementary_herm_d(K, k, 9, b)
        assert len(set(r.order.tolist())) == k
        KY = K[np.ix_(r.order, r.order)]
        sign, ld = np.linalg.slogdet(KY)
        assert sign > 0 and abs(r.loglik - ld) <= 1e-10 * max(1.0, abs(ld))
        LY = r.L[r.order, :]
        assert np.allclose(np.triu(LY, 1), 0.0)
        assert np.max(np.abs(LY @ LY.T - KY)) <= 1e-12 * k


def test_elementary_brute_force_law(oracle_mod):
    """P(Y = S) = det(K_S) for |S| = k; also = |det(K - 1_{S^c})|."""
    n, k, draws = 7, 3, 200_000
    K = W.projection_kernel(n, k, seed=11)
    subsets = list(itertools.combinations(range(n), k))
    p = np.array([np.linalg.det(K[np.ix_(S, S)]) for S in subsets])
    for S, ps in zip(subsets, p):
        comp = np.ones(n)
        comp[list(S)] = 0
        assert abs(ps - abs(np.linalg.det(K - np.diag(comp)))) <= 1e-12
    assert abs(p.sum() - 1.0) <= 1e-12
    index = {S: i for i, S in enumerate(subsets)}
    counts = np.zeros(len(subsets))
    for b in range(draws):
        r = oracle_mod.elementary_herm_d(K, k, 5, b)
        counts[index[tuple(sorted(r.order.tolist()))]] += 1
    ok, rep = check_subset_frequencies(p, counts)
    assert ok, rep


def test_elementary_marginals(oracle_mod):
    n, k = 24, 10
    K = W.projection_kernel(n, k, seed=4)
    masks = np.array([oracle_mod.elementary_herm_d(K, k, 2, b).mask for b in range(40_000)])
    ok, rep = check_marginals(K, masks)
    assert ok, rep


def test_elementary_ust(oracle_mod):
    K = W.ust_kernel(10, 10)
    edges = W.grid_edges(10, 10)
    want = -W.log_num_spanning_trees_grid(10, 10)
    for b in range(3):
        r = oracle_mod.elementary_herm_d(K, 99, 0, b)
        assert W.is_spanning_tree(100, edges, r.mask)
        assert abs(r.loglik - want) <= 1e-9 * abs(want)
