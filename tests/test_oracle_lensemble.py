"""Pins of the oracle's L-ensemble -> marginal kernel conversion, K = I - (L + I)^{-1}
(the "natural extension ... for converting a Hermitian L-ensemble kernel into a
marginal kernel").  The oracle is the plain definition (library inverse); these
checks pin it independently:
  * spectral map: L = V diag(lam) V^T  =>  K = V diag(lam / (1 + lam)) V^T;
  * special cases: L = 0 -> K = 0; L = c I -> K = c / (1 + c) I; ln det(L + I);
  * the law: P(Y = S) = det(L_S) / det(L + I) equals |det(K - 1_{S^c})| for every S (brute force),
    and the CPU sampler on the converted K reproduces it (frequencies)."""
import itertools

import numpy as np
import pytest

from tests.stats_util import check_subset_frequencies, masks_to_index


def _lens(n, seed, scale=10.0, complex_=False):
    rng = np.random.default_rng(seed)
    lam = rng.uniform(0, scale, n)
    G = (rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if complex_ else 0))
    V, _ = np.linalg.qr(G)
    return (V * lam) @ V.conj().T, V, lam


def test_spectral_map_and_special_cases(oracle_mod):
    L, V, lam = _lens(40, 1)
    K, ld = oracle_mod.lensemble_to_marginal(L)
    want = (V * (lam / (1 + lam))) @ V.T
    assert np.max(np.abs(K - want)) <= 1e-12
    assert abs(ld - np.sum(np.log1p(lam))) <= 1e-10
    K0, ld0 = oracle_mod.lensemble_to_marginal(np.zeros((5, 5)))
    assert np.max(np.abs(K0)) == 0.0 and ld0 == 0.0
    Kc, _ = oracle_mod.lensemble_to_marginal(3.0 * np.eye(6))
    assert np.max(np.abs(Kc - 0.75 * np.eye(6))) <= 1e-15


def test_law_matches_lensemble(oracle_mod):
    n = 6
    L, _, _ = _lens(n, 3, scale=3.0)
    K, ld = oracle_mod.lensemble_to_marginal(L)
    Z = np.exp(ld)
    p = np.zeros(1 << n)
    for s in range(1 << n):
        S = [i for i in range(n) if (s >> i) & 1]
        pl = np.linalg.det(L[np.ix_(S, S)]) / Z if S else 1.0 / Z
        comp = np.array([0.0 if (s >> i) & 1 else 1.0 for i in range(n)])
        assert abs(pl - abs(np.linalg.det(K - np.diag(comp)))) <= 1e-12
        p[s] = pl
    masks, _ = oracle_mod.sample_many(0, K, 4, 0, 200_000)
    counts = np.bincount(masks_to_index(masks), minlength=1 << n).astype(float)
    ok, rep = check_subset_frequencies(p, counts)
    assert ok, rep
