"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Each test names the passage it pins.  None of them re-types the oracle's loop:
they check closed forms, library determinants/factorizations, brute-force
subset probabilities and combinatorial invariants.
"""
import json
import os

import numpy as np
import pytest

import workloads as W
from tests.stats_util import (check_marginals, check_subset_frequencies, masks_to_index,
                              subset_probabilities)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))
KINDS = ("herm_d", "herm_z", "lu_z")


def _run(o, kind, K, seed=0, b=0, forced=None):
    return {"herm_d": o.sample_herm_d, "herm_z": o.sample_herm_z, "lu_z": o.sample_lu_z}[kind](
        K, seed, b, forced)


def _cast(kind, K):
    return np.asarray(K, dtype=np.float64 if kind == "herm_d" else np.complex128)


# ----------------------------------------------------------------- decision rule
@pytest.mark.parametrize("kind", KINDS)
def test_diagonal_kernel_closed_form(oracle_mod, kind):
    """K = diag(p): independent Bernoullis.  Decision u_k <= p_k (reading R1),
    loglik = sum ln(p or 1-p), factor diagonal = p - 1_{Y^c}."""
    rng = np.random.default_rng(5)
    n = 40
    p = rng.uniform(0, 1, n)
    p[:3] = [0.0, 1.0, 0.5]
    for b in range(5):
        r = _run(oracle_mod, kind, _cast(kind, np.diag(p)), seed=11, b=b)
        u = np.array([oracle_mod.uniform(11, j, b) for j in range(n)])
        keep = u <= p
        assert np.array_equal(r.mask.astype(bool), keep)
        want = np.sum(np.log(np.where(keep, p, 1 - p)))
        assert r.loglik == pytest.approx(want, rel=1e-14, abs=1e-14)
        assert np.allclose(np.real(np.diagonal(r.factor)), p - (~keep), atol=0, rtol=0)
        assert r.mask[0] == 0 and r.mask[1] == 1


@pytest.mark.parametrize("kind", KINDS)
def test_zero_and_identity(oracle_mod, kind):
    """SPEC examples: K = 0 -> empty set, loglik 0; K = I -> all, loglik 0."""
    for K, allin in ((np.zeros((3, 3)), False), (np.eye(3), True)):
        r = _run(oracle_mod, kind, _cast(kind, K))
        assert r.mask.tolist() == ([1, 1, 1] if allin else [0, 0, 0])
        assert r.loglik == 0.0


def test_empty_kernel(oracle_mod):
    for kind in KINDS:
        r = _run(oracle_mod, kind, _cast(kind, np.zeros((0, 0))))
        assert r.mask.shape == (0,) and r.loglik == 0.0 and r.n_kept == 0


def test_nonhermitian_2x2_example(oracle_mod):
    """K = [[.5, 1], [.25, .5]] = D^-1 K0 D (K0 rank-1 projection):
    exactly one of {0}, {1}; loglik ln 0.5 (Prop. 2 + PAPER.md:452-455)."""
    K = np.array([[0.5, 1.0], [0.25, 0.5]], dtype=np.complex128)
    masks, lls = oracle_mod.sample_many(oracle_mod.LU_Z, K, 3, 0, 20000)
    assert np.all(masks.sum(axis=1) == 1)
    assert np.allclose(lls, np.log(0.5), rtol=1e-15)
    frac = masks[:, 0].mean()
    assert abs(frac - 0.5) < 4 * np.sqrt(0.25 / 20000)


# ----------------------------------------------------------------- sampler law (brute force)
def _brute(oracle_mod, kind_id, K, draws, seed=2):
    masks, lls = oracle_mod.sample_many(kind_id, K, seed, 0, draws)
    idx = masks_to_index(masks)
    counts = np.bincount(idx, minlength=1 << K.shape[0]).astype(float)
    p = subset_probabilities(K)
    ok, rep = check_subset_frequencies(p, counts)
    # the likelihood of every draw is its subset's probability
    assert np.allclose(np.exp(lls), p[idx], rtol=1e-9, atol=1e-300)
    return ok, rep


def test_brute_force_herm_d(oracle_mod):
    """|det(K - 1_{S^c})| law (Theorem 'Factorization-based DPP sampling',
    PAPER.md:389-423) for a Haar real kernel, n = 8, 10^6 draws."""
    K = W.haar_kernel(8, seed=1)
    ok, rep = _brute(oracle_mod, oracle_mod.HERM_D, K, 1_000_000)
    assert ok, rep


def test_brute_force_herm_z(oracle_mod):
    K = W.haar_kernel(6, seed=2, complex_=True)
    ok, rep = _brute(oracle_mod, oracle_mod.HERM_Z, K, 400_000)
    assert ok, rep


def test_brute_force_lu_z_similarity(oracle_mod):
    """Non-Hermitian D^-1 K D (Prop. 2): same law as K."""
    K0 = W.haar_kernel(6, seed=3, complex_=True)
    K = W.similarity(K0, seed=3)
    assert np.allclose(subset_probabilities(K), subset_probabilities(K0), atol=1e-12)
    ok, rep = _brute(oracle_mod, oracle_mod.LU_Z, K, 400_000)
    assert ok, rep


def test_brute_force_aztec_d2(oracle_mod):
    """Aztec diamond d = 2: n = 16, exactly 8 tilings each with probability 1/8
    (all tilings equally likely; 2^{d(d+1)/2} tilings)."""
    K = W.aztec_kernel(2)
    assert K.shape == (16, 16)
    masks, lls = oracle_mod.sample_many(oracle_mod.LU_Z, K, 9, 0, 80_000)
    assert all(W.is_aztec_tiling(2, m) for m in masks[:2000])
    assert np.allclose(lls, -3 * np.log(2.0), atol=1e-12)
    idx = masks_to_index(masks)
    vals, counts = np.unique(idx, return_counts=True)
    assert len(vals) == 8
    assert np.all(np.abs(counts - 10_000) < 4.5 * np.sqrt(80_000 / 8 * 7 / 8))


def test_marginals_herm_d(oracle_mod):
    """Inclusion frequencies match diag(K) (Definition 1)."""
    K = W.haar_kernel(24, seed=4, spectrum="beta")
    masks, _ = oracle_mod.sample_many(oracle_mod.HERM_D, K, 5, 0, 100_000)
    ok, rep = check_marginals(K, masks)
    assert ok, rep
    # pairwise marginals det(K_{ij}) on a few pairs
    N = masks.shape[0]
    for i, j in [(0, 1), (3, 17), (22, 23)]:
        pij = K[i, i] * K[j, j] - K[i, j] * K[j, i]
        f = np.mean(masks[:, i] & masks[:, j])
        assert abs(f - pij) < 4.5 * np.sqrt(pij * (1 - pij) / N)


# ----------------------------------------------------------------- likelihood + factor identities
@pytest.mark.parametrize("kind", KINDS)
def test_loglik_is_log_det_and_factor(oracle_mod, kind):
    """loglik = ln|det(K - 1_{Y^c})| (LAPACK slogdet) and the returned factor
    reproduces K - 1_{Y^c} (Listing 1 caption)."""
    n = 96
    if kind == "herm_d":
        K = W.haar_kernel(n, seed=6)
    elif kind == "herm_z":
        K = W.haar_kernel(n, seed=6, complex_=True)
    else:
        K = W.similarity(W.haar_kernel(n, seed=6, complex_=True), seed=6)
    for b in range(3):
        r = _run(oracle_mod, kind, K, seed=1, b=b)
        M = K - np.diag(1.0 - r.mask)
        _, ld = np.linalg.slogdet(M)
        assert r.loglik == pytest.approx(ld, rel=1e-10)
        F = r.factor
        L = np.tril(F, -1) + np.eye(n)
        if kind == "lu_z":
            R = L @ np.triu(F)
        else:
            D = np.real(np.diagonal(F))
            R = (L * D[None, :]) @ L.conj().T
            if kind == "herm_z":
                assert np.all(np.imag(np.diagonal(F)) == 0)
        assert np.max(np.abs(R - M)) <= 1e-10 * max(1.0, np.max(np.abs(K)))
        assert r.n_kept == int(r.mask.sum())


def test_hermitian_upper_untouched(oracle_mod):
    K = W.haar_kernel(20, seed=8)
    r = oracle_mod.sample_herm_d(K)
    iu = np.triu_indices(20, 1)
    assert np.array_equal(r.factor[iu], K[iu])


def test_lu_of_real_kernel_matches_ldl(oracle_mod):
    """Prop. 2 with D = I, and LU vs LDL^H specialisation:
    for symmetric K the LU sampler and the LDL^T sampler make the same decisions."""
    K = W.haar_kernel(64, seed=9)
    for b in range(3):
        a = oracle_mod.sample_herm_d(K, 4, b)
        c = oracle_mod.sample_lu_z(K.astype(np.complex128), 4, b)
        assert a.n_ties == 0
        assert np.array_equal(a.mask, c.mask)
        assert a.loglik == pytest.approx(c.loglik, rel=1e-12)


def test_similarity_invariance_of_decisions(oracle_mod):
    """The Schur complements of D^-1 K D have the same diagonals (Prop. 2), so
    with the same uniforms the decisions match those on K."""
    K0 = W.haar_kernel(64, seed=10, complex_=True)
    K = W.similarity(K0, seed=10)
    for b in range(3):
        a = oracle_mod.sample_herm_z(K0, 2, b)
        c = oracle_mod.sample_lu_z(K, 2, b)
        assert np.array_equal(a.mask, c.mask)
        assert a.loglik == pytest.approx(c.loglik, rel=1e-11)


# ----------------------------------------------------------------- projections, forced replay, prefix
@pytest.mark.parametrize("kind", ["herm_d", "herm_z"])
def test_projection_cardinality(oracle_mod, kind):
    """Projection kernels give samples of cardinality = rank."""
    for n, r in ((64, 20), (100, 99), (33, 1)):
        K = W.projection_kernel(n, r, seed=n + r, complex_=(kind == "herm_z"))
        for b in range(4):
            res = _run(oracle_mod, kind, K, 3, b)
            assert res.n_kept == r


@pytest.mark.parametrize("kind", KINDS)
def test_forced_replay(oracle_mod, kind):
    """Forcing the decisions of a sample reproduces it; forcing any S gives
    loglik = ln|det(K - 1_{S^c})| (SPEC log_likelihood_of)."""
    n = 40
    K = W.haar_kernel(n, seed=12, complex_=(kind != "herm_d"))
    r = _run(oracle_mod, kind, K, 5, 0)
    r2 = _run(oracle_mod, kind, K, 5, 0, forced=r.mask)
    assert np.array_equal(r.mask, r2.mask) and r.loglik == r2.loglik
    assert np.array_equal(r.factor, r2.factor)
    S = (np.arange(n) % 3 == 0).astype(np.uint8)
    r3 = _run(oracle_mod, kind, K, 5, 0, forced=S)
    _, ld = np.linalg.slogdet(K - np.diag(1.0 - S))
    assert r3.loglik == pytest.approx(ld, rel=1e-10)


@pytest.mark.parametrize("kind", KINDS)
def test_prefix_property(oracle_mod, kind):
    """Loop invariant: pivots [0:m) depend only on K[0:m,0:m]
    and u[0:m) -> the sample of the leading block equals the prefix, bitwise."""
    n, m = 150, 61
    K = W.haar_kernel(n, seed=13, complex_=(kind != "herm_d"))
    if kind == "lu_z":
        K = W.similarity(K, seed=13)
    full = _run(oracle_mod, kind, K, 8, 3)
    pre = _run(oracle_mod, kind, np.asfortranarray(K[:m, :m]), 8, 3)
    assert np.array_equal(full.mask[:m], pre.mask)
    if kind == "lu_z":
        assert np.array_equal(full.factor[:m, :m], pre.factor)
    else:
        il = np.tril_indices(m)
        assert np.array_equal(full.factor[:m, :m][il], pre.factor[il])


def test_determinism(oracle_mod):
    K = W.haar_kernel(50, seed=14)
    a = oracle_mod.sample_herm_d(K, 99, 7)
    b = oracle_mod.sample_herm_d(K, 99, 7)
    assert np.array_equal(a.mask, b.mask) and a.loglik == b.loglik
    c = oracle_mod.sample_herm_d(K, 99, 8)
    assert not np.array_equal(a.mask, c.mask)


def test_tie_and_range_diagnostics(oracle_mod):
    """Reading R8 / R3: a pivot within tie_tol of its uniform is reported; pivots
    outside [-1e-8, 1+1e-8] are counted, never clamped."""
    u0 = oracle_mod.uniform(0, 0, 0)
    K = np.diag([u0 + 5e-10, 1.5, -0.2])
    r = oracle_mod.sample_herm_d(K, 0, 0)
    assert r.n_ties == 1 and r.first_tie == 0 and r.mask[0] == 1
    assert r.n_out_of_range == 2
    assert r.mask[1] == 1 and r.mask[2] == 0
    assert r.loglik == pytest.approx(np.log(u0 + 5e-10) + np.log(1.5) + np.log(1.2), rel=1e-14)


# ----------------------------------------------------------------- paper workloads
def test_ust_small_grid(oracle_mod):
    """UST of a 10x10 grid: every sample is a spanning tree and has loglik
    -ln tau(G) (Kirchhoff; PAPER.md:81-83 for the 40x40 analogue)."""
    rows = cols = 10
    K = W.ust_kernel(rows, cols)
    edges = W.grid_edges(rows, cols)
    want = -W.log_num_spanning_trees_grid(rows, cols)
    for b in range(4):
        r = oracle_mod.sample_herm_d(K, 0, b)
        assert W.is_spanning_tree(rows * cols, edges, r.mask)
        assert r.loglik == pytest.approx(want, rel=1e-10)


@pytest.mark.slow
def test_ust_40x40_paper_pin(oracle_mod):
    """Config 1 / Fig. 1: 3120 edges, 1599 kept, a spanning
    tree, loglik -1794.24 as printed (closed form -1794.2382014120)."""
    K = W.ust_kernel(40, 40)
    assert K.shape == (GOLD["ust_40x40_ground_set"]["value"],) * 2
    r = oracle_mod.sample_herm_d(K, 0, 0)
    assert r.n_kept == 1599
    assert W.is_spanning_tree(1600, W.grid_edges(40, 40), r.mask)
    closed = -W.log_num_spanning_trees_grid(40, 40)
    assert closed == pytest.approx(-1794.2382014120, abs=1e-9)
    assert r.loglik == pytest.approx(closed, rel=1e-10)
    assert round(r.loglik, GOLD["ust_40x40_loglik"]["digits_after_point"]) == GOLD["ust_40x40_loglik"]["value"]


def test_aztec_d10_paper_pin(oracle_mod):
    """Fig. 3: order-10 Aztec diamond, n = 400; each sample is
    a perfect tiling with 110 dominoes and loglik -38.1231 = -55 ln 2."""
    K = W.aztec_kernel(10)
    assert K.shape == (400, 400)
    for b in range(2):
        r = oracle_mod.sample_lu_z(K, 0, b)
        assert W.is_aztec_tiling(10, r.mask)
        assert r.loglik == pytest.approx(-55 * np.log(2.0), rel=1e-10)
        assert round(r.loglik, 4) == GOLD["aztec_d10_loglik"]["value"]
        assert r.max_abs_imag_pivot < 1e-10


# ------------------------------------------------------------------ greedy MAP
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_map_diag_closed_form(oracle_mod, kind):
    """K = diag(p): the greedy decisions are p_j >= 1/2 (include at exactly 1/2, reading R18) and
    the log-likelihood is sum ln max(p, 1 - p)."""
    p = np.array([0.1, 0.5, 0.9, 0.49, 0.51, 0.0, 1.0, 0.25])
    K = np.diag(p).astype(np.complex128 if kind else np.float64)
    r = oracle_mod.greedy_map(kind, K)
    assert np.array_equal(r.mask, (p >= 0.5).astype(np.uint8))
    want = np.sum(np.log(np.where(p >= 0.5, p, 1 - p)))
    assert abs(r.loglik - want) <= 1e-15
    assert r.n_ties == 1 and r.first_tie == 1   # p = 1/2 exactly


@pytest.mark.parametrize("kind,n", [(0, 10), (1, 9), (2, 9), (0, 60)])
def test_map_is_greedy_on_leading_minors(oracle_mod, kind, n):
    """At every pivot j the greedy result takes the more probable branch: with Y_j the decisions
    on [0, j], P(Y cap [0,j] = Y_j) = |det((K - 1_{Y^c})[0:j+1, 0:j+1])| (the leading principal
    minors of K - 1_{S^c}, PAPER.md:452-455 applied to the restriction, Def. 1), so the chosen
    minor must be >= the one with decision j flipped.  Also loglik = ln|det(K - 1_{Y^c})|."""
    K = W.haar_kernel(n, seed=100 + n, complex_=(kind != 0))
    if kind == 2:
        K = W.similarity(K, seed=n)
    r = oracle_mod.greedy_map(kind, K)
    keep = r.mask.astype(bool)
    for j in range(n):
        M = K[: j + 1, : j + 1].copy()
        M[np.arange(j + 1), np.arange(j + 1)] -= (~keep[: j + 1]).astype(float)
        alt = M.copy()
        alt[j, j] += 1.0 if not keep[j] else -1.0
        assert abs(np.linalg.det(M)) >= abs(np.linalg.det(alt)) * (1 - 1e-12), j
    Kd = K.copy()
    Kd[np.arange(n), np.arange(n)] -= (~keep).astype(float)
    assert abs(r.loglik - np.linalg.slogdet(Kd)[1]) <= 1e-10 * max(1.0, abs(r.loglik))


def test_map_deterministic_and_brute_force_likelihood(oracle_mod):
    """The greedy result is deterministic and its likelihood is the brute-force probability
    |det(K - 1_{Y^c})| of the returned set."""
    n = 8
    K = W.haar_kernel(n, seed=5)
    r1 = oracle_mod.greedy_map(0, K)
    r2 = oracle_mod.greedy_map(0, K)
    assert np.array_equal(r1.mask, r2.mask) and r1.loglik == r2.loglik
    from tests.stats_util import subset_probabilities
    p = subset_probabilities(K)
    idx = int(sum(int(v) << j for j, v in enumerate(r1.mask)))
    assert abs(np.log(p[idx]) - r1.loglik) <= 1e-10 * abs(r1.loglik)
