"""Pins of the single-precision oracle functions (oracle_sample_herm_s / _lu_c; reading R19:
fp32 factorization as in the paper's single-precision runs; decisions against
the fp32 pivot promoted to fp64; fp64 likelihood accumulation).

Independent of the oracle's loop: the diag(p) closed form in fp32, brute-force subset
frequencies vs |det(K - 1_{S^c})| of the fp32 kernel (numpy fp64 det), agreement with the pinned
fp64 oracle within fp32 rounding, and the UST / Aztec structural pins.
"""
import numpy as np
import pytest

import workloads as W
from tests.stats_util import check_subset_frequencies, masks_to_index, subset_probabilities


@pytest.mark.parametrize("kind", ["herm_s", "lu_c"])
def test_fp32_diagonal_closed_form(oracle_mod, kind):
    rng = np.random.default_rng(9)
    n = 40
    p = rng.uniform(0, 1, n).astype(np.float32)
    p[:3] = [0.0, 1.0, 0.5]
    K = np.diag(p).astype(np.float32 if kind == "herm_s" else np.complex64)
    fn = oracle_mod.sample_herm_s if kind == "herm_s" else oracle_mod.sample_lu_c
    for b in range(4):
        r = fn(K, 13, b)
        u = np.array([oracle_mod.uniform(13, j, b) for j in range(n)])
        keep = u <= p.astype(np.float64)
        assert np.array_equal(r.mask.astype(bool), keep)
        piv = np.where(keep, p, (p - np.float32(1.0)).astype(np.float32)).astype(np.float64)
        assert r.loglik == pytest.approx(np.sum(np.log(np.abs(piv))), rel=1e-14, abs=1e-14)
        assert r.factor.dtype == (np.float32 if kind == "herm_s" else np.complex64)


@pytest.mark.parametrize("kind,n,draws", [("herm_s", 6, 300_000), ("lu_c", 6, 300_000)])
def test_fp32_brute_force_law(oracle_mod, kind, n, draws):
    """P(Y = S) = |det(K - 1_{S^c})| for the fp32 kernel, within reading R12."""
    if kind == "herm_s":
        K = W.haar_kernel(n, seed=21).astype(np.float32)
    else:
        K = W.similarity(W.haar_kernel(n, seed=21, complex_=True), seed=21).astype(np.complex64)
    masks, lls = oracle_mod.sample_many(3 if kind == "herm_s" else 4, K, 5, 0, draws)
    p = subset_probabilities(K.astype(np.float64 if kind == "herm_s" else np.complex128))
    idx = masks_to_index(masks)
    counts = np.bincount(idx, minlength=1 << n).astype(float)
    ok, rep = check_subset_frequencies(p, counts)
    assert ok, rep
    assert np.allclose(np.exp(lls), p[idx], rtol=2e-5)


@pytest.mark.parametrize("kind,n", [("herm_s", 200), ("lu_c", 150)])
def test_fp32_matches_fp64_oracle(oracle_mod, kind, n):
    """The fp32 sample agrees with the (pinned) fp64 oracle on the same kernel: identical decisions
    up to the first pivot within 1e-3 of its uniform, loglik within 1e-4 relative, factor within
    1e-3 max|K| -- fp32 rounding (eps 6e-8) grown over n pivots."""
    if kind == "herm_s":
        K64 = W.haar_kernel(n, seed=4)
        r32 = oracle_mod.sample_herm_s(K64.astype(np.float32), 3, 0)
        r64 = oracle_mod.sample_herm_d(K64.astype(np.float32).astype(np.float64), 3, 0)
    else:
        K64 = W.similarity(W.haar_kernel(n, seed=4, complex_=True), seed=4)
        r32 = oracle_mod.sample_lu_c(K64.astype(np.complex64), 3, 0)
        r64 = oracle_mod.sample_lu_z(K64.astype(np.complex64).astype(np.complex128), 3, 0)
    r64t = (oracle_mod.sample_herm_d if kind == "herm_s" else oracle_mod.sample_lu_z)(
        K64.astype(np.float32 if kind == "herm_s" else np.complex64).astype(
            np.float64 if kind == "herm_s" else np.complex128), 3, 0, tie_tol=1e-3)
    k = r64t.first_tie if r64t.n_ties else n
    assert k > 20
    assert np.array_equal(r32.mask[:k], r64.mask[:k])
    if r64t.n_ties == 0:
        assert abs(r32.loglik - r64.loglik) <= 1e-4 * abs(r64.loglik)
        part = np.tril if kind == "herm_s" else (lambda A: A)
        assert np.max(np.abs(part(r32.factor) - part(r64.factor))) <= 1e-3 * np.max(np.abs(K64))


def test_fp32_ust_and_aztec_structure(oracle_mod):
    """Structural pins in fp32: UST of the 10x10 grid (spanning trees, loglik -ln tau(G)) and the
    order-10 Aztec diamond on the balanced kernel (perfect tilings, loglik -55 ln 2)."""
    K = W.ust_kernel(10, 10).astype(np.float32)
    edges = W.grid_edges(10, 10)
    want = -W.log_num_spanning_trees_grid(10, 10)
    for b in range(3):
        r = oracle_mod.sample_herm_s(K, 0, b)
        assert W.is_spanning_tree(100, edges, r.mask)
        assert abs(r.loglik - want) <= 1e-4 * abs(want)
    M = W.aztec_kernel_balanced(10, storage="natural").numpy().astype(np.complex64)
    for b in range(3):
        r = oracle_mod.sample_lu_c(M, 0, b)
        assert W.is_aztec_tiling(10, r.mask)
        assert abs(r.loglik + 55 * np.log(2.0)) <= 1e-4 * 55 * np.log(2.0)
