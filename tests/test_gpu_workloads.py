"""GPU checks on the paper's workloads (BASELINE.json configs) -- through the C ABI.

* config 0: n = 256 Haar kernel; brute force at n <= 12 (10^6 draws on the GPU) with the
  reading-#12 3-sigma criteria; marginals vs diag(K).
* config 1: UST of the 40x40 grid, batch of samples: spanning trees with the closed-form
  likelihood -ln tau = -1794.2382 (paper: exp(-1794.24)).
* config 2: Aztec tilings with loglik -d(d+1)/2 ln 2: d = 10 / 20 in
  the plain gauge, d = 80 (n = 25600, the config itself) in the balanced gauge (reading R13).
* config 3: n = 16384 Beta(1/2,1/2) kernel at the bench's launch configuration: prefix parity
  against the oracle on K[:m,:m] (loop invariant) + full-size invariants.
"""
import json
import os

import numpy as np
import pytest

import workloads as W
from tests.gpu_util import (assert_factor_close, assert_loglik_close, check_decisions, compare_masks, from_device,
                            to_device)
from tests.stats_util import (check_marginals, check_subset_frequencies, masks_to_index,
                              subset_probabilities)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


@pytest.mark.parametrize("kind,n,draws", [("herm_d", 8, 1_000_000), ("herm_d", 12, 1_000_000),
                                          ("herm_z", 7, 400_000), ("lu_z", 7, 400_000)])
def test_brute_force_law_gpu(oracle_mod, kind, n, draws):
    """P(Y = S) = |det(K - 1_{S^c})| within reading #12's 3-sigma criteria."""
    K = W.haar_kernel(n, seed=n, complex_=(kind != "herm_d"))
    if kind == "lu_z":
        K = W.similarity(K, seed=n)
    Kc = to_device(K, kind)
    s = dpp.sample_batched(kind, Kc, draws, seed=31, b0=0, opts=dpp.make_opts(batch_chunk=65535))
    masks = s.mask.cpu().numpy()
    lls = s.loglik.cpu().numpy()
    p = subset_probabilities(K)
    idx = masks_to_index(masks)
    counts = np.bincount(idx, minlength=1 << n).astype(float)
    ok, rep = check_subset_frequencies(p, counts)
    assert ok, rep
    assert np.allclose(np.exp(lls), p[idx], rtol=1e-9)
    # the first draws agree with the oracle bit for bit
    om, ol = oracle_mod.sample_many({"herm_d": 0, "herm_z": 1, "lu_z": 2}[kind], K, 31, 0, 2000)
    assert np.array_equal(masks[:2000], om)
    assert np.allclose(lls[:2000], ol, rtol=1e-12)


def test_config0_n256_marginals_and_parity(oracle_mod):
    """Config 0: n = 256, lam ~ U(0,1), Philox seed 0."""
    K = W.haar_kernel(256, seed=0)
    Kc = to_device(K, "herm_d")
    N = 20000
    s = dpp.sample_batched("herm_d", Kc, N, seed=0, b0=0, opts=dpp.make_opts(batch_chunk=4096))
    masks = s.mask.cpu().numpy()
    ok, rep = check_marginals(K, masks)
    assert ok, rep
    for b in (0, 1, 2, N - 1):
        o = oracle_mod.sample_herm_d(K, 0, b)
        compare_masks(masks[b], o)
        if o.n_ties == 0:
            assert_loglik_close(float(s.loglik[b]), o.loglik)
    # single in-place sample b = 0 with its factor
    o = oracle_mod.sample_herm_d(K, 0, 0)
    Kc2 = to_device(K, "herm_d")
    s0 = dpp.sample("herm_d", Kc2, 0)
    compare_masks(s0.mask.cpu().numpy(), o)
    assert_factor_close(from_device(Kc2, 256), o.factor, K, "herm_d")


def test_config1_ust_40x40_batch(oracle_mod):
    """Config 1: UST of the 40x40 grid (n = 3120, rank 1599), batch of samples."""
    K = W.ust_kernel(40, 40)
    edges = W.grid_edges(40, 40)
    closed = -W.log_num_spanning_trees_grid(40, 40)
    Kc = to_device(K, "herm_d")
    batch = 64
    s = dpp.sample_batched("herm_d", Kc, batch, seed=0, b0=0)
    masks, lls = s.mask.cpu().numpy(), s.loglik.cpu().numpy()
    for b in range(batch):
        assert masks[b].sum() == 1599
        assert W.is_spanning_tree(1600, edges, masks[b])
        assert abs(lls[b] - closed) <= 1e-9 * abs(closed)
        assert round(lls[b], 2) == GOLD["ust_40x40_loglik"]["value"]
    o = oracle_mod.sample_herm_d(K, 0, 0)
    compare_masks(masks[0], o)


@pytest.mark.parametrize("d", [10, 20])
def test_config2_aztec(oracle_mod, d):
    """Config 2 scaled down: Aztec diamond tilings, plain gauge."""
    K = W.aztec_kernel(d)
    Kc = to_device(K, "lu_z")
    batch = 4
    s = dpp.sample_batched("lu_z", Kc, batch, seed=0, b0=0)
    masks, lls = s.mask.cpu().numpy(), s.loglik.cpu().numpy()
    want = -d * (d + 1) / 2 * np.log(2.0)
    for b in range(batch):
        assert W.is_aztec_tiling(d, masks[b])
        assert abs(lls[b] - want) <= 1e-8 * abs(want)
    if d == 10:
        assert round(lls[0], 4) == GOLD["aztec_d10_loglik"]["value"]
        o = oracle_mod.sample_lu_z(K, 0, 0)
        compare_masks(masks[0], o)


def test_config2_aztec_d80_balanced(oracle_mod):
    """Config 2 itself: order-80 Aztec diamond, n = 25600 complex128 non-Hermitian LU sampler on
    the balanced-gauge Kenyon kernel (reading R13), in place at the default nb = 64 with
    lookahead.  Every sample is a perfect tiling with 80*81 = 6480 dominoes and likelihood
    exp(-3240 ln 2) (paper: e^{-2245.8}); the leading 1024 x 1024 block of the
    factor and its decisions equal the oracle's sample of K[:1024, :1024] (prefix property)."""
    d, m = 80, 1024
    n = 4 * d * d
    Kc = W.aztec_kernel_balanced(d, device="cuda")
    assert Kc.shape == (n, n)
    Kpre = Kc[:m, :m].cpu().numpy().T.copy()
    s = dpp.sample("lu_z", Kc, 0)
    torch.cuda.synchronize()
    mask = s.mask.cpu().numpy()
    assert int(mask.sum()) == GOLD["aztec_d80_dominoes"]["value"]
    assert W.is_aztec_tiling(d, mask)
    want = -d * (d + 1) / 2 * np.log(2.0)
    ll = float(s.loglik)
    assert abs(ll - want) <= 1e-9 * abs(want), (ll, want)
    assert round(ll, 1) == GOLD["aztec_d80_loglik"]["value"]
    info = s.info_dicts()[0]
    assert info["n_kept"] == 6480 and info["n_ties"] == 0
    # every one of the 25600 decisions against the oracle's uniforms (LU pivot = U_jj)
    check_decisions(mask, torch.diagonal(Kc).cpu().numpy(), 0, 0, oracle_mod)
    o = oracle_mod.sample_lu_z(Kpre, 0, 0)
    compare_masks(mask[:m], o)
    if o.n_ties == 0:
        assert_factor_close(Kc[:m, :m].cpu().numpy().T, o.factor, Kpre, "lu_z")


def test_config3_n16384_prefix_parity(oracle_mod):
    """Config 3 at full size, in the bench's launch configuration (nb = 128, lookahead 1):
    decisions/factor of the leading m x m block equal the oracle's sample of K[:m,:m];
    loglik = sum ln|D|; randomized check of L D L^T = K - 1_{Y^c}."""
    n, m = 16384, 1536
    Kc = W.haar_kernel_torch(n, seed=0, spectrum="beta")
    K0 = Kc.clone()
    Kpre = Kc[:m, :m].cpu().numpy().T.copy()
    s = dpp.sample("herm_d", Kc, 0, opts=dpp.make_opts(nb=128, lookahead=1))
    torch.cuda.synchronize()
    mask = s.mask.cpu().numpy()
    o = oracle_mod.sample_herm_d(Kpre, 0, 0)
    k = compare_masks(mask[:m], o)
    F = Kc[:m, :m].cpu().numpy().T
    if o.n_ties == 0:
        assert_factor_close(F, o.factor, Kpre, "herm_d")
        lpre = float(np.sum(np.log(np.abs(np.diagonal(F)))))
        assert_loglik_close(lpre, o.loglik)
    assert k == m or o.n_ties > 0
    # full-size invariants
    D = torch.diagonal(Kc)
    assert abs(float(torch.log(D.abs()).sum()) - float(s.loglik)) <= 1e-10 * abs(float(s.loglik))
    assert 0.4 * n < int(s.mask.sum()) < 0.6 * n
    # every one of the 16384 decisions against the oracle's uniforms (not only the prefix)
    check_decisions(mask, D.cpu().numpy(), 0, 0, oracle_mod)
    # randomized factor check on the GPU: (L D L^T) x vs (K - 1_{Y^c}) x
    Lt = torch.tril(Kc.T, -1) + torch.eye(n, dtype=torch.float64, device="cuda")  # natural L
    Kn = torch.tril(K0.T) + torch.tril(K0.T, -1).T
    x = torch.randn(n, 3, dtype=torch.float64, device="cuda")
    lhs = Lt @ (D[:, None] * (Lt.T @ x))
    rhs = Kn @ x - (1.0 - s.mask.double())[:, None] * x
    err = float((lhs - rhs).abs().max() / (Kn.abs().max() * x.abs().max()))
    assert err < 1e-9, err
