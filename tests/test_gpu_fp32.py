"""GPU parity of the single-precision samplers (dpp_sample_herm_s / dpp_sample_lu_c; SURVEY §8(f)
rank 2, reading R19) against the fp32 oracle, through the C ABI.

Tolerances (derived from fp32 arithmetic, R19): both sides round every entry to fp32
(eps = 6e-8) but in different orders (the GPU blocks the factorization, fuses multiply-adds and
scales by 1/p), so entries drift by O(n eps) relative to max|K|: factors within 3e-4 max|K| for
n <= 1000, loglik within 3e-5 relative.  Decisions are compared bit for bit up to the first pivot
whose uniform lies within 1e-4 of the oracle's fp32 pivot (the fp32 analogue of reading R8).
"""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import from_device, to_device

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402

FTOL, LTOL, TIE32 = 3e-4, 3e-5, 1e-4


def _kernel(kind, n, seed):
    if kind == "herm_s":
        return W.haar_kernel(n, seed=seed).astype(np.float32)
    return W.similarity(W.haar_kernel(n, seed=seed, complex_=True), seed=seed).astype(np.complex64)


@pytest.mark.parametrize("kind,n,nb,la,flags", [
    ("herm_s", 1, 0, 1, 0), ("herm_s", 100, 0, 1, 0), ("herm_s", 300, 0, 1, 0), ("herm_s", 1000, 0, 0, 0),
    ("herm_s", 1000, 64, 1, 0), ("herm_s", 2125, 0, 1, 0), ("herm_s", 2125, 256, 1, 0),
    # the FP32 SIMT updates (DPP_FLAG_FP32_SIMT) instead of the default 3xTF32 tensor-core updates
    ("herm_s", 300, 0, 1, 2), ("herm_s", 2125, 0, 1, 2), ("herm_s", 1000, 64, 0, 2),
    ("lu_c", 130, 0, 1, 0), ("lu_c", 600, 0, 1, 0), ("lu_c", 600, 32, 0, 0), ("lu_c", 1100, 0, 1, 0),
    ("lu_c", 600, 0, 1, 2), ("lu_c", 1100, 128, 1, 2)])
def test_fp32_matches_fp32_oracle(oracle_mod, kind, n, nb, la, flags):
    K = _kernel(kind, n, n + 3)
    fn = oracle_mod.sample_herm_s if kind == "herm_s" else oracle_mod.sample_lu_c
    o = fn(K, 7, 0, tie_tol=TIE32)
    Kc = to_device(K, kind)
    s = dpp.sample(kind, Kc, 7, opts=dpp.make_opts(nb=nb, lookahead=la, flags=flags))
    torch.cuda.synchronize()
    mask = s.mask.cpu().numpy()
    k = o.first_tie if o.n_ties else n
    assert np.array_equal(mask[:k], o.mask[:k]), np.flatnonzero(mask[:k] != o.mask[:k])[:5]
    if o.n_ties == 0:
        part = np.tril if kind == "herm_s" else (lambda A: A)
        d = np.max(np.abs(part(from_device(Kc, n)) - part(o.factor))) if n else 0.0
        assert d <= FTOL * float(np.max(np.abs(K))), d
        assert abs(float(s.loglik) - o.loglik) <= LTOL * abs(o.loglik) + 1e-6


def test_fp32_batched_and_structure(oracle_mod):
    """Batched fp32 UST samples of the 20x20 grid are spanning trees; the order-10
    Aztec diamond in fp32 gives perfect tilings with loglik -55 ln 2."""
    K = W.ust_kernel(20, 20).astype(np.float32)
    edges = W.grid_edges(20, 20)
    s = dpp.sample_batched("herm_s", to_device(K, "herm_s"), 32, seed=1, b0=0)
    masks, lls = s.mask.cpu().numpy(), s.loglik.cpu().numpy()
    want = -W.log_num_spanning_trees_grid(20, 20)
    for b in range(32):
        assert W.is_spanning_tree(400, edges, masks[b])
        assert abs(lls[b] - want) <= 1e-4 * abs(want)
    o = oracle_mod.sample_herm_s(K, 1, 0, tie_tol=TIE32)
    kk = o.first_tie if o.n_ties else len(o.mask)
    assert np.array_equal(masks[0][:kk], o.mask[:kk])
    M = W.aztec_kernel_balanced(10, storage="natural").numpy().astype(np.complex64)
    s = dpp.sample_batched("lu_c", to_device(M, "lu_c"), 8, seed=2, b0=0)
    for b in range(8):
        assert W.is_aztec_tiling(10, s.mask[b].cpu().numpy())
        assert abs(float(s.loglik[b]) + 55 * np.log(2.0)) <= 1e-4 * 55 * np.log(2.0)


def test_fp32_bench_configuration_prefix(oracle_mod):
    """The herm_s bench configuration (n = 16384, the configs[3] kernel rounded to fp32, nb = 128):
    the leading 1536 x 1536 block's decisions equal the fp32 oracle's (prefix property)."""
    n, m = 16384, 1536
    Kc = W.haar_kernel_torch(n, seed=0, spectrum="beta").to(torch.float32)
    Kpre = Kc[:m, :m].cpu().numpy().T.copy()
    s = dpp.sample("herm_s", Kc, 0, opts=dpp.make_opts(nb=128, lookahead=1))
    torch.cuda.synchronize()
    o = oracle_mod.sample_herm_s(Kpre, 0, 0, tie_tol=TIE32)
    k = o.first_tie if o.n_ties else m
    assert np.array_equal(s.mask.cpu().numpy()[:k], o.mask[:k])
    assert 0.4 * n < int(s.mask.sum()) < 0.6 * n
