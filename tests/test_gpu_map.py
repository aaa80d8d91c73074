"""GPU parity of greedy MAP inference (dpp_map_{herm_d,herm_z,lu_z}, reading
R18) against the oracle's greedy_map: decisions bit-exact (prefix before a tie), factor within
1e-9 max|K|, loglik within 1e-10 relative -- at sizes spanning several tiles with ragged tails,
with and without lookahead."""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import assert_factor_close, assert_loglik_close, compare_masks, from_device, to_device

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402

KIND = {"herm_d": 0, "herm_z": 1, "lu_z": 2}


@pytest.mark.parametrize("kind,n,la", [("herm_d", 1, 1), ("herm_d", 300, 1), ("herm_d", 1000, 0),
                                        ("herm_d", 2125, 1), ("herm_z", 200, 1), ("herm_z", 777, 0),
                                        ("lu_z", 130, 1), ("lu_z", 600, 1), ("lu_z", 600, 0)])
def test_map_matches_oracle(oracle_mod, kind, n, la):
    K = W.haar_kernel(n, seed=n + 1, complex_=(kind != "herm_d"))
    if kind == "lu_z":
        K = W.similarity(K, seed=n)
    o = oracle_mod.greedy_map(KIND[kind], K)
    Kc = to_device(K, kind)
    s = dpp.greedy_map(kind, Kc, opts=dpp.make_opts(lookahead=la))
    torch.cuda.synchronize()
    compare_masks(s.mask.cpu().numpy(), o)
    info = s.info_dicts()[0]
    assert info["n_ties"] == o.n_ties
    if o.n_ties == 0:
        assert_factor_close(from_device(Kc, n), o.factor, K, kind)
        assert_loglik_close(float(s.loglik), o.loglik)
        assert info["n_kept"] == o.n_kept


def test_map_diag_closed_form():
    p = np.array([0.1, 0.5, 0.9, 0.49, 0.51, 0.0, 1.0, 0.25])
    Kc = to_device(np.diag(p), "herm_d")
    s = dpp.greedy_map("herm_d", Kc)
    assert np.array_equal(s.mask.cpu().numpy(), (p >= 0.5).astype(np.uint8))
    assert abs(float(s.loglik) - np.sum(np.log(np.where(p >= 0.5, p, 1 - p)))) <= 1e-15
