"""GPU test of the 1D block-column-cyclic entry point (dpp_sample_herm_d_dist) at world size 1
(one GPU per run here): same decisions, factor and loglik as the oracle; the block-cyclic update
addressing mode of the DMMA kernel is exercised on every step."""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import assert_factor_close, assert_loglik_close, compare_masks

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402
from paper_1905_00165_b200 import dist as D  # noqa: E402


@pytest.mark.parametrize("n", [1, 128, 300, 1000, 2049])
def test_dist_world1_matches_oracle(oracle_mod, n):
    K = W.haar_kernel(n, seed=n)
    o = oracle_mod.sample_herm_d(K, 5, 0)
    comm = dpp.dpp_comm_init(D.unique_id(), 1, 0)
    try:
        Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
        loc = D.to_local(Kc, n, 128, 1, 0)
        mask = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        info = torch.empty(32, dtype=torch.uint8, device="cuda")
        work = torch.empty(dpp.dpp_dist_workspace_bytes(dpp.DPP_OP_HERM_D, n, 1), dtype=torch.uint8, device="cuda")
        dpp.dpp_sample_herm_d_dist(comm, n, loc, loc.shape[1], 5, mask, ll, info, None, work)
        torch.cuda.synchronize()
        compare_masks(mask[:n].cpu().numpy(), o)
        if o.n_ties == 0:
            F = D.from_local([loc], n, 128, 1, Kc).cpu().numpy().T
            assert_factor_close(F, o.factor, K, "herm_d")
            assert_loglik_close(float(ll), o.loglik)
        i = dpp.Sample(mask, ll, info).info_dicts()[0]
        assert i["n_kept"] == o.n_kept
    finally:
        dpp.dpp_comm_destroy(comm)
