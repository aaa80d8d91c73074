"""GPU test of the 1D block-column-cyclic entry points (dpp_sample_herm_{d,z}_dist) at world size 1
(one GPU per run here): same decisions, factor and loglik as the oracle; the block-cyclic update
addressing mode of the DMMA kernel is exercised on every step, with and without the distributed
lookahead schedule (two prioritised streams, double-buffered messages)."""
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

CASES = [("herm_d", n, la) for n in (1, 128, 300, 1000, 2049) for la in (1, 0)] + \
        [("herm_z", n, la) for n in (1, 64, 200, 777) for la in (1, 0)]


@pytest.mark.parametrize("kind,n,la", CASES)
def test_dist_world1_matches_oracle(oracle_mod, kind, n, la):
    cplx = kind == "herm_z"
    nb = 64 if cplx else 128
    K = W.haar_kernel(n, seed=n, complex_=cplx)
    o = (oracle_mod.sample_herm_z if cplx else oracle_mod.sample_herm_d)(K, 5, 0)
    comm = dpp.dpp_comm_init(D.unique_id(), 1, 0)
    try:
        Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
        loc = D.to_local(Kc, n, nb, 1, 0)
        mask = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        info = torch.empty(32, dtype=torch.uint8, device="cuda")
        op = dpp.DPP_OP_HERM_Z if cplx else dpp.DPP_OP_HERM_D
        opts = dpp.make_opts(lookahead=la)
        work = torch.empty(dpp.dpp_dist_workspace_bytes(op, n, 1, opts), dtype=torch.uint8, device="cuda")
        fn = dpp.dpp_sample_herm_z_dist if cplx else dpp.dpp_sample_herm_d_dist
        fn(comm, n, loc, loc.shape[1], 5, mask, ll, info, opts, work)
        torch.cuda.synchronize()
        compare_masks(mask[:n].cpu().numpy(), o)
        if o.n_ties == 0:
            F = D.from_local([loc], n, nb, 1, Kc).cpu().numpy().T
            assert_factor_close(F, o.factor, K, kind)
            assert_loglik_close(float(ll), o.loglik)
        i = dpp.Sample(mask, ll, info).info_dicts()[0]
        assert i["n_kept"] == o.n_kept
    finally:
        dpp.dpp_comm_destroy(comm)


def test_dist_rejects_bad_nb():
    comm = dpp.dpp_comm_init(D.unique_id(), 1, 0)
    try:
        assert dpp.dpp_dist_workspace_bytes(dpp.DPP_OP_HERM_D, 100, 1, dpp.make_opts(nb=64)) == 0
        assert dpp.dpp_dist_workspace_bytes(dpp.DPP_OP_LU_Z, 100, 1) == 0
        loc = torch.zeros((100, 100), dtype=torch.float64, device="cuda")
        mask = torch.empty(100, dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        work = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
        with pytest.raises(dpp.DppError):
            dpp.dpp_sample_herm_d_dist(comm, 100, loc, 100, 0, mask, ll, None, dpp.make_opts(nb=64), work)
    finally:
        dpp.dpp_comm_destroy(comm)


@pytest.mark.parametrize("kind,n", [("herm_d", 32768), ("herm_z", 16384)])
def test_dist_full_size_bench_configuration(oracle_mod, kind, n):
    """configs[4] at (half of) its size in the bench's launch configuration (block-cyclic layout,
    lookahead, one rank): the leading 1024 x 1024 block's decisions equal the oracle's sample of
    K[:1024, :1024] (prefix property), loglik = sum ln|D| over the returned factor,
    and about half of the items are kept (lambda ~ U(0,1))."""
    cplx = kind == "herm_z"
    nb = 64 if cplx else 128
    loc = W.haar_kernel_bcc_torch(n, nb, 1, 0, seed=0, spectrum="uniform", complex_=cplx)
    m = 1024
    Kpre = loc[:m, :m].cpu().numpy().T.copy()  # local storage == column-major storage at world size 1
    comm = dpp.dpp_comm_init(D.unique_id(), 1, 0)
    try:
        mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        op = dpp.DPP_OP_HERM_Z if cplx else dpp.DPP_OP_HERM_D
        work = torch.empty(dpp.dpp_dist_workspace_bytes(op, n, 1), dtype=torch.uint8, device="cuda")
        fn = dpp.dpp_sample_herm_z_dist if cplx else dpp.dpp_sample_herm_d_dist
        fn(comm, n, loc, n, 0, mask, ll, None, None, work)
        torch.cuda.synchronize()
    finally:
        dpp.dpp_comm_destroy(comm)
    o = (oracle_mod.sample_herm_z if cplx else oracle_mod.sample_herm_d)(Kpre, 0, 0)
    compare_masks(mask[:m].cpu().numpy(), o)
    d = torch.diagonal(loc[:n, :n]).real if cplx else torch.diagonal(loc[:n, :n])
    assert abs(float(torch.log(d.abs()).sum()) - float(ll)) <= 1e-10 * abs(float(ll))
    assert 0.4 * n < int(mask.sum()) < 0.6 * n
