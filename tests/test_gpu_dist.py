"""GPU tests of the 1D block-column-cyclic entry points (SURVEY §8(e) mode 2; PAPER.md:579-588,
629-633 distributed): same decisions, factor and loglik as the oracle, with and without the
distributed lookahead schedule (two prioritised streams per rank, double-buffered messages).

* world size 1 over NCCL (dpp_sample_herm_{d,z}_dist);
* P = 2, 3, 4 VIRTUAL ranks on one GPU (dpp_comm_init_local + *_dist_local): the same per-step
  code with the broadcast as a device copy per receiver -- non-owner unpack, r != 0 block-cyclic
  tile addressing, message double-buffering and every rank's copy of the result;
* two real processes over NCCL when two GPUs are visible."""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import assert_factor_close, assert_loglik_close, check_decisions, compare_masks

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402
from paper_1905_00165_b200 import dist as D  # noqa: E402

# la = 2: lookahead with grouped steps (G = 3) at every size (dpp_opts_t.group_min_rows < 0; by
# default groups form only while more than 6144 / 2048 trailing rows remain, beyond these sizes)
CASES = [("herm_d", n, la) for n in (1, 128, 300, 1000, 2049) for la in (1, 0)] + \
        [("herm_z", n, la) for n in (1, 64, 200, 777) for la in (1, 0)] + \
        [("herm_d", 1000, 2), ("herm_d", 2049, 2), ("herm_d", 640, 2), ("herm_d", 1300, 2), ("herm_z", 777, 2),
         ("herm_z", 450, 2), ("herm_z", 1000, 2)]


def _dist_opts(la):
    return dpp.make_opts(lookahead=1, group_min_rows=-1) if la == 2 else dpp.make_opts(lookahead=la)


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
        opts = _dist_opts(la)
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
    # every decision (not only the prefix) against the oracle's uniforms
    check_decisions(mask.cpu().numpy(), d.cpu().numpy(), 0, 0, oracle_mod)


LOCAL_CASES = [("herm_d", n, P, la) for n, P in ((1000, 2), (2049, 3), (1300, 4), (129, 2)) for la in (1, 0, 2)] + \
              [("herm_z", n, P, la) for n, P in ((777, 2), (640, 3), (450, 4)) for la in (1, 0, 2)]


@pytest.mark.parametrize("kind,n,P,la", LOCAL_CASES)
def test_dist_virtual_ranks_match_oracle(oracle_mod, kind, n, P, la):
    """P virtual ranks on one GPU through the same run_dist step code: every rank's mask and loglik
    equal the oracle's, and the factor reassembled from all ranks' local columns equals the oracle's
    factor element by element."""
    cplx = kind == "herm_z"
    nb = 64 if cplx else 128
    K = W.haar_kernel(n, seed=n + P, complex_=cplx)
    o = (oracle_mod.sample_herm_z if cplx else oracle_mod.sample_herm_d)(K, 7, 0)
    Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
    locs = [D.to_local(Kc, n, nb, P, r) for r in range(P)]
    res = D.sample_local(locs, n, 7, complex_=cplx, opts=_dist_opts(la))
    for r in range(P):
        compare_masks(res["masks"][r].cpu().numpy(), o)
    infos = dpp.Sample(res["masks"], res["loglik"], res["info"]).info_dicts()
    if o.n_ties == 0:
        F = D.from_local(locs, n, nb, P, Kc).cpu().numpy().T
        assert_factor_close(F, o.factor, K, kind)
        for r in range(P):
            assert_loglik_close(float(res["loglik"][r]), o.loglik)
            assert infos[r]["n_kept"] == o.n_kept and infos[r]["n_ties"] == o.n_ties
            assert abs(infos[r]["min_abs_pivot"] - o.min_abs_pivot) <= 1e-9 * np.max(np.abs(K))


@pytest.mark.parametrize("paired", [False, True, 2])
def test_dist_virtual_ranks_bitwise_vs_one_rank(paired):
    """The decomposition does not change the arithmetic of any element: P = 1, 2, 4 give bit-identical
    masks, logliks and factors (each trailing element sees the same sequence of K = nb updates, or of
    K = 2 nb updates of the paired steps: the same stacked operands whether L21 is read in place or
    from the messages)."""
    n, nb = 1500, 128
    K = W.haar_kernel(n, seed=41)
    Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
    ref = None
    for P in (1, 2, 4):
        locs = [D.to_local(Kc, n, nb, P, r) for r in range(P)]
        opts = (dpp.make_opts(group=2, group_min_rows=-1) if paired == 2 else _dist_opts(2)) if paired else None
        res = D.sample_local(locs, n, 3, opts=opts)
        F = D.from_local(locs, n, nb, P, Kc)
        cur = (res["masks"][0].clone(), res["loglik"][0].clone(), torch.tril(F))
        if ref is None:
            ref = cur
        else:
            assert torch.equal(cur[0], ref[0]) and torch.equal(cur[1], ref[1]) and torch.equal(cur[2], ref[2]), P


def _nccl_worker(rank, world, uid, n, results):
    import workloads as W_
    torch.cuda.set_device(rank)
    K = W_.haar_kernel(n, seed=5)
    Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
    loc = D.to_local(Kc, n, 128, world, rank)
    comm = dpp.dpp_comm_init(uid, world, rank)
    try:
        mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        work = torch.empty(dpp.dpp_dist_workspace_bytes(dpp.DPP_OP_HERM_D, n, world), dtype=torch.uint8,
                           device="cuda")
        dpp.dpp_sample_herm_d_dist(comm, n, loc, loc.shape[1], 9, mask, ll, None, None, work)
        torch.cuda.synchronize()
        results[rank] = (mask.cpu().numpy(), float(ll), loc.cpu().numpy())
    finally:
        dpp.dpp_comm_destroy(comm)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL across processes)")
def test_dist_two_processes_nccl(oracle_mod):
    import torch.multiprocessing as mp
    n, world = 1200, 2
    uid = D.unique_id()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_nccl_worker, args=(world, uid, n, results), nprocs=world, join=True)
    K = W.haar_kernel(n, seed=5)
    o = oracle_mod.sample_herm_d(K, 9, 0)
    locs = [torch.from_numpy(results[r][2]) for r in range(world)]
    F = D.from_local(locs, n, 128, world, torch.zeros(1, dtype=torch.float64)).numpy().T
    for r in range(world):
        compare_masks(results[r][0], o)
        if o.n_ties == 0:
            assert_loglik_close(results[r][1], o.loglik)
    if o.n_ties == 0:
        assert_factor_close(F, o.factor, K, "herm_d")
