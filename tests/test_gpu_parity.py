"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): kept sets bit-exact wherever every |u_k - d_k| > 1e-9
(tie pivots reported, prefix compared), factor entries within 1e-9 relative to max|K|,
log-likelihood within 1e-10 relative.  Sizes span several tiles and a ragged tail.
"""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import (assert_factor_close, assert_loglik_close, compare_masks, from_device,
                            to_device)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402


def _kernel(kind, n, seed, spectrum="uniform"):
    if kind == "herm_d":
        return W.haar_kernel(n, seed=seed, spectrum=spectrum)
    K = W.haar_kernel(n, seed=seed, spectrum=spectrum, complex_=True)
    return W.similarity(K, seed=seed) if kind == "lu_z" else K


def _oracle(oracle_mod, kind, K, seed=0, b=0, forced=None):
    return {"herm_d": oracle_mod.sample_herm_d, "herm_z": oracle_mod.sample_herm_z,
            "lu_z": oracle_mod.sample_lu_z}[kind](K, seed, b, forced)


def _gpu_single(kind, K, seed, opts=None, ld=None):
    n = K.shape[0]
    Kc = to_device(K, kind, ld)
    s = dpp.sample(kind, Kc, seed, opts=opts)
    torch.cuda.synchronize()
    return s, from_device(Kc, n), Kc


def _assert_info_pivots(info, o, K):
    """min_j |final pivot_j| and (LU) max_j |Im p_j| agree with the oracle's within the factor
    tolerance (the pivots are factor entries: R16)."""
    scale = float(np.max(np.abs(K))) if np.size(K) else 1.0
    assert abs(info["min_abs_pivot"] - o.min_abs_pivot) <= 1e-9 * scale, (info["min_abs_pivot"], o.min_abs_pivot)
    assert abs(info["max_abs_imag_pivot"] - o.max_abs_imag_pivot) <= 1e-9 * scale, (
        info["max_abs_imag_pivot"], o.max_abs_imag_pivot)


def test_philox_matches_oracle_and_curand(oracle_mod):
    from tests.philox_tool import curand_philox
    for seed, j0, b in [(0, 0, 0), (123456789, 1000, 7), (2**63 + 11, 2**33, 2**40 + 1)]:
        u = dpp.uniforms(seed, j0, b, 512).cpu().numpy()
        want = np.array([oracle_mod.uniform(seed, j0 + i, b) for i in range(512)])
        assert np.array_equal(u, want)
        rows = [((j0 + i) & 0xFFFFFFFF, (j0 + i) >> 32, b & 0xFFFFFFFF, b >> 32, seed & 0xFFFFFFFF, seed >> 32)
                for i in range(0, 512, 37)]
        for (c0, c1, c2, c3, k0, k1), r, i in zip(rows, curand_philox(rows), range(0, 512, 37)):
            x = (r[1] << 32) | r[0]
            assert u[i] == (2 * (x >> 12) + 1) / 2.0**53


@pytest.mark.parametrize("kind,n,nb,la", [
    ("herm_d", 1, 128, 1), ("herm_d", 2, 32, 0), ("herm_d", 127, 128, 1), ("herm_d", 128, 128, 1),
    ("herm_d", 129, 128, 1), ("herm_d", 300, 32, 1), ("herm_d", 777, 128, 1), ("herm_d", 777, 64, 0),
    ("herm_d", 1031, 128, 1),
    ("herm_z", 1, 64, 1), ("herm_z", 65, 64, 1), ("herm_z", 200, 32, 0), ("herm_z", 333, 64, 1),
    ("lu_z", 1, 64, 1), ("lu_z", 64, 64, 1), ("lu_z", 130, 32, 1), ("lu_z", 333, 64, 0), ("lu_z", 517, 64, 1),
])
def test_single_sample_parity(oracle_mod, kind, n, nb, la):
    K = _kernel(kind, n, seed=n + nb)
    seed = 1000 + n
    o = _oracle(oracle_mod, kind, K, seed)
    s, F, _ = _gpu_single(kind, K, seed, dpp.make_opts(nb=nb, lookahead=la))
    compare_masks(s.mask.cpu().numpy(), o)
    info = s.info_dicts()[0]
    assert info["n_ties"] == o.n_ties
    if o.n_ties == 0:
        assert_factor_close(F, o.factor, K, kind)
        assert_loglik_close(float(s.loglik), o.loglik)
        assert info["n_kept"] == o.n_kept
        assert info["n_out_of_range"] == o.n_out_of_range
        _assert_info_pivots(info, o, K)
    if kind != "lu_z":  # strict upper triangle never touched
        iu = np.triu_indices(n, 1)
        assert np.array_equal(F[iu], np.asarray(K)[iu])


@pytest.mark.parametrize("kind", ["herm_d", "herm_z", "lu_z"])
def test_forced_replay_parity(oracle_mod, kind):
    """Forced decisions (replay) make the factor comparable even past a tie."""
    n = 260
    K = _kernel(kind, n, seed=3)
    S = (np.random.default_rng(4).uniform(size=n) < 0.5).astype(np.uint8)
    o = _oracle(oracle_mod, kind, K, 9, forced=S)
    forced = torch.from_numpy(S).cuda()
    s, F, _ = _gpu_single(kind, K, 9, dpp.make_opts(forced=forced))
    assert np.array_equal(s.mask.cpu().numpy(), S)
    assert_factor_close(F, o.factor, K, kind)
    assert_loglik_close(float(s.loglik), o.loglik)


def test_empty_and_trivial():
    for kind in ("herm_d", "herm_z", "lu_z"):
        Kc = torch.zeros((1, 1), dtype=torch.float64 if kind == "herm_d" else torch.complex128, device="cuda")
        mask = torch.empty(1, dtype=torch.uint8, device="cuda")
        ll = torch.full((), 7.0, dtype=torch.float64, device="cuda")
        info = torch.empty(32, dtype=torch.uint8, device="cuda")
        work = dpp.workspace(kind, 0)
        getattr(dpp, f"dpp_sample_{kind}")(0, Kc, 1, 0, mask, ll, info, None, work)
        torch.cuda.synchronize()
        assert float(ll) == 0.0
        i = dpp.Sample(mask, ll, info).info_dicts()[0]
        assert i["n_kept"] == 0 and i["first_tie"] == -1
        for K, want in ((np.zeros((5, 5)), 0), (np.eye(5), 5)):
            s, F, _ = _gpu_single(kind, K, 0)
            assert int(s.mask.sum()) == want and float(s.loglik) == 0.0


def test_errors():
    Kc = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    mask = torch.empty(4, dtype=torch.uint8, device="cuda")
    ll = torch.empty((), dtype=torch.float64, device="cuda")
    work = dpp.workspace("herm_d", 4)
    with pytest.raises(dpp.DppError, match="invalid"):
        dpp.dpp_sample_herm_d(4, Kc, 3, 0, mask, ll, None, None, work)  # ld < n
    with pytest.raises(dpp.DppError, match="workspace"):
        dpp.dpp_sample_herm_d(4, Kc, 4, 0, mask, ll, None, None, work, work_bytes=16)
    with pytest.raises(dpp.DppError, match="invalid"):
        dpp.dpp_sample_herm_d(4, Kc, 4, 0, mask, ll, None, dpp.make_opts(nb=48), work)


def test_leading_dimension_and_odd_ld(oracle_mod):
    """ld > n, including an odd ld (unaligned fallback of the real update kernel)."""
    K = _kernel("herm_d", 300, seed=5)
    o = oracle_mod.sample_herm_d(K, 3, 0)
    for ld in (301, 320):
        s, F, _ = _gpu_single("herm_d", K, 3, ld=ld)
        compare_masks(s.mask.cpu().numpy(), o)
        assert_factor_close(F, o.factor, K, "herm_d")
        assert_loglik_close(float(s.loglik), o.loglik)


@pytest.mark.parametrize("kind", ["herm_d", "herm_z", "lu_z"])
def test_batched_parity(oracle_mod, kind):
    n, batch, b0, seed = 150, 6, 5, 77
    K = _kernel(kind, n, seed=8)
    Kc = to_device(K, kind)
    s = dpp.sample_batched(kind, Kc, batch, seed, b0, opts=dpp.make_opts(batch_chunk=4))
    torch.cuda.synchronize()
    masks, lls = s.mask.cpu().numpy(), s.loglik.cpu().numpy()
    for i in range(batch):
        o = _oracle(oracle_mod, kind, K, seed, b0 + i)
        compare_masks(masks[i], o)
        if o.n_ties == 0:
            assert_loglik_close(lls[i], o.loglik)
    # K is read-only in the batched call
    assert np.array_equal(from_device(Kc, n), np.asarray(K, dtype=from_device(Kc, n).dtype))
    # distinct kernels per sample (strideK > 0)
    Ks = [_kernel(kind, n, seed=20 + i) for i in range(3)]
    Kst = torch.stack([to_device(k, kind) for k in Ks])
    s2 = dpp.sample_batched(kind, Kst, 3, seed, 0)
    torch.cuda.synchronize()
    for i in range(3):
        o = _oracle(oracle_mod, kind, Ks[i], seed, i)
        compare_masks(s2.mask[i].cpu().numpy(), o)


def test_host_entry_point_matches_batched(oracle_mod):
    n, batch = 200, 3
    K = _kernel("herm_d", n, seed=11)
    Kh = torch.from_numpy(np.ascontiguousarray(K.T)).pin_memory()
    mask = torch.empty((batch, n), dtype=torch.uint8).pin_memory()
    ll = torch.empty(batch, dtype=torch.float64).pin_memory()
    info = torch.empty((batch, 32), dtype=torch.uint8).pin_memory()
    work = torch.empty(dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_D | dpp.DPP_OP_HOST, batch, n), dtype=torch.uint8,
                       device="cuda")
    dpp.dpp_sample_herm_d_host(batch, n, Kh, n, 0, 5, 0, mask, ll, info, None, work)
    for i in range(batch):
        o = oracle_mod.sample_herm_d(K, 5, i)
        compare_masks(mask[i].numpy(), o)
        assert_loglik_close(float(ll[i]), o.loglik)


@pytest.mark.parametrize("kind,n", [("herm_d", 1300), ("herm_z", 500), ("lu_z", 400)])
def test_host_async_pipelined_matches_sync(kind, n):
    """The stream-ordered host entry points (*_host_async), four calls in flight on two streams with
    two workspaces (each call's H2D overlapping the previous call's factorization), give bit for bit
    the samples of the synchronous *_host calls."""
    K = _kernel(kind, n, seed=n)
    npdt = np.float64 if kind == "herm_d" else np.complex128
    Kh = torch.from_numpy(np.ascontiguousarray(np.asarray(K, dtype=npdt).T)).pin_memory()
    op = {"herm_d": dpp.DPP_OP_HERM_D, "herm_z": dpp.DPP_OP_HERM_Z, "lu_z": dpp.DPP_OP_LU_Z}[kind] | dpp.DPP_OP_HOST
    sync_fn = getattr(dpp, f"dpp_sample_{kind}_host")
    async_fn = getattr(dpp, f"dpp_sample_{kind}_host_async")
    works = [torch.empty(dpp.dpp_workspace_bytes(op, 1, n), dtype=torch.uint8, device="cuda") for _ in range(2)]
    strs = [torch.cuda.Stream(), torch.cuda.Stream()]
    steps = 4
    ma = [torch.empty((1, n), dtype=torch.uint8).pin_memory() for _ in range(steps)]
    la = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(steps)]
    for i in range(steps):
        async_fn(1, n, Kh, n, 0, 13, i, ma[i], la[i], None, None, works[i % 2], stream=strs[i % 2])
    torch.cuda.synchronize()
    ms = torch.empty((1, n), dtype=torch.uint8).pin_memory()
    ls = torch.empty(1, dtype=torch.float64).pin_memory()
    for i in range(steps):
        sync_fn(1, n, Kh, n, 0, 13, i, ms, ls, None, None, works[0])
        assert torch.equal(ma[i], ms), i
        assert float(la[i][0]) == float(ls[0]), i


def test_blocking_and_lookahead_invariance():
    """Blocked = unblocked decisions: nb and lookahead do not change the sample."""
    K = _kernel("herm_d", 900, seed=12)
    ref = None
    for nb, la in ((32, 0), (64, 1), (128, 0), (128, 1)):
        s, F, _ = _gpu_single("herm_d", K, 21, dpp.make_opts(nb=nb, lookahead=la))
        m = s.mask.cpu().numpy()
        if ref is None:
            ref = (m, float(s.loglik), F)
        else:
            assert np.array_equal(m, ref[0])
            assert abs(float(s.loglik) - ref[1]) <= 1e-10 * abs(ref[1])
            assert np.max(np.abs(np.tril(F - ref[2]))) <= 1e-9


@pytest.mark.parametrize("kind,n,nb", [("herm_d", 2125, 128), ("herm_d", 1130, 64), ("herm_z", 1111, 64),
                                         ("herm_z", 700, 32)])
def test_split_chain_bitwise(kind, n, nb):
    """The split chain (P0 / LT on the chain stream, P1 / LR on a third stream) computes the same
    tiles with the same arithmetic as the whole panel and lookahead launches: bit-identical mask,
    loglik and factor, in place and batched (where it is off)."""
    K = _kernel(kind, n, seed=n + 3)
    a, Fa, _ = _gpu_single(kind, K, 8, dpp.make_opts(nb=nb))
    b, Fb, _ = _gpu_single(kind, K, 8, dpp.make_opts(nb=nb, flags=dpp.DPP_FLAG_NO_SPLIT_CHAIN))
    assert np.array_equal(a.mask.cpu().numpy(), b.mask.cpu().numpy())
    assert float(a.loglik) == float(b.loglik)
    assert np.array_equal(Fa, Fb)


def test_determinism_bitwise():
    K = _kernel("herm_d", 700, seed=13)
    a, Fa, _ = _gpu_single("herm_d", K, 4)
    b, Fb, _ = _gpu_single("herm_d", K, 4)
    assert np.array_equal(a.mask.cpu().numpy(), b.mask.cpu().numpy())
    assert float(a.loglik) == float(b.loglik)
    assert np.array_equal(Fa, Fb)


def test_large_parity_2048(oracle_mod):
    """Many tiles (16 at nb=128) plus a ragged tail: n = 2048 + 77."""
    n = 2125
    K = _kernel("herm_d", n, seed=14, spectrum="beta")
    o = oracle_mod.sample_herm_d(K, 0, 0)
    s, F, _ = _gpu_single("herm_d", K, 0)
    compare_masks(s.mask.cpu().numpy(), o)
    if o.n_ties == 0:
        assert_factor_close(F, o.factor, K, "herm_d")
        assert_loglik_close(float(s.loglik), o.loglik)


# Schedules and kernels selected through dpp_opts_t (the library reads no environment): the
# cp.async fallback update kernel for every GEMM, unpaired trailing updates (G = 1), the default
# pairing G = 2 engaged at every size (group_min_rows < 0; by default it starts only above 6144
# trailing rows for real 128-blocks, 8192 for LU), G = 3 and 4, and nb wider than the tile
# (256 real; 128 complex), which runs as grouped 128- (64-) wide sub-blocks.
OPT_CASES = {
    "generic": dict(flags=1),
    "no_split_chain": dict(flags=4),
    "unpaired": dict(group=1),
    "pair_all_sizes": dict(group=2, group_min_rows=-1),
    "group3": dict(group=3, group_min_rows=-1),
    "group4": dict(group=4, group_min_rows=-1),
    "nb_wide": dict(nb=-1),
}


@pytest.mark.parametrize("case", list(OPT_CASES))
@pytest.mark.parametrize("kind,n", [("herm_d", 2125), ("herm_d", 1130), ("herm_z", 555), ("lu_z", 480)])
def test_schedule_options_parity(oracle_mod, case, kind, n):
    """Each option gives the oracle's sample element by element (decisions, factor, loglik, info),
    in place and batched, at sizes where several groups form and a ragged tail stays ungrouped
    (1130: an even remainder, so the head block is taken)."""
    kw = dict(OPT_CASES[case])
    if kw.get("nb") == -1:
        kw["nb"] = 256 if kind == "herm_d" else 128
    opts = dpp.make_opts(**kw)
    K = _kernel(kind, n, seed=n)
    o = _oracle(oracle_mod, kind, K, 5)
    s, F, _ = _gpu_single(kind, K, 5, opts)
    compare_masks(s.mask.cpu().numpy(), o)
    info = s.info_dicts()[0]
    assert info["n_ties"] == o.n_ties
    if o.n_ties == 0:
        assert_factor_close(F, o.factor, K, kind)
        assert_loglik_close(float(s.loglik), o.loglik)
        _assert_info_pivots(info, o, K)
    if n < 1500:  # batched: samples b0 .. b0 + 2 of the same (read-only) kernel
        sb = dpp.sample_batched(kind, to_device(K, kind), 3, seed=5, b0=1, opts=opts)
        torch.cuda.synchronize()
        for b in range(3):
            ob = _oracle(oracle_mod, kind, K, 5, 1 + b)
            compare_masks(sb.mask[b].cpu().numpy(), ob)
            if ob.n_ties == 0:
                assert_loglik_close(float(sb.loglik[b]), ob.loglik)


def test_many_caller_streams_bitwise():
    """More caller streams (6) than the library's pool of stream pairs (4): batched and in-place
    calls rotated over them with separate workspaces give bit for bit the serial results (masks,
    loglik, factors) -- the pair reassignment keeps every call stream-ordered."""
    ns = 6
    for kind, n in (("herm_d", 700), ("lu_z", 300)):
        K = _kernel(kind, n, seed=31)
        Kd = to_device(K, kind)
        ref = []
        for i in range(ns):
            sb = dpp.sample_batched(kind, Kd, 1, seed=3, b0=i)
            Kc = to_device(K, kind)
            si = dpp.sample(kind, Kc, 3 + i)
            torch.cuda.synchronize()
            ref.append((sb.mask.clone(), sb.loglik.clone(), si.mask.clone(), si.loglik.clone(), Kc.clone()))
        strs = [torch.cuda.Stream() for _ in range(ns)]
        outs = []
        for rep in range(2):
            for i in range(ns):
                with torch.cuda.stream(strs[i]):
                    sb = dpp.sample_batched(kind, Kd, 1, seed=3, b0=i, stream=strs[i])
                    Kc = to_device(K, kind)
                    si = dpp.sample(kind, Kc, 3 + i, stream=strs[i])
                outs.append((i, sb, si, Kc))
        torch.cuda.synchronize()
        for i, sb, si, Kc in outs:
            r = ref[i]
            assert torch.equal(sb.mask, r[0]) and torch.equal(sb.loglik, r[1]), (kind, i)
            assert torch.equal(si.mask, r[2]) and torch.equal(si.loglik, r[3]), (kind, i)
            assert torch.equal(Kc, r[4]), (kind, i)


@pytest.mark.parametrize("n", [4500, 8192])
def test_host_equals_device_path(oracle_mod, n):
    """The _host entry point sees the same operations per element as the device path, so mask and
    loglik equal the batched call's bit for bit; the leading block also matches the oracle (prefix
    property)."""
    Kc = W.haar_kernel_torch(n, seed=3, spectrum="beta")
    sb = dpp.sample_batched("herm_d", Kc, 1, seed=4, b0=0)
    Kh = Kc.cpu().pin_memory()
    mh = torch.empty((1, n), dtype=torch.uint8).pin_memory()
    lh = torch.empty(1, dtype=torch.float64).pin_memory()
    work = torch.empty(dpp.dpp_workspace_bytes(dpp.DPP_OP_HERM_D | dpp.DPP_OP_HOST, 1, n), dtype=torch.uint8,
                       device="cuda")
    dpp.dpp_sample_herm_d_host(1, n, Kh, n, 0, 4, 0, mh, lh, None, None, work)
    assert np.array_equal(mh[0].numpy(), sb.mask[0].cpu().numpy())
    assert float(lh[0]) == float(sb.loglik[0])
    m = 600
    o = oracle_mod.sample_herm_d(Kc[:m, :m].cpu().numpy().T.copy(), 4, 0)
    compare_masks(mh[0].numpy()[:m], o)


@pytest.mark.parametrize("kind,n,kw", [("herm_d", 1130, {}), ("herm_d", 2125, dict(group_min_rows=-1)),
                                       ("herm_d", 700, dict(group=1)), ("herm_z", 555, {}),
                                       ("herm_z", 555, dict(group_min_rows=-1))])
def test_deferred_copy_bitwise(kind, n, kw):
    """The batched entry points on a device kernel defer the workspace copy into the first updates
    (they read K itself); the sample is bit for bit the in-place call's (which factors the caller's
    copy), for a shared kernel, a strided batch of distinct kernels, and an odd leading dimension
    (no deferral: K's columns are not 16-byte aligned).  K stays unmodified."""
    opts = dpp.make_opts(**kw)
    Ks = [_kernel(kind, n, seed=n + i) for i in range(3)]
    ref = []
    for i, K in enumerate(Ks):
        Kc = to_device(K, kind)
        si = dpp.sample(kind, Kc, 11, opts=opts)
        torch.cuda.synchronize()
        ref.append((si.mask.clone(), si.loglik.clone(), si.info.clone()))
    for ld in (n, n + 1):
        Kd = to_device(Ks[0], kind, ld)
        K0 = Kd.clone()
        sb = dpp.sample_batched(kind, Kd, 2, seed=11, b0=0, opts=opts)
        torch.cuda.synchronize()
        assert torch.equal(Kd, K0), "batched call wrote its read-only K"
        assert torch.equal(sb.mask[0], ref[0][0]) and float(sb.loglik[0]) == float(ref[0][1]), (kind, ld)
        assert torch.equal(sb.info[0], ref[0][2]), (kind, ld)
    Kst = torch.stack([to_device(K, kind) for K in Ks])  # strided batch: sample b of kernel b
    for b in range(3):
        sb = dpp.sample_batched(kind, Kst[b:b + 1], 1, seed=11, b0=0, opts=opts)
        torch.cuda.synchronize()
        assert torch.equal(sb.mask[0], ref[b][0]) and float(sb.loglik[0]) == float(ref[b][1]), (kind, b)
    sb = dpp.sample_batched(kind, Kst, 3, seed=11, b0=0, opts=opts)
    torch.cuda.synchronize()
    assert torch.equal(sb.mask[0], ref[0][0]) and float(sb.loglik[0]) == float(ref[0][1])
