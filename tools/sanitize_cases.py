"""Small invocations of every kernel family, for compute-sanitizer (SURVEY §4 tier T6).

Run under each tool, one per process:
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck --error-exitcode 9 \
        python tools/sanitize_cases.py [case ...]
Sizes are small (n <= 300) so racecheck finishes in minutes but still span several tiles and a
ragged tail: herm_d n = 300 (nb 128: a 44-row head block + 2 full tiles), complex n = 150 (nb 64).
Every call goes through the C ABI; results are only checked to be finite here (parity is the
tests' job).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1905_00165_b200 as dpp  # noqa: E402
import workloads as W  # noqa: E402


def _col(K):
    return torch.from_numpy(np.ascontiguousarray(K.T)).cuda()


def _finite(*ts):
    for t in ts:
        assert torch.isfinite(t.double() if not t.is_complex() else t.abs()).all(), "non-finite result"


def case_inplace():
    for kind, n, cplx in (("herm_d", 300, False), ("herm_z", 150, True)):
        for la in (0, 1):
            Kc = _col(W.haar_kernel(n, seed=3, complex_=cplx))
            s = dpp.sample(kind, Kc, 11, opts=dpp.make_opts(lookahead=la))
            torch.cuda.synchronize()
            _finite(s.loglik)
    for la in (0, 1):
        Kc = _col(W.similarity(W.haar_kernel(150, seed=3, complex_=True), seed=2))
        s = dpp.sample("lu_z", Kc, 11, opts=dpp.make_opts(lookahead=la))
        torch.cuda.synchronize()
        _finite(s.loglik)


def case_grouped():
    # paired (G = 2) and G = 3 trailing updates engaged at small n
    for g in (2, 3):
        Kc = _col(W.haar_kernel(520, seed=4))
        s = dpp.sample("herm_d", Kc, 5, opts=dpp.make_opts(group=g, group_min_rows=-1))
        torch.cuda.synchronize()
        _finite(s.loglik)
    Kc = _col(W.similarity(W.haar_kernel(270, seed=3, complex_=True), seed=2))
    s = dpp.sample("lu_z", Kc, 5, opts=dpp.make_opts(group=2, group_min_rows=-1))
    torch.cuda.synchronize()
    _finite(s.loglik)


def case_batched():
    K = _col(W.haar_kernel(300, seed=5))
    s = dpp.sample_batched("herm_d", K, 3, seed=1, b0=7)
    Kz = _col(W.haar_kernel(150, seed=5, complex_=True))
    s2 = dpp.sample_batched("herm_z", Kz, 3, seed=1)
    Kl = _col(W.similarity(W.haar_kernel(150, seed=5, complex_=True), seed=1))
    s3 = dpp.sample_batched("lu_z", Kl, 3, seed=1)
    torch.cuda.synchronize()
    _finite(s.loglik, s2.loglik, s3.loglik)


def case_generic():
    # odd ld: the cp.async fallback update kernel
    n, ld = 200, 201
    K = W.haar_kernel(n, seed=6)
    Kc = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    Kc[:, :n] = _col(K)
    s = dpp.sample("herm_d", Kc, 3)
    torch.cuda.synchronize()
    _finite(s.loglik)


def case_single():
    K = _col(W.haar_kernel(300, seed=7)).float()
    s = dpp.sample("herm_s", K, 3)
    Kz = _col(W.similarity(W.haar_kernel(150, seed=7, complex_=True), seed=3)).to(torch.complex64)
    s2 = dpp.sample("lu_c", Kz, 3)
    torch.cuda.synchronize()
    _finite(s.loglik, s2.loglik)


def case_map():
    Kc = _col(W.haar_kernel(300, seed=8))
    s = dpp.greedy_map("herm_d", Kc)
    torch.cuda.synchronize()
    _finite(s.loglik)


def case_host():
    n = 300
    K = torch.from_numpy(np.ascontiguousarray(W.haar_kernel(n, seed=9).T)).pin_memory()
    mask = torch.empty((2, n), dtype=torch.uint8).pin_memory()
    ll = torch.empty(2, dtype=torch.float64).pin_memory()
    op = dpp.DPP_OP_HERM_D | dpp.DPP_OP_HOST
    work = torch.empty(dpp.dpp_workspace_bytes(op, 2, n), dtype=torch.uint8, device="cuda")
    dpp.dpp_sample_herm_d_host(2, n, K, n, 0, 1, 0, mask, ll, None, None, work)
    _finite(ll)


def case_elementary():
    n, k = 300, 24
    K = _col(W.projection_kernel(n, k, seed=10))
    for batch in (3, 200):  # per-step kernels / the fused one-CTA-per-sample kernel
        order, ll, ties = dpp.elementary(K, k, batch=batch, seed=2)
        torch.cuda.synchronize()
        _finite(ll)


def case_lensemble():
    for cplx in (False, True):
        L = W.haar_kernel(200, seed=11, complex_=cplx) * 5.0
        Lc = _col(L)
        dpp.lensemble_to_marginal(Lc)
        torch.cuda.synchronize()
        _finite(Lc)


def case_dist():
    from paper_1905_00165_b200 import dist as D
    for cplx, n in ((False, 300), (True, 150)):
        nb = 64 if cplx else 128
        K = W.haar_kernel(n, seed=12, complex_=cplx)
        full = _col(K)
        for P in (1, 2):
            locs = [D.to_local(full, n, nb, P, r) for r in range(P)]
            res = D.sample_local(locs, n, 5, complex_=cplx)
            torch.cuda.synchronize()
            _finite(res["loglik"])


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        print(f"case {nm}: ok", flush=True)
