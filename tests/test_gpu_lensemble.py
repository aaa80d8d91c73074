"""GPU parity of the L-ensemble -> marginal conversion (dpp_lensemble_to_marginal_d)
against the oracle's plain definition K = I - (L + I)^{-1}: lower triangle within 1e-10 * cond(L + I),
ln det(L + I) within 1e-10 relative; the converted kernel then samples like any marginal kernel."""
import numpy as np
import pytest

from tests.gpu_util import from_device, to_device

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402


def _lens(n, seed, scale, complex_=False):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if complex_ else 0.0)
    V, _ = np.linalg.qr(G)
    lam = rng.uniform(0, scale, n)
    L = (V * lam) @ V.conj().T
    L = 0.5 * (L + L.conj().T)
    if complex_:
        L[np.diag_indices(n)] = L.diagonal().real
    return L, lam


@pytest.mark.parametrize("n,scale,cplx", [(1, 3.0, False), (100, 10.0, False), (300, 10.0, False),
                                           (1000, 50.0, False), (2049, 10.0, False), (1, 2.0, True),
                                           (200, 10.0, True), (777, 20.0, True)])
def test_lensemble_matches_oracle(oracle_mod, n, scale, cplx):
    L, lam = _lens(n, n, scale, cplx)
    K, ld = oracle_mod.lensemble_to_marginal(L)
    Lc = to_device(L, "herm_z" if cplx else "herm_d")
    logdet = dpp.lensemble_to_marginal(Lc)
    torch.cuda.synchronize()
    Kg = from_device(Lc, n)
    cond = 1.0 + float(np.max(lam))
    assert np.max(np.abs(np.tril(Kg) - np.tril(K))) <= 1e-10 * cond
    assert abs(float(logdet) - ld) <= 1e-10 * max(1.0, abs(ld))
    # the strict upper triangle is untouched
    assert np.array_equal(np.triu(Kg, 1), np.triu(L, 1))


def test_lensemble_then_sample(oracle_mod):
    """The converted kernel drives the sampler: decisions equal the oracle's on K."""
    n = 500
    L, _ = _lens(n, 7, 5.0)
    K, _ = oracle_mod.lensemble_to_marginal(L)
    Lc = to_device(L, "herm_d")
    dpp.lensemble_to_marginal(Lc)
    s = dpp.sample("herm_d", Lc, 3)
    o = oracle_mod.sample_herm_d(K, 3, 0)
    k = o.first_tie if o.n_ties else n
    assert np.array_equal(s.mask.cpu().numpy()[:k], o.mask[:k])


def test_lensemble_edge_cases(oracle_mod):
    """n = 0 gives logdet 0; L = 0 gives K = 0 and logdet 0; L = c I gives c / (1 + c) I."""
    work = torch.empty(max(dpp.dpp_lensemble_workspace_bytes(dpp.DPP_OP_HERM_D, 0), 256), dtype=torch.uint8, device="cuda")
    logdet = torch.full((), 5.0, dtype=torch.float64, device="cuda")
    A = torch.empty((1, 1), dtype=torch.float64, device="cuda")
    dpp.dpp_lensemble_to_marginal_d(0, A, 1, logdet, work)
    assert float(logdet) == 0.0
    for c in (0.0, 3.0):
        n = 200
        Lc = to_device(c * np.eye(n), "herm_d")
        ld = dpp.lensemble_to_marginal(Lc)
        K = from_device(Lc, n)
        assert np.max(np.abs(np.tril(K) - c / (1 + c) * np.eye(n))) <= 1e-14
        assert abs(float(ld) - n * np.log1p(c)) <= 1e-10 * max(1.0, n * np.log1p(c))


def test_lensemble_bench_size_residual():
    """n = 16384 (the bench's size): (I - K)(L + I) = I checked on random vectors with torch
    (harness arithmetic), and ln det(L + I) against the spectrum the kernel was built from."""
    n = 16384
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    Q, _ = torch.linalg.qr(torch.randn(n, n, generator=g, device="cuda", dtype=torch.float64))
    lam = 10.0 * torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    L = (Q * lam[None, :]) @ Q.T
    del Q
    L = 0.5 * (L + L.T)
    Lc = L.clone()  # symmetric: column-major storage == L
    logdet = dpp.lensemble_to_marginal(Lc)
    # column-major storage: K(i, l) = Lc[l, i], so the lower triangle of K is triu(Lc) transposed
    Ku = torch.triu(Lc)
    K = Ku.T + torch.triu(Lc, 1)
    x = torch.randn(n, 4, generator=g, device="cuda", dtype=torch.float64)
    z = L @ x + x
    y = z - K @ z  # (I - K)(L + I) x
    assert float((y - x).abs().max()) <= 1e-9 * float(x.abs().max()) * (1.0 + float(lam.max()))
    assert abs(float(logdet) - float(torch.log1p(lam).sum())) <= 1e-9 * float(torch.log1p(lam).sum())
