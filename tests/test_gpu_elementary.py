"""GPU parity of the elementary (projection) DPP sampler (dpp_elementary_herm_d; Listing 2,
PAPER.md:514-537, reading R20) against the oracle's elementary_herm_d: identical items in the same
pivot order (before the first draw the oracle flags as a tie), loglik within 1e-10 relative; plus
ln det(K_Y), cardinality and UST spanning trees on the GPU results."""
import numpy as np
import pytest

import workloads as W
from tests.gpu_util import to_device

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1905_00165_b200 as dpp  # noqa: E402


@pytest.mark.parametrize("n,k,batch", [(1, 1, 1), (50, 7, 3), (300, 40, 5), (2000, 150, 4), (5000, 10, 2)])
def test_elementary_matches_oracle(oracle_mod, n, k, batch):
    K = W.projection_kernel(n, k, seed=n + k)
    order, ll, ties = dpp.elementary(to_device(K, "herm_d"), k, batch=batch, seed=3, b0=10)
    torch.cuda.synchronize()
    order, ll, ties = order.cpu().numpy(), ll.cpu().numpy(), ties.cpu().numpy()
    for s in range(batch):
        o = oracle_mod.elementary_herm_d(K, k, 3, 10 + s)
        m = o.first_tie if o.n_ties else k
        assert np.array_equal(order[s][:m], o.order[:m])
        if o.n_ties == 0:
            assert abs(ll[s] - o.loglik) <= 1e-10 * max(1.0, abs(o.loglik))
        Y = order[s]
        assert len(set(Y.tolist())) == k
        sign, ld = np.linalg.slogdet(K[np.ix_(Y, Y)])
        assert sign > 0 and abs(ll[s] - ld) <= 1e-9 * max(1.0, abs(ld))


def test_elementary_ust_gpu(oracle_mod):
    K = W.ust_kernel(20, 20)
    edges = W.grid_edges(20, 20)
    want = -W.log_num_spanning_trees_grid(20, 20)
    order, ll, _ = dpp.elementary(to_device(K, "herm_d"), 399, batch=8, seed=1)
    for s in range(8):
        mask = np.zeros(K.shape[0], dtype=np.uint8)
        mask[order[s].cpu().numpy()] = 1
        assert W.is_spanning_tree(400, edges, mask)
        assert abs(float(ll[s]) - want) <= 1e-9 * abs(want)


def test_elementary_edge_cases(oracle_mod):
    """k = n (K = I: every item, loglik 0), k = 0 (empty sample), batch = 0 (no work)."""
    n = 37
    K = np.eye(n)
    order, ll, ties = dpp.elementary(to_device(K, "herm_d"), n, batch=2, seed=0)
    for s in range(2):
        assert sorted(order[s].cpu().numpy().tolist()) == list(range(n))
        assert abs(float(ll[s])) <= 1e-14
    order, ll, _ = dpp.elementary(to_device(W.projection_kernel(20, 5, seed=1), "herm_d"), 0, batch=3)
    assert order.shape == (3, 0) and np.all(ll.cpu().numpy() == 0.0)
    work = torch.empty(256, dtype=torch.uint8, device="cuda")
    dpp.dpp_elementary_herm_d(0, 10, 3, to_device(np.eye(10), "herm_d"), 10, 0, 0, None, None, None, work)
    with pytest.raises(dpp.DppError):  # k > n
        dpp.dpp_elementary_workspace_bytes(1, 4, 5) or dpp.dpp_elementary_herm_d(
            1, 4, 5, to_device(np.eye(4), "herm_d"), 4, 0, 0, None, None, None, work)


def test_elementary_bench_configuration(oracle_mod):
    """The bench's configuration (n = 5000, rank 500, the paper's elementary-sampler figure): the
    first samples equal the oracle's item for item."""
    n, k = 5000, 500
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    Q, _ = torch.linalg.qr(torch.randn(n, k, generator=g, device="cuda", dtype=torch.float64))
    Kc = (Q @ Q.T).contiguous()
    order, ll, _ = dpp.elementary(Kc, k, batch=2, seed=0, b0=0)
    K = Kc.cpu().numpy()
    for s in range(2):
        o = oracle_mod.elementary_herm_d(K, k, 0, s)
        m = o.first_tie if o.n_ties else k
        assert np.array_equal(order[s].cpu().numpy()[:m], o.order[:m])
        if o.n_ties == 0:
            assert abs(float(ll[s]) - o.loglik) <= 1e-9 * abs(o.loglik)


@pytest.mark.parametrize("n,k", [(300, 40), (2000, 150)])
def test_elementary_fused_batch(oracle_mod, n, k):
    """Batches of at least one sample per SM run all k steps of a sample in one CTA (one launch):
    the samples still equal the oracle's item for item."""
    K = W.projection_kernel(n, k, seed=7 + n)
    batch = 160
    order, ll, _ = dpp.elementary(to_device(K, "herm_d"), k, batch=batch, seed=2, b0=0)
    torch.cuda.synchronize()
    order, ll = order.cpu().numpy(), ll.cpu().numpy()
    for s in (0, 1, 77, batch - 1):
        o = oracle_mod.elementary_herm_d(K, k, 2, s)
        m = o.first_tie if o.n_ties else k
        assert np.array_equal(order[s][:m], o.order[:m])
        if o.n_ties == 0:
            assert abs(ll[s] - o.loglik) <= 1e-10 * max(1.0, abs(o.loglik))
