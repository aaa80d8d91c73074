import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, workloads as W, paper_1905_00165_b200 as dpp
from tests.gpu_util import from_device, to_device
oracle.build()
for n in (300, 1000):
    K = W.haar_kernel(n, seed=n + 3).astype(np.float32)
    o = oracle.sample_herm_s(K, 7, 0, tie_tol=1e-4)
    forced = torch.from_numpy(o.mask.astype(np.uint8)).cuda()
    res = {}
    for name, fl in (("tc32", 0), ("simt", 2)):
        Kc = to_device(K, "herm_s")
        s = dpp.sample("herm_s", Kc, 7, opts=dpp.make_opts(forced=forced, flags=fl))
        torch.cuda.synchronize()
        res[name] = from_device(Kc, n)
        print(n, name, "max|F - oracle| lower:", float(np.max(np.abs(np.tril(res[name] - o.factor)))), "loglik", float(s.loglik), o.loglik)
    d = np.abs(np.tril(res["tc32"] - res["simt"]))
    i, j = np.unravel_index(np.argmax(d), d.shape)
    print(n, "tc32 vs simt max", d.max(), "at", i, j, "diag diff", np.max(np.abs(np.diag(res["tc32"]) - np.diag(res["simt"]))))
    # per column block error
    print("col blocks", [float(d[:, c:c+16].max()) for c in range(0, n, 16)][:20])
