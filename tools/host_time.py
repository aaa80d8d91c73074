"""Host enqueue time of one C4 sample against its GPU time (is the host behind the GPU anywhere?).
Usage: python tools/host_time.py [flags]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_00165_b200 as dpp  # noqa: E402
import workloads as W  # noqa: E402

n = 16384
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
Kc = W.haar_kernel_torch(n, seed=0, spectrum="beta")
opts = dpp.make_opts(nb=128, lookahead=1, flags=flags)
op = dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED
work = torch.empty(dpp.dpp_workspace_bytes(op, 1, n, opts), dtype=torch.uint8, device="cuda")
mask = torch.empty((1, n), dtype=torch.uint8, device="cuda")
ll = torch.empty(1, dtype=torch.float64, device="cuda")
for b in range(2):
    dpp.dpp_sample_herm_d_batched(1, n, Kc, n, 0, 0, b, mask, ll, None, opts, work)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for b in range(3):
    # a 20 ms spin first, so the host finishes enqueueing before the GPU starts when it can
    torch.cuda._sleep(40_000_000)
    e0.record()
    t0 = time.perf_counter()
    dpp.dpp_sample_herm_d_batched(1, n, Kc, n, 0, 0, 5 + b, mask, ll, None, opts, work)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"flags {flags}: host enqueue {1e3 * (t1 - t0):.2f} ms, GPU (after a head start) {e0.elapsed_time(e1):.3f} ms")
for b in range(3):
    torch.cuda.synchronize()
    e0.record()
    t0 = time.perf_counter()
    dpp.dpp_sample_herm_d_batched(1, n, Kc, n, 0, 0, 5 + b, mask, ll, None, opts, work)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"flags {flags}: host enqueue {1e3 * (t1 - t0):.2f} ms, GPU (no head start) {e0.elapsed_time(e1):.3f} ms")
