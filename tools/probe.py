"""The roofline probe alone (for ncu): one launch of the trailing-update kernel on every SM with the
shape of the C4 sample's largest trailing update (m = 16384 - 512, K = 384), after one warm-up launch.
Usage: python tools/probe.py [m] [K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_00165_b200 as dpp  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384 - 512
K = int(sys.argv[2]) if len(sys.argv) > 2 else 384
g = torch.Generator(device="cuda"); g.manual_seed(5)
W = torch.randn(K, m, dtype=torch.float64, device="cuda", generator=g)
L = torch.randn(K, m, dtype=torch.float64, device="cuda", generator=g)
C = torch.zeros(m, m, dtype=torch.float64, device="cuda")
for _ in range(2):
    ms = dpp.dpp_probe_update_d(m, K, W, L, m, C, m)
flops = m * (m + 1) / 2 * 2.0 * K
print(f"m {m} K {K}: {ms:.4f} ms, {flops / ms / 1e9:.3f} TF/s, algorithmic C bytes {m * (m + 1) / 2 * 16:.4e}")
