"""Launch timeline of ONE configs[3] sample (n = 16384 fp64, one caller stream, every stage bracketed
by CUDA events on the stream it is launched on -- dpp_profile_end_records), and where its time goes:
the intervals during which no trailing-update (stage 3b) kernel runs, attributed to the block steps
whose chain (diag tile -> panel -> lookahead column) they fall in.
Usage: python tools/timeline.py [n] [flags] [batch: 0 = one C4 sample; B = a UST batch] > timeline.json     (a GPU diagnostic, not a test)
"""
from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1905_00165_b200 as dpp  # noqa: E402
import workloads as W  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    B = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    if B:
        import numpy as np
        n = 3120
        Kc = torch.from_numpy(np.ascontiguousarray(W.ust_kernel(40, 40).T)).cuda()
    else:
        Kc = W.haar_kernel_torch(n, seed=0, spectrum="beta")
    nbatch = max(B, 1)
    opts = dpp.make_opts(nb=128, lookahead=1, flags=flags)
    op = dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED
    work = torch.empty(dpp.dpp_workspace_bytes(op, nbatch, n, opts), dtype=torch.uint8, device="cuda")
    mask = torch.empty((nbatch, n), dtype=torch.uint8, device="cuda")
    ll = torch.empty(nbatch, dtype=torch.float64, device="cuda")
    for b in range(2):
        dpp.dpp_sample_herm_d_batched(nbatch, n, Kc, n, 0, 0, b, mask, ll, None, opts, work)
    torch.cuda.synchronize()
    # one sample without profiling events: its time alone
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plain = []
    for b in range(3):
        t0.record()
        dpp.dpp_sample_herm_d_batched(nbatch, n, Kc, n, 0, 0, 3 + b, mask, ll, None, opts, work)
        t1.record()
        torch.cuda.synchronize()
        plain.append(t0.elapsed_time(t1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dpp.dpp_profile_begin()
    e0.record()
    dpp.dpp_sample_herm_d_batched(nbatch, n, Kc, n, 0, 0, 7, mask, ll, None, opts, work)
    e1.record()
    torch.cuda.synchronize()
    agg, rows = dpp.dpp_profile_end_records()
    total = e0.elapsed_time(e1)
    t_start = min(r[1] for r in rows)
    t_end = max(r[2] for r in rows)
    # union of the trailing-update intervals; the gaps between them
    tr = sorted((r[1], r[2]) for r in rows if r[0] == "update_trailing")
    union, gaps = 0.0, []
    lo, hi = tr[0]
    for a, b in tr[1:]:
        if a > hi:
            union += hi - lo
            gaps.append((hi, a))
            lo, hi = a, b
        else:
            hi = max(hi, b)
    union += hi - lo
    if tr[0][0] > t_start:
        gaps.insert(0, (t_start, tr[0][0]))
    if hi < t_end:
        gaps.append((hi, t_end))
    gap_ms = sum(b - a for a, b in gaps)
    # per-step chain: the diag launches mark the steps
    diag = [r for r in rows if r[0] == "diag"]
    steps = []
    for i, d in enumerate(diag):
        nxt = diag[i + 1][1] if i + 1 < len(diag) else t_end
        seg = [r for r in rows if d[1] <= r[1] < nxt]
        chain = [r for r in seg if r[0] in ("diag", "panel", "update_lookahead")]
        trail = [r for r in seg if r[0] == "update_trailing"]
        steps.append({"step": i, "t0": round(d[1] - t_start, 3), "step_ms": round(nxt - d[1], 4),
                      "diag_us": round(1e3 * (d[2] - d[1]), 1),
                      "panel_us": round(1e3 * sum(r[2] - r[1] for r in seg if r[0] == "panel"), 1),
                      "lookahead_us": round(1e3 * sum(r[2] - r[1] for r in seg if r[0] == "update_lookahead"), 1),
                      "chain_span_us": round(1e3 * (max(r[2] for r in chain) - d[1]), 1) if chain else None,
                      "trailing_us": round(1e3 * sum(r[2] - r[1] for r in trail), 1)})
    gap_by_step = [0.0] * len(diag)
    for a, b in gaps:
        for i, d in enumerate(diag):
            nxt = diag[i + 1][1] if i + 1 < len(diag) else t_end
            gap_by_step[i] += max(0.0, min(b, nxt) - max(a, d[1]))
    for s, g in zip(steps, gap_by_step):
        s["no_trailing_us"] = round(1e3 * g, 1)
    out = {"n": n, "batch": nbatch, "flags": flags, "sample_ms_no_events": [round(x, 3) for x in plain], "sample_ms": round(total, 3), "launches": len(rows),
           "trailing_union_ms": round(union, 3), "no_trailing_ms": round(gap_ms, 3),
           "trailing_tflops_while_running": round(agg["update_trailing"]["flops"] / (union / 1e3) / 1e12, 3),
           "no_trailing_ms_in_last_48_steps": round(1e3 * sum(gap_by_step[-48:]) / 1e3, 3),
           "stages": agg, "steps": steps,
           "raw_steps_88_90_112_114": [[r[0], round(1e3 * (r[1] - t_start), 1), round(1e3 * (r[2] - r[1]), 1)]
                                        for r in rows if any(diag[i][1] <= r[1] < (diag[i + 1][1] if i + 1 < len(diag) else t_end)
                                                             for i in (88, 89, 90, 112, 113, 114) if i < len(diag))]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
