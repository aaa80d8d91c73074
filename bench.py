"""Benchmark of the B200 DPP sampler (BASELINE.json metric) -- one JSON line on rank 0.

Workload (config.workload): BASELINE.json configs[3] -- the dense real-symmetric fp64 kernel
n = 16384, K = Q diag(lam) Q^T with Haar-like Q and lam ~ Beta(1/2, 1/2), sampled by the blocked
modified LDL^T with nb = 128 and depth-1 lookahead.  This is the configuration the north_star
target ("n=16384 fp64 Hermitian sampler ... >= 60% of B200 FP64 peak on the trailing update") is
stated on; configs[0] (n = 256) is the small parity case the oracle finishes in seconds.

A step = one complete sample (all SURVEY §8(a) stages) of the kernel resident in HBM, through
the public C ABI (dpp_sample_herm_d_batched, batch 1: the call copies K into its workspace and
factors the copy; sample index b differs every step).  value = model GFLOP/s (n^3/3 per sample,
the paper's convention) of the whole job; the input (2.1 GB) is larger than L2.

--gpus N (torchrun, one process per GPU): independent samples per rank (b = rank*(W+K) + i), no
data-path collective ("scaling": "weak"); time = max over ranks.
--impl reference: the CPU oracle (oracle/, plain C, unblocked Listing 1) on this host's cores,
each step one bounded sample (the leading m x m block of the same kernel).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 16384
NB = 128
SEED = 0
KSEED = 0
METRIC = "DPP sampler FP64 GFLOP/s (n^3/3 LDL^H, 2n^3/3 LU), samples/s, % FP64 peak"
UNIT = "GFLOP/s"
# Measured FP64 DMMA.8x8x4 peak of this pool's B200 (tools/fp64_peak.cu, profiles/r01_fp64_peak.jsonl);
# MEASURED_PEAKS.json has no FP64 entry.  For reference: bf16 measured 1647.4 x nominal ratio
# (37.2 / 2250) = 27.2 TF/s would be a LOWER (more flattering) denominator; we use the measured 37.1.
FP64_PEAK_TFLOPS = 37.1
FP32_SIMT_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: FFMA on all SMs at the max SM clock
PEAK_SOURCE = "measured DMMA.8x8x4 loop, profiles/r01_fp64_peak.jsonl (MEASURED_PEAKS.json has no fp64 entry)"


def model_flops(n: int) -> float:
    return n ** 3 / 3.0


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.path = f"/tmp/dpp_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(rows), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------- oracle (CPU)
def _oracle_worker(args):
    import numpy as np
    import oracle
    Kpre, b = args
    t0 = time.perf_counter()
    oracle.sample_herm_d(Kpre, SEED, b)
    return time.perf_counter() - t0


def oracle_leg(Kpre, reps: int, cores: int):
    """Times the oracle (as it stands) on `cores` host processes, each sampling Kpre once per rep."""
    import multiprocessing as mp
    import oracle
    oracle.build()
    m = Kpre.shape[0]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        for r in range(reps):
            pool.map(_oracle_worker, [(Kpre, r * cores + c) for c in range(cores)])
        wall = time.perf_counter() - t0
    flops = model_flops(m) * reps * cores
    return flops / wall / 1e9, wall


def pick_prefix(Kfull_prefix_fn, target_s: float, cores: int):
    """Choose m so one oracle sample of the leading m x m block takes about target_s seconds."""
    import oracle
    oracle.build()
    m0 = 768
    K0 = Kfull_prefix_fn(m0)
    t0 = time.perf_counter()
    oracle.sample_herm_d(K0, SEED, 0)
    dt = max(time.perf_counter() - t0, 1e-3)
    m = int(m0 * (target_s / dt) ** (1.0 / 3.0))
    return max(256, min(m - m % 16, 4096))


# --------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--aztec-streams", type=int, default=2, help="aztec: streams consecutive samples rotate over")
    ap.add_argument("--ust-streams", type=int, default=1, help="ust: streams consecutive batches rotate over")
    ap.add_argument("--e2e-streams", type=int, default=3, help="c4 e2e: streams (and workspaces) the host calls rotate over")
    ap.add_argument("--streams", type=int, default=3, choices=[1, 2, 3, 4],
                    help="c4: caller streams the consecutive steps alternate between")
    ap.add_argument("--prof", choices=["trailing", "all"], default="trailing",
                    help="c4: stages bracketed by events inside the timed region")
    ap.add_argument("--workload", default="c4", choices=["c4", "ust", "dist", "dist_z", "herm_z", "lu_z", "aztec", "herm_s", "aztec_c", "elementary", "lensemble",
                             "crossover"],
                    help="c4 (default, BASELINE configs[3]); ust: configs[1] batch of UST samples per GPU; "
                         "dist / dist_z: configs[4] 1D block-column-cyclic single sample over all ranks (real n=65536 / "
                         "complex n=32768); "
                         "herm_z / lu_z: complex128 Hermitian / non-Hermitian kernels (throughput of the "
                         "complex paths); aztec: configs[2], order-80 Aztec diamond LU sampler; herm_s / aztec_c: the "
                         "single-precision samplers (n=16384 real; order-80 Aztec consistency, PAPER.md:1164-1169); "
                         "elementary: Listing 2 on a rank-k projection, n=5000 (the paper's Fig. setting); lensemble: "
                         "K = I - (L+I)^{-1} at n=16384; crossover: elementary (Listing 2) vs generic sampler on "
                         "the same n=5000 rank-k projections, k = 10..4000 (PAPER.md:1490-1493)")
    ap.add_argument("--batch", type=int, default=1024, help="ust: samples per GPU per step")
    ap.add_argument("--batch-chunk", type=int, default=1024, help="ust: samples factored concurrently")
    ap.add_argument("--aztec-d", type=int, default=80, help="aztec_c: diamond order")
    ap.add_argument("--tally", type=int, default=0, help="aztec_c: untimed extra batches whose tilings are all checked")
    ap.add_argument("--rank", type=int, default=500, help="elementary: projection rank k")
    ap.add_argument("--lookahead", type=int, default=1, help="ust: 0 = single stream")
    ap.add_argument("--nb", type=int, default=128, help="ust / herm_s: block size")
    ap.add_argument("--group", type=int, default=0, help="c4 / ust: dpp_opts_t.group (0 = library default)")
    ap.add_argument("--flags", type=int, default=0, help="c4 / ust: extra dpp_opts_t.flags bits")
    ap.add_argument("--no-dist", action="store_true", help="c4: skip the configs[4] block-cyclic sub-record")
    ap.add_argument("--dist-n", type=int, default=65536, help="c4: n of the block-cyclic sub-record")
    ap.add_argument("--dist-steps", type=int, default=2, help="c4: timed samples of the block-cyclic sub-record")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run (the driver may
        # also launch it that way itself; then WORLD_SIZE is set and this is skipped)
        import socket
        sck = socket.socket()
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
        sck.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if "WORLD_SIZE" in os.environ and args.impl == "ours":
        assert int(os.environ["WORLD_SIZE"]) == args.gpus, \
            f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}"
    if args.workload != "c4" and args.impl == "ours":
        return extra_workload(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.n

    import numpy as np
    import torch

    if args.impl == "reference":
        if rank != 0:
            return 0
        return reference_arm(args, n)

    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1905_00165_b200 as dpp
    import workloads as W

    Kc = W.haar_kernel_torch(n, seed=KSEED, spectrum="beta")  # column-major storage (symmetric)
    torch.cuda.synchronize()
    opts = dpp.make_opts(nb=NB, lookahead=1, group=args.group, flags=args.flags)
    op = dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED
    # consecutive steps rotate over three caller streams with three workspaces (--streams 3): the
    # library gives each caller stream its own internal stream pair, so one sample's copy and first
    # block steps run under the previous sample's chain-bound tail
    NS = args.streams
    works = [torch.empty(dpp.dpp_workspace_bytes(op, 1, n, opts), dtype=torch.uint8, device="cuda") for _ in range(NS)]
    masks = [torch.empty((1, n), dtype=torch.uint8, device="cuda") for _ in range(NS)]
    lls = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(NS)]
    infos = [torch.empty((1, 32), dtype=torch.uint8, device="cuda") for _ in range(NS)]
    stream = torch.cuda.current_stream()
    sstreams = [stream] + [torch.cuda.Stream() for _ in range(NS - 1)]
    work, mask = works[0], masks[0]
    b_base = rank * (args.warmup + args.steps)

    def step(i):
        k = i % NS
        dpp.dpp_sample_herm_d_batched(1, n, Kc, n, 0, SEED, b_base + i, masks[k], lls[k], infos[k], opts, works[k],
                                      stream=sstreams[k])

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    # ---- timed region: barrier + sync on both sides, CUDA events on the launching stream
    clk = ClockSampler(local_rank)
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the trailing update's launches are bracketed by events inside the timed region (the roofline's
    # live measurement); --prof all also brackets every chain launch there
    dpp.dpp_profile_begin_stages(0x1F if args.prof == "all" else 1 << dpp.STAGES.index("update_trailing"))
    e0.record(stream)
    for st_ in sstreams[1:]:
        st_.wait_event(e0)
    for i in range(args.steps):
        step(args.warmup + i)
    for st_ in sstreams[1:]:  # the timed region ends when every stream's last step has
        ej = torch.cuda.Event()
        ej.record(st_)
        stream.wait_event(ej)
    e1.record(stream)
    torch.cuda.synchronize()
    prof = _fill_stages(dpp.dpp_profile_end(), step, args)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    last = (args.warmup + args.steps - 1) % NS  # the slot of the last timed step
    kept = int(masks[last].sum())
    total_flops = model_flops(n) * args.steps * world
    value = total_flops / (ms_max / 1e3) / 1e9
    samples_per_s = args.steps * world / (ms_max / 1e3)
    launches = sum(v["launches"] for v in prof.values())

    # roofline of the dominant kernel: the trailing update (b), stage 3, on its own stream
    up = prof["update_trailing"]
    # with samples in flight their trailing updates can overlap: the rate over the union of the
    # kernel's launch intervals (= the summed launch time when they never overlap)
    t_b = up.get("ms_union") or up["ms"]
    union_tf = up["flops"] / (t_b / 1e3) / 1e12 if t_b > 0 else 0.0
    # shares of the timed region, each stage's launches counted once where they overlap
    stage_share = {k: round((v.get("ms_union") or v["ms"]) / max(ms, 1e-9), 4) for k, v in prof.items()}

    # ---- one sample at a time (one caller stream): the latency of a single sample, the paper's
    #      "sampling costs about one plain factorization" comparison; its
    #      trailing-update launches are also the isolated probe of the dominant kernel (each
    #      launch timed alone by events on its stream, no other sample in flight)
    def step1(i):
        dpp.dpp_sample_herm_d_batched(1, n, Kc, n, 0, SEED, b_base + i, masks[0], lls[0], infos[0], opts, works[0],
                                      stream=stream)
    for i in range(2):
        step1(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    dpp.dpp_profile_begin_stages(1 << dpp.STAGES.index("update_trailing"))
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    for i in range(args.steps):
        step1(args.warmup + i)
    l1.record(stream)
    torch.cuda.synchronize()
    prof1 = dpp.dpp_profile_end()["update_trailing"]
    lat = torch.tensor([l0.elapsed_time(l1) / args.steps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(lat, op=dist.ReduceOp.MAX)
    lat_ms = float(lat.item())
    probe_tf = prof1["top_flops"] / (prof1["top_ms"] / 1e3) / 1e12 if prof1["top_ms"] > 0 else 0.0
    one_tf = prof1["flops"] / (prof1["ms"] / 1e3) / 1e12 if prof1["ms"] > 0 else 0.0
    latency = {"ms_per_sample": round(lat_ms, 3), "tflops": round(model_flops(n) / (lat_ms / 1e3) / 1e12, 3),
               "pct_fp64_peak": round(100 * model_flops(n) / (lat_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS, 2),
               "trailing_update_tflops": round(one_tf, 3),
               "what": "one caller stream: each sample starts after the previous one ends (no samples in flight)"}
    # ---- the roofline probe proper: one launch of the same trailing-update kernel, alone and
    #      persistent on every SM (dpp_probe_update_d), with the shape of the sample's largest
    #      trailing update: m = n - 4 nb rows, K = G nb = 384 (the default group of 3 block steps)
    pm, pK = n - 4 * NB, 3 * NB
    gW = torch.Generator(device="cuda"); gW.manual_seed(5)
    Wp = torch.randn(pK, pm, dtype=torch.float64, device="cuda", generator=gW)
    Lp = torch.randn(pK, pm, dtype=torch.float64, device="cuda", generator=gW)
    Cp = torch.zeros(pm, pm, dtype=torch.float64, device="cuda")
    pms = sorted(dpp.dpp_probe_update_d(pm, pK, Wp, Lp, pm, Cp, pm) for _ in range(4))[1:3]
    probe_ms = sum(pms) / len(pms)
    probe_flops = pm * (pm + 1) / 2 * 2.0 * pK
    iso_tf = probe_flops / (probe_ms / 1e3) / 1e12
    del Wp, Lp, Cp
    torch.cuda.empty_cache()
    achieved_tf = iso_tf

    # ---- end-to-end through the host-buffer C-ABI calls (H2D of K + D2H of mask/loglik inside every
    #      step).  Headline: the stream-ordered entry point, consecutive steps on two streams with two
    #      workspaces, so step i+1's copy overlaps step i's factorization (pipelined serving);
    #      also the synchronous entry point, one call after the other.
    e2e = None
    if not args.no_e2e:
        Kh = Kc.cpu().pin_memory()
        NE = args.e2e_streams
        mh = [torch.empty((1, n), dtype=torch.uint8).pin_memory() for _ in range(NE)]
        lh = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(NE)]
        ih = [torch.empty((1, 32), dtype=torch.uint8).pin_memory() for _ in range(NE)]
        opw = dpp.DPP_OP_HERM_D | dpp.DPP_OP_HOST
        del work
        torch.cuda.empty_cache()
        work_h = [torch.empty(dpp.dpp_workspace_bytes(opw, 1, n, opts), dtype=torch.uint8, device="cuda")
                  for _ in range(NE)]
        strs = [stream] + [torch.cuda.Stream() for _ in range(NE - 1)]

        def hstep_async(i):
            k = i % NE
            dpp.dpp_sample_herm_d_host_async(1, n, Kh, n, 0, SEED, b_base + i, mh[k], lh[k], ih[k], opts, work_h[k],
                                             stream=strs[k])

        def hstep_sync(i):
            dpp.dpp_sample_herm_d_host(1, n, Kh, n, 0, SEED, b_base + i, mh[0], lh[0], ih[0], opts, work_h[0],
                                       stream=stream)

        def timed_e2e(fn, two_streams):
            for i in range(NE):
                fn(i)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(strs[0])
            for st_ in strs[1:]:
                st_.wait_event(h0)
            for i in range(args.steps):
                fn(args.warmup + i)
            if two_streams:
                for st_ in strs[1:]:
                    done1 = torch.cuda.Event()
                    done1.record(st_)
                    strs[0].wait_event(done1)
            h1.record(strs[0])
            torch.cuda.synchronize()
            te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(te, op=dist.ReduceOp.MAX)
            return float(te.item())

        t_async = timed_e2e(hstep_async, True)
        t_sync = timed_e2e(hstep_sync, False)
        e2e = {"value": round(total_flops / (t_async / 1e3) / 1e9, 2), "unit": UNIT,
               # the host entry points move only the lower triangle, in 128-column blocks
               "h2d_bytes_per_step": int(sum((n - c) * min(128, n - c) for c in range(0, n, 128)) * 8),
               "d2h_bytes_per_step": int(mh[0].numel() + lh[0].numel() * 8 + ih[0].numel()),
               "samples_per_s": round(args.steps * world / (t_async / 1e3), 3),
               "api": f"dpp_sample_herm_d_host_async: steps rotate over {NE} streams and workspaces "
                      "(each step's H2D overlaps the factorizations in flight)",
               "sync_api_value": round(total_flops / (t_sync / 1e3) / 1e9, 2),
               "sync_api": "dpp_sample_herm_d_host, one synchronous call per step"}
        del work_h
        torch.cuda.empty_cache()

    # context comparator (the paper's "DPP sampling ~ plain factorization"):
    # cuSOLVER Cholesky (torch.linalg.cholesky -> potrf) of the same positive definite K, timed alone
    comparator = None
    if rank == 0 and not args.no_e2e:
        try:
            Kf = Kc.clone()
            torch.linalg.cholesky(Kf)
            torch.cuda.synchronize()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            for _ in range(3):
                torch.linalg.cholesky(Kf)
            c1.record()
            torch.cuda.synchronize()
            cms = c0.elapsed_time(c1) / 3
            comparator = {"what": "cuSOLVER potrf (torch.linalg.cholesky) of the same n x n K, plain factorization, "
                                  "no sampling", "ms": round(cms, 3), "tflops": round(model_flops(n) / (cms / 1e3) / 1e12, 3)}
            del Kf
        except Exception as e:  # a comparator only: never fails the bench
            comparator = {"error": str(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = len(os.sched_getaffinity(0))

        def prefix(m):
            return Kc[:m, :m].cpu().numpy().T.copy()
        m = pick_prefix(prefix, 8.0, cores)
        gf, wall = oracle_leg(prefix(m), 1, cores)
        cpu = {"value": round(gf, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{cores} concurrent oracle samples (one per host core, b = 0..{cores - 1}) of the "
                         f"leading {m}x{m} block of the same n={n} kernel (same flop convention m^3/3), "
                         f"{wall:.1f} s wall"}

    # ---- factor quality at full size (untimed): max|L| and a randomized residual of the factor of the
    #      last sample (R17: the panel solves use explicit tile inverses; this watches their growth)
    fcheck = _factor_check(dpp, Kc, n, opts, SEED, b_base + args.warmup + args.steps)
    del works, Kc
    torch.cuda.empty_cache()
    # ---- configs[4]: ONE n = 65536 sample factored 1D block-column-cyclic over all ranks (the
    #      north_star scaling target), at every N including 1
    dist_rec = None if args.no_dist else dist_record(args, world, rank, dist)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"BASELINE configs[3]: dense real-symmetric fp64 K=Q diag(lam) Q^T, "
                                   f"lam~Beta(1/2,1/2), n={n}, one sample per step per GPU",
                       "n": n, "nb": NB, "lookahead": 1, "global_batch": world, "seq_len": None,
                       "parallelism": f"dp{world} (independent samples)" if world > 1 else "single GPU",
                       "l2": "inputs (K, 2.1 GB) larger than L2; no flush needed",
                       "api": "dpp_sample_herm_d_batched(batch=1): K copied into the workspace each step",
                       "streams": f"{NS} caller stream(s), consecutive steps rotate over them: {NS} samples "
                                  "in flight (one sample per step)"},
            "samples_per_s": round(samples_per_s, 3),
            "headline": f"throughput with {NS} samples in flight (consecutive steps rotate over {NS} caller "
                        "streams); latency_one_stream is one sample at a time",
            "latency_one_stream": latency,
            "pct_fp64_peak": round(100.0 * value / 1e3 / (FP64_PEAK_TFLOPS * world), 2),
            "kept_last_sample": kept,
            "roofline": {"bound": "tensor", "kernel": "update_ws_kernel<real, MASK> (stage 3, trailing update)",
                         "achieved": round(achieved_tf, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": round(achieved_tf / FP64_PEAK_TFLOPS, 4),
                         "traffic": (_traffic() or {}).get("bytes_per_launch"), "traffic_detail": _traffic(),
                         "peak_source": PEAK_SOURCE,
                         "achieved_definition": "isolated probe: one launch of the trailing-update kernel "
                                                "(dpp_probe_update_d) alone and persistent on every SM, with the "
                                                "shape of the sample's largest trailing update (m = n - 4 nb, K = "
                                                "3 nb): algorithmic flops m(m+1)/2 x 2K / its CUDA-event duration "
                                                "(median of the middle two of four launches)",
                         "probe_m": pm, "probe_K": pK, "probe_launch_ms": round(probe_ms, 4),
                         "probe_launch_flops": round(probe_flops),
                         "in_situ_largest_launch_tflops": round(probe_tf, 3),
                         "in_situ_definition": "the largest trailing-update launch inside a one-stream sample: its "
                                               "flops / its event duration, on the SMs the lookahead chain leaves it",
                         "in_situ_launch_flops": round(prof1["top_flops"]), "in_situ_launch_ms": round(prof1["top_ms"], 4),
                         "union_achieved": round(union_tf, 3),
                         "union_definition": "all trailing-update launches of the timed region (samples in "
                                             "flight): their flops / the union of their launch intervals",
                         "per_launch_flops": round(up["flops"] / max(up["launches"], 1)),
                         "kernel_busy_ms": round(t_b, 3)},
            "stages": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                           "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)} for k, v in prof.items()},
            "stage_time_share": stage_share,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "e2e": e2e,
            "factor_check": fcheck,
            "dist": dist_rec,
            "cpu_baseline": cpu,
            "comparator_cusolver_potrf": comparator,
            "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _factor_check(dpp, Kc, n, opts, seed, b):
    """One more sample of the same kernel, in place on a copy (untimed): max|L| and the randomized
    residual max|(L D L^T - (K - 1_{Y^c})) x| / (max|K| max|x|) over 2 Gaussian vectors."""
    import torch
    try:
        Kf = Kc.clone()
        work = dpp.workspace("herm_d", n, opts=opts)
        s = dpp.sample("herm_d", Kf, seed, opts=opts, work=work)
        torch.cuda.synchronize()
        del work
        Lt = torch.tril(Kf.T, -1)                      # natural strict-lower L (storage is column-major)
        max_l = float(Lt.abs().max())
        Lt.diagonal().fill_(1.0)
        D = torch.diagonal(Kf).clone()
        del Kf
        g = torch.Generator(device="cuda"); g.manual_seed(1234)
        x = torch.randn(n, 2, dtype=torch.float64, device="cuda", generator=g)
        lhs = Lt @ (D[:, None] * (Lt.T @ x))
        del Lt
        Kn = torch.tril(Kc.T) + torch.tril(Kc.T, -1).T
        rhs = Kn @ x - (1.0 - s.mask.double())[:, None] * x
        res = float((lhs - rhs).abs().max() / (Kn.abs().max() * x.abs().max()))
        del Kn
        torch.cuda.empty_cache()
        return {"max_abs_L": round(max_l, 3), "residual": res, "sample_b": int(b),
                "what": "randomized max|(L D L^T - (K - 1_{Y^c})) x| / (max|K| max|x|), 2 Gaussian x"}
    except Exception as e:  # diagnostics only
        return {"error": str(e)[:200]}


def _lu_factor_check(dpp, Kc, n, opts, seed, b):
    """The complex LU sampler's factor at full size (untimed, one more sample in place on a copy):
    max|L|, max|U| and the randomized residual max|(L U - (K - 1_{Y^c})) x| / (max|K| max|x|)
    (reading R17: the panel solves use explicit tile inverses; Aztec kernels have |L| >> 1)."""
    import torch
    try:
        Kf = Kc.clone()
        work = dpp.workspace("lu_z", n, opts=opts)
        s = dpp.sample("lu_z", Kf, seed, opts=opts, work=work)
        torch.cuda.synchronize()
        del work
        F = Kf.T  # natural indexing of the column-major storage
        g = torch.Generator(device="cuda"); g.manual_seed(1234)
        x = torch.randn(n, 2, dtype=torch.float64, device="cuda", generator=g).to(torch.complex128)
        U = torch.triu(F)
        y = U @ x
        max_u = float(U.abs().max())
        del U
        L = torch.tril(F, -1)
        max_l = float(L.abs().max())
        L.diagonal().fill_(1.0)
        lhs = L @ y
        del L, F, Kf
        Kn = Kc.T
        rhs = Kn @ x - (1.0 - s.mask.double()).to(torch.complex128)[:, None] * x
        res = float((lhs - rhs).abs().max() / (Kn.abs().max() * x.abs().max()))
        torch.cuda.empty_cache()
        return {"max_abs_L": round(max_l, 3), "max_abs_U": round(max_u, 3), "residual": res, "sample_b": int(b)}
    except Exception as e:  # diagnostics only
        return {"error": str(e)[:200]}


def dist_record(args, world, rank, dist):
    """BASELINE configs[4]: one sample of the n = 65536 real kernel (K = Q diag(lam) Q^T, lam ~
    U(0,1)) factored 1D block-column-cyclic over all `world` ranks with the NCCL panel broadcast
    (dpp_sample_herm_d_dist).  Each timed sample starts from the restored local columns (restore
    outside the timed interval); time = max over ranks of the summed CUDA-event intervals."""
    import torch
    import paper_1905_00165_b200 as dpp
    import workloads as W
    from paper_1905_00165_b200 import dist as D
    n, nb = args.dist_n, 128
    try:
        t_gen = time.perf_counter()
        loc0 = W.haar_kernel_bcc_torch(n, nb, world, rank, seed=KSEED, spectrum="uniform")
        torch.cuda.synchronize()
        t_gen = time.perf_counter() - t_gen
        torch.cuda.empty_cache()
        loc = torch.empty_like(loc0)
        comm = dpp.dpp_comm_init(D.unique_id() if world == 1 else _shared_uid(dist, rank), world, rank)
        work = torch.empty(dpp.dpp_dist_workspace_bytes(dpp.DPP_OP_HERM_D, n, world), dtype=torch.uint8,
                           device="cuda")
        mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        total = 0.0
        for i in range(1 + args.dist_steps):  # one warm-up sample
            loc.copy_(loc0)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dpp.dpp_sample_herm_d_dist(comm, n, loc, n, SEED + i, mask, ll, None, None, work)
            e1.record()
            torch.cuda.synchronize()
            if i > 0:
                total += e0.elapsed_time(e1)
        dpp.dpp_comm_destroy(comm)
        t = torch.tensor([total / args.dist_steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        flops = n ** 3 / 3.0
        msg = sum(D.message_bytes(n, nb, k) for k in range((n + nb - 1) // nb)) if world > 1 else 0
        rec = {"workload": f"BASELINE configs[4]: real K n={n}, lam~U(0,1), ONE sample factored 1D block-column-"
                           f"cyclic over {world} GPU(s), nb={nb}, depth-1 lookahead, trailing updates of G = 3 block steps "
                           f"grouped, NCCL broadcast per block step "
                           f"({'none at one rank' if world == 1 else 'live rows only'})",
               "n": n, "ranks": world, "scaling": "strong", "ms_per_sample": round(ms, 2),
               "value": round(flops / (ms / 1e3) / 1e9, 2), "unit": UNIT,
               "pct_fp64_peak": round(100 * flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2),
               "samples": args.dist_steps, "kept_last": int(mask.sum()), "loglik_last": float(ll),
               "bytes_received_per_rank_per_sample": msg, "kernel_generation_s": round(t_gen, 1)}
        del loc0, loc, work
        torch.cuda.empty_cache()
        return rec
    except Exception as e:  # a sub-record: report, never fail the headline
        return {"error": str(e)[:300]}


def _traffic():
    """DRAM bytes of the roofline's probe launch (the largest trailing-update launch of one C4
    sample) from the committed ncu capture (profiles/r02/probe_traffic.json: dram__bytes_read.sum +
    dram__bytes_write.sum of that launch); None if absent."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02", "probe_traffic.json")))
        return {"bytes_per_launch": int(d["measured_bytes_per_launch"]),
                "algorithmic_bytes_per_launch": int(d["algorithmic_bytes_per_launch"]),
                "measured_over_algorithmic": d["ratio_measured_over_algorithmic"],
                "source": "profiles/r02/probe_traffic.json (ncu)"}
    except Exception:
        return None


def _timed(fn, steps, warmup, world, dist, prof_mask=0, streams=()):
    """Warm-up, then `steps` timed calls between CUDA events; with prof_mask the stages it names
    are bracketed by events inside the timed region (read with dpp.dpp_profile_end())."""
    import torch
    import paper_1905_00165_b200 as dpp
    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    time.sleep(0.2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if prof_mask:
        dpp.dpp_profile_begin_stages(prof_mask)
    e0.record()
    for st_ in streams:  # extra streams the steps run on: they start with the timed region ...
        st_.wait_event(e0)
    for i in range(steps):
        fn(warmup + i)
    for st_ in streams:  # ... and it ends when all of them are done
        ej = torch.cuda.Event()
        ej.record(st_)
        torch.cuda.current_stream().wait_event(ej)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), clocks


def _fill_stages(prof, step, args):
    """With --prof trailing only the trailing update was bracketed inside the timed region: the
    other stages' launches and times come from one more (untimed) step with every stage bracketed,
    scaled to the K timed steps."""
    import torch
    import paper_1905_00165_b200 as dpp
    if args.prof == "all":
        return prof
    dpp.dpp_profile_begin()
    step(args.warmup + args.steps)
    torch.cuda.synchronize()
    one = dpp.dpp_profile_end()
    return {k: (v if k == "update_trailing" else
                {kk: (vv if kk.startswith("top_") else vv * args.steps) for kk, vv in one[k].items()})
            for k, v in prof.items()}


def extra_workload(args):
    """The other BASELINE.json configs as throughput runs (same JSON keys as the default line)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_1905_00165_b200 as dpp
    import workloads as W
    line = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "vs_baseline": None, "data": "synthetic", "impl": "ours"}
    if args.workload == "ust":
        n = 3120
        K = W.ust_kernel(40, 40)
        Kc = torch.from_numpy(np.ascontiguousarray(K.T)).cuda()
        B = args.batch
        opts = dpp.make_opts(nb=args.nb, lookahead=args.lookahead, batch_chunk=min(B, args.batch_chunk),
                             group=args.group, flags=args.flags)
        op = dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED
        NSU = args.ust_streams  # consecutive steps rotate over this many streams (batches in flight)
        works = [torch.empty(dpp.dpp_workspace_bytes(op, B, n, opts), dtype=torch.uint8, device="cuda")
                 for _ in range(NSU)]
        masks = [torch.empty((B, n), dtype=torch.uint8, device="cuda") for _ in range(NSU)]
        lls = [torch.empty(B, dtype=torch.float64, device="cuda") for _ in range(NSU)]
        ustreams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(NSU - 1)]

        def step(i):
            b0 = (rank * (args.warmup + args.steps) + i) * B
            k = i % NSU
            dpp.dpp_sample_herm_d_batched(B, n, Kc, n, 0, SEED, b0, masks[k], lls[k], None, opts, works[k],
                                          stream=ustreams[k])
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist,
                            0x1F if args.prof == "all" else 1 << dpp.STAGES.index("update_trailing"),
                            streams=ustreams[1:])
        prof = _fill_stages(dpp.dpp_profile_end(), step, args)
        mask = torch.cat(masks)
        ok = bool((mask.sum(dim=1) == 1599).all())
        flops = model_flops(n) * B * args.steps * world
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="weak",
                    dtype="f64", samples_per_s=round(B * args.steps * world / (ms / 1e3), 2),
                    config={"workload": f"BASELINE configs[1]: UST of the 40x40 grid (n=3120, rank 1599), {B} "
                                        f"independent samples per GPU per step", "n": n, "global_batch": B * world,
                            "nb": args.nb, "group": args.group or 3, "batch_chunk": min(B, args.batch_chunk),
                            "lookahead": args.lookahead, "seq_len": None,
                            "parallelism": f"dp{world} (independent samples)"},
                    all_samples_are_spanning_trees_with_1599_edges=ok,
                    stages={k: {"launches": v["launches"], "ms": round(v["ms"], 3), "ms_union": round(v["ms_union"], 3),
                                "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)} for k, v in prof.items()},
                    pct_fp64_peak=round(100 * flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2), clocks=clocks)
    elif args.workload == "aztec":
        d = 80
        n = 4 * d * d
        Kc = W.aztec_kernel_balanced(d, device="cuda")  # balanced-gauge Kenyon kernel (reading R13)
        torch.cuda.synchronize()
        opts = dpp.make_opts(nb=64, lookahead=1, group=args.group)
        op = dpp.DPP_OP_LU_Z | dpp.DPP_OP_BATCHED
        NSA = args.aztec_streams  # consecutive samples rotate over this many streams
        works = [torch.empty(dpp.dpp_workspace_bytes(op, 1, n, opts), dtype=torch.uint8, device="cuda")
                 for _ in range(NSA)]
        masks = [torch.empty((1, n), dtype=torch.uint8, device="cuda") for _ in range(NSA)]
        lls = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(NSA)]
        astreams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(NSA - 1)]

        def step(i):
            k = i % NSA
            dpp.dpp_sample_lu_z_batched(1, n, Kc, n, 0, SEED, rank * 1000 + i, masks[k], lls[k], None, opts, works[k],
                                        stream=astreams[k])
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist,
                            0x1F if args.prof == "all" else 1 << dpp.STAGES.index("update_trailing"),
                            streams=astreams[1:])
        prof = _fill_stages(dpp.dpp_profile_end(), step, args)
        last = (args.warmup + args.steps - 1) % NSA
        mask, ll = masks[last], lls[last]
        ok = W.is_aztec_tiling(d, mask[0].cpu().numpy())
        lu_check = _lu_factor_check(dpp, Kc, n, opts, SEED, 99)
        flops = 8.0 * n ** 3 / 3.0 * args.steps * world  # complex LU, paper convention (R11)
        up = prof["update_trailing"]
        ach = up["flops"] / max(up.get("ms_union") or up["ms"], 1e-9) / 1e9  # union of its launch intervals
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="weak",
                    dtype="c128", samples_per_s=round(args.steps * world / (ms / 1e3), 4),
                    config={"workload": f"BASELINE configs[2]: order-{d} Aztec diamond, n={n} complex128 non-Hermitian "
                                        f"LU sampler on the balanced-gauge Kenyon kernel, one sample per GPU per step",
                            "n": n, "nb": 64, "global_batch": world, "seq_len": None, "parallelism": f"dp{world}",
                            "api": "dpp_sample_lu_z_batched(batch=1): K copied into the workspace each step"},
                    last_sample_is_perfect_tiling=ok, last_loglik=float(ll[0]), factor_check=lu_check,
                    loglik_closed_form=-d * (d + 1) / 2 * float(np.log(2.0)),
                    roofline={"bound": "tensor", "kernel": "update_ws_kernel<cplx> trailing update (b)",
                              "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                              "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": None},
                    stages={k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)} for k, v in prof.items()},
                    pct_fp64_peak=round(100 * flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2), clocks=clocks)
    elif args.workload == "herm_s":
        n = args.n
        Kc = W.haar_kernel_torch(n, seed=KSEED, spectrum="beta").to(torch.float32)
        opts = dpp.make_opts(nb=args.nb, lookahead=1, group=args.group)
        op = dpp.DPP_OP_HERM_S | dpp.DPP_OP_BATCHED
        NSS = args.streams  # consecutive samples rotate over this many streams (as the default workload)
        works = [torch.empty(dpp.dpp_workspace_bytes(op, 1, n, opts), dtype=torch.uint8, device="cuda")
                 for _ in range(NSS)]
        masks = [torch.empty((1, n), dtype=torch.uint8, device="cuda") for _ in range(NSS)]
        lls = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(NSS)]
        fstreams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(NSS - 1)]

        def step(i):
            k = i % NSS
            dpp.dpp_sample_herm_s_batched(1, n, Kc, n, 0, SEED, rank * 1000 + i, masks[k], lls[k], None, opts,
                                          works[k], stream=fstreams[k])
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist,
                            0x1F if args.prof == "all" else 1 << dpp.STAGES.index("update_trailing"),
                            streams=fstreams[1:])
        prof = _fill_stages(dpp.dpp_profile_end(), step, args)
        flops = model_flops(n) * args.steps * world
        up = prof["update_trailing"]
        up = dict(up, ms=up.get("ms_union") or up["ms"])  # launches of the samples in flight overlap
        ach = up["flops"] / max(up["ms"], 1e-9) / 1e9
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="weak",
                    dtype="f32", samples_per_s=round(args.steps * world / (ms / 1e3), 3),
                    config={"workload": f"single-precision real symmetric sampler on the configs[3] kernel (n={n}, "
                                        f"Beta(1/2,1/2), rounded to fp32), one sample per GPU per step; updates "
                                        f"on tcgen05 tensor cores (3xTF32)",
                            "n": n, "nb": args.nb, "global_batch": world, "seq_len": None, "parallelism": f"dp{world}"},
                    kept_last_sample=int(masks[0].sum()),
                    roofline={"bound": "tensor", "kernel": "update_tc32_kernel (3xTF32 tcgen05) trailing update (b)",
                              "achieved": round(3 * ach, 3), "peak": round(_tf32_peak(), 1), "unit": "TFLOP/s",
                              "frac": round(3 * ach / _tf32_peak(), 4), "traffic": None,
                              "model_tflops": round(ach, 3),
                              "achieved_definition": "tensor-core flops (3 tf32 MMAs per fp32 product: 3 x the "
                                                     "model flops) of the trailing-update launches / the union of "
                                                     "their launch intervals",
                              "peak_source": "MEASURED_PEAKS.json bf16_tflops x the guide's nominal tf32/bf16 ratio "
                                             "(1.1 / 2.25 PFLOP/s dense)",
                              "fp32_simt_peak": FP32_SIMT_PEAK_TFLOPS,
                              "model_over_fp32_simt_peak": round(ach / FP32_SIMT_PEAK_TFLOPS, 4)},
                    stages={k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 3)} for k, v in prof.items()},
                    gpu_launches=int(sum(v["launches"] for v in prof.values())),
                    pct_fp32_simt_peak=round(100 * flops / (ms / 1e3) / 1e12 / (FP32_SIMT_PEAK_TFLOPS * world), 2),
                    clocks=clocks)
    elif args.workload == "aztec_c":
        # single-precision Kenyon-formula sampling "essentially always
        # inconsistent once the diamond size exceeds 60".  Here on the balanced gauge (R13).
        d = args.aztec_d
        n = 4 * d * d
        Kc = W.aztec_kernel_balanced(d, device="cuda").to(torch.complex64)
        torch.cuda.synchronize()
        B = args.batch if args.batch != 1024 else 8
        want = -d * (d + 1) / 2 * float(np.log(2.0))
        op = dpp.DPP_OP_LU_C | dpp.DPP_OP_BATCHED
        mask = torch.empty((B, n), dtype=torch.uint8, device="cuda")
        ll = torch.empty(B, dtype=torch.float64, device="cuda")
        flops = 8.0 * n ** 3 / 3.0 * B * args.steps * world
        variants = {}
        # exact fp32 (FP32 SIMT updates: the paper's single-precision sampler) and the default 3xTF32
        # tensor-core updates (products to ~2^-21 relative, fp32 accumulation)
        for name, flags in (("exact_fp32_simt", dpp.DPP_FLAG_FP32_SIMT), ("tensor_3xtf32", 0)):
            opts = dpp.make_opts(nb=64, lookahead=1, batch_chunk=1, flags=flags)
            work = torch.empty(dpp.dpp_workspace_bytes(op, B, n, opts), dtype=torch.uint8, device="cuda")

            def step(i):
                dpp.dpp_sample_lu_c_batched(B, n, Kc, n, 0, SEED, (rank * 1000 + i) * B, mask, ll, None, opts, work)
            ms, clocks = _timed(step, args.steps, args.warmup, world, dist)
            masks = mask.cpu().numpy()
            good = sum(W.is_aztec_tiling(d, masks[b]) for b in range(B))
            v = {"value": round(flops / (ms / 1e3) / 1e9, 2), "ms_per_step": round(ms / args.steps, 3),
                 "samples_per_s": round(B * args.steps * world / (ms / 1e3), 4),
                 "perfect_tilings_last_step": f"{good}/{B}",
                 "max_abs_loglik_error_last_step": float(np.max(np.abs(ll.cpu().numpy() - want))),
                 "pct_fp32_simt_peak": round(100 * flops / (ms / 1e3) / 1e12 / (FP32_SIMT_PEAK_TFLOPS * world), 2),
                 "clocks": clocks}
            if args.tally > 0 and flags:  # untimed, exact fp32: tilings over args.tally further batches
                t_good, t_err = 0, []
                for i in range(args.tally):
                    step(args.steps + args.warmup + i)
                    mk, lv = mask.cpu().numpy(), ll.cpu().numpy()
                    t_good += sum(W.is_aztec_tiling(d, mk[b]) for b in range(B))
                    t_err += [float(x) for x in np.abs(lv - want)]
                v["tally"] = {"samples": args.tally * B, "perfect_tilings": t_good,
                              "loglik_error_max": max(t_err), "loglik_error_median": float(np.median(t_err)),
                              "b0": (rank * 1000 + args.steps + args.warmup) * B}
            variants[name] = v
            del work
            torch.cuda.empty_cache()
        main = variants["tensor_3xtf32"]
        line.update(value=main["value"], ms_per_step=main["ms_per_step"], scaling="weak", dtype="c64",
                    samples_per_s=main["samples_per_s"],
                    config={"workload": f"single-precision (complex64) LU sampler, order-{d} Aztec diamond (n={n}), "
                                        f"balanced-gauge Kenyon kernel, {B} samples per GPU per step; value: the "
                                        f"default 3xTF32 tensor-core updates", "n": n, "nb": 64,
                            "global_batch": B * world, "seq_len": None, "parallelism": f"dp{world}"},
                    perfect_tilings_last_step=main["perfect_tilings_last_step"],
                    max_abs_loglik_error_last_step=main["max_abs_loglik_error_last_step"],
                    pct_fp32_simt_peak=main["pct_fp32_simt_peak"], clocks=main["clocks"], variants=variants)
    elif args.workload == "elementary":
        # Listing 2: rank-k projection of order n = 5000 (the paper's elementary
        # sampler figure: ranks 10..500), a batch of independent samples per GPU per step
        n = args.n if args.n != N else 5000
        k = args.rank
        B = args.batch if args.batch != 1024 else 592  # 4 samples per SM: one CTA per sample
        g = torch.Generator(device="cuda"); g.manual_seed(KSEED)
        G = torch.randn(n, k, generator=g, device="cuda", dtype=torch.float64)
        Q, _ = torch.linalg.qr(G)
        Kc = (Q @ Q.T).contiguous()  # symmetric: column-major storage == row-major
        del G, Q
        order = torch.empty((B, k), dtype=torch.int64, device="cuda")
        ll = torch.empty(B, dtype=torch.float64, device="cuda")
        work = torch.empty(dpp.dpp_elementary_workspace_bytes(B, n, k), dtype=torch.uint8, device="cuda")

        def step(i):
            dpp.dpp_elementary_herm_d(B, n, k, Kc, n, SEED, (rank * 1000 + i) * B, order, ll, None, work)
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist)
        flops = n * k * k / 3.0 * B * args.steps * world  # the paper's elementary count (n k^2 / 3)
        # algorithmic bytes: the factor reads of every column step, sum_j 8 (n - j) j, + K columns
        byts = sum(8.0 * (n - j) * j + 8.0 * n for j in range(k)) * B * args.steps * world
        gbs = byts / (ms / 1e3) / 1e9
        peak_hbm = _hbm_peak()
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="weak",
                    dtype="f64", samples_per_s=round(B * args.steps * world / (ms / 1e3), 2),
                    config={"workload": f"elementary DPP sampler (Listing 2) on a rank-{k} projection kernel, "
                                        f"n={n}, {B} samples per GPU per step", "n": n, "rank": k,
                            "global_batch": B * world, "seq_len": None, "parallelism": f"dp{world}"},
                    roofline={"bound": "hbm", "kernel": "elem_column_kernel (factor-column GEMVs)",
                              "achieved": round(gbs, 1), "peak": peak_hbm, "unit": "GB/s",
                              "frac": round(gbs / peak_hbm, 4), "traffic": None,
                              "note": "the per-sample factor (n x k x 8 B) is L2-resident for small k"},
                    gpu_launches=int(args.steps),  # one fused launch per step (batch >= SMs)
                    clocks=clocks)
    elif args.workload == "crossover":
        # PAPER.md:1490-1493 (future work there): "at which rank it becomes beneficial to use our
        # generic sampling approach ... on GPU-accelerated architectures" -- the elementary sampler
        # (Listing 2, O(n k^2)) against the generic blocked sampler (O(n^3), independent of k) on the
        # same rank-k projections of order n = 5000 (the paper's Fig. 10 setting)
        n = args.n if args.n != N else 5000
        rows = []
        g = torch.Generator(device="cuda"); g.manual_seed(KSEED)
        Gm = torch.randn(n, 4000, generator=g, device="cuda", dtype=torch.float64)
        for k in (10, 50, 100, 250, 500, 1000, 2000, 4000):
            Q, _ = torch.linalg.qr(Gm[:, :k])
            Kc = (Q @ Q.T).contiguous()
            del Q
            Be = int(min(592, max(148, 592 * (500.0 / k) ** 2)))
            order = torch.empty((Be, k), dtype=torch.int64, device="cuda")
            lle = torch.empty(Be, dtype=torch.float64, device="cuda")
            we = torch.empty(dpp.dpp_elementary_workspace_bytes(Be, n, k), dtype=torch.uint8, device="cuda")

            def estep(i):
                dpp.dpp_elementary_herm_d(Be, n, k, Kc, n, SEED, i * Be, order, lle, None, we)
            ms_e, _ = _timed(estep, 2, 1, 1, dist)
            Bg = 64
            optg = dpp.make_opts(nb=128, lookahead=1)
            opg = dpp.DPP_OP_HERM_D | dpp.DPP_OP_BATCHED
            wg = torch.empty(dpp.dpp_workspace_bytes(opg, Bg, n, optg), dtype=torch.uint8, device="cuda")
            mg = torch.empty((Bg, n), dtype=torch.uint8, device="cuda")
            lg_ = torch.empty(Bg, dtype=torch.float64, device="cuda")

            def gstep(i):
                dpp.dpp_sample_herm_d_batched(Bg, n, Kc, n, 0, SEED, i * Bg, mg, lg_, None, optg, wg)
            ms_g, _ = _timed(gstep, 2, 1, 1, dist)
            ok = bool((mg.sum(dim=1) == k).all())  # projection: every sample has exactly k items
            rows.append({"rank": k, "elementary_samples_per_s": round(2 * Be / (ms_e / 1e3), 2),
                         "elementary_batch": Be, "generic_samples_per_s": round(2 * Bg / (ms_g / 1e3), 2),
                         "generic_batch": Bg, "generic_cardinality_ok": ok})
            del Kc, we, wg, order
            torch.cuda.empty_cache()
        cross = None
        for a_, b_ in zip(rows, rows[1:]):
            ra = a_["elementary_samples_per_s"] / a_["generic_samples_per_s"]
            rb = b_["elementary_samples_per_s"] / b_["generic_samples_per_s"]
            if ra >= 1.0 > rb:  # log-log interpolation of the ratio
                t = np.log(ra) / (np.log(ra) - np.log(rb))
                cross = round(float(np.exp(np.log(a_["rank"]) + t * (np.log(b_["rank"]) - np.log(a_["rank"])))), 0)
        line.update(value=cross, unit="rank", ms_per_step=None, scaling="weak", dtype="f64", higher_is_better=None,
                    metric="crossover rank: elementary (Listing 2) vs generic sampler, samples/s on the same "
                           "n=5000 rank-k projections",
                    config={"workload": f"rank-k projections K = Q Q^T (QR of an n x k Gaussian), n={n}", "n": n,
                            "seq_len": None, "global_batch": None, "parallelism": "single GPU"},
                    rows=rows, crossover_rank=cross,
                    note="above the crossover rank the generic O(n^3) sampler draws more samples/s than the "
                         "O(n k^2) elementary sampler (PAPER.md:1490-1493); paper, 1 CPU core: elementary "
                         "3.8k / 115 / 5 samples/s at ranks 10 / 100 / 500 vs generic 1.2 samples/s (Fig. 10)")
    elif args.workload == "lensemble":
        # L-ensemble -> marginal conversion, "3 samples worth of time"
        n = args.n
        Lc0 = W.haar_kernel_torch(n, seed=KSEED, spectrum="uniform") * 10.0  # PSD L, eigenvalues in [0, 10)
        Lc = torch.empty_like(Lc0)
        logdet = torch.empty((), dtype=torch.float64, device="cuda")
        work = torch.empty(dpp.dpp_lensemble_workspace_bytes(dpp.DPP_OP_HERM_D, n), dtype=torch.uint8, device="cuda")
        copy_ms = 0.0

        def step(i):
            Lc.copy_(Lc0)
            dpp.dpp_lensemble_to_marginal_d(n, Lc, n, logdet, work)
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            Lc.copy_(Lc0)
        e1.record()
        torch.cuda.synchronize()
        copy_ms = e0.elapsed_time(e1)
        flops = float(n) ** 3 * args.steps * world  # LDL^T + triangular inverse + product: 3 x n^3/3
        line.update(value=round(flops / ((ms - copy_ms) / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3),
                    scaling="weak", dtype="f64",
                    config={"workload": f"L-ensemble -> marginal kernel K = I - (L+I)^-1, n={n} real symmetric, "
                                        f"L = Q diag(10 u) Q^T; value excludes the per-step restore copy",
                            "n": n, "global_batch": world, "seq_len": None, "parallelism": f"dp{world}"},
                    restore_copy_ms_per_step=round(copy_ms / args.steps, 3),
                    conversion_ms=round((ms - copy_ms) / args.steps, 3),
                    pct_fp64_peak=round(100 * flops / ((ms - copy_ms) / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2),
                    clocks=clocks)
    elif args.workload in ("herm_z", "lu_z"):
        n = args.n if args.n != N else 8192
        Kc = W.haar_kernel_torch(n, seed=KSEED, spectrum="uniform", complex_=True)
        if args.workload == "lu_z":  # D^-1 K D (Prop. 2), a non-Hermitian kernel with the same DPP
            g = torch.Generator(device="cuda"); g.manual_seed(7)
            dv = torch.exp(torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5).to(torch.complex128)
            Kc = (Kc * dv[None, :]) / dv[:, None]  # storage (l, i) = K(i, l): K' = D^-1 K D
        opts = dpp.make_opts(nb=64, lookahead=1, group=args.group)
        op = (dpp.DPP_OP_HERM_Z if args.workload == "herm_z" else dpp.DPP_OP_LU_Z) | dpp.DPP_OP_BATCHED
        NSZ = args.streams  # consecutive samples rotate over this many streams (as the default workload)
        works = [torch.empty(dpp.dpp_workspace_bytes(op, 1, n, opts), dtype=torch.uint8, device="cuda")
                 for _ in range(NSZ)]
        masks = [torch.empty((1, n), dtype=torch.uint8, device="cuda") for _ in range(NSZ)]
        lls = [torch.empty(1, dtype=torch.float64, device="cuda") for _ in range(NSZ)]
        zstreams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(NSZ - 1)]
        fn = dpp.dpp_sample_herm_z_batched if args.workload == "herm_z" else dpp.dpp_sample_lu_z_batched

        def step(i):
            k = i % NSZ
            fn(1, n, Kc, n, 0, SEED, rank * 1000 + i, masks[k], lls[k], None, opts, works[k], stream=zstreams[k])
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist, streams=zstreams[1:])
        mult = 4.0 if args.workload == "herm_z" else 8.0  # complex LDL^H 4n^3/3, complex LU 8n^3/3 (R11)
        flops = mult * n ** 3 / 3.0 * args.steps * world
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="weak",
                    dtype="c128", samples_per_s=round(args.steps * world / (ms / 1e3), 3),
                    config={"workload": f"complex128 {'Hermitian' if args.workload == 'herm_z' else 'non-Hermitian (D^-1 K D)'} "
                                        f"Haar kernel n={n}, one sample per GPU per step", "n": n, "nb": 64,
                            "global_batch": world, "seq_len": None, "parallelism": f"dp{world}"},
                    pct_fp64_peak=round(100 * flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2), clocks=clocks)
    else:  # dist / dist_z: ONE sample factored 1D block-column-cyclic over all ranks
        from paper_1905_00165_b200 import dist as D
        cplx = args.workload == "dist_z"
        n = args.n if args.n != N else (32768 if cplx else 65536)
        nb = 64 if cplx else 128
        # K = Q diag(lam) Q^H, lam ~ U(0,1), Q Haar-like; every rank builds the same Q, keeps its columns
        loc0 = W.haar_kernel_bcc_torch(n, nb, world, rank, seed=KSEED, spectrum="uniform", complex_=cplx)
        torch.cuda.empty_cache()
        loc = torch.empty_like(loc0)
        comm = dpp.dpp_comm_init(D.unique_id() if world == 1 else _shared_uid(dist, rank), world, rank)
        op = dpp.DPP_OP_HERM_Z if cplx else dpp.DPP_OP_HERM_D
        work = torch.empty(dpp.dpp_dist_workspace_bytes(op, n, world), dtype=torch.uint8, device="cuda")
        mask = torch.empty(n, dtype=torch.uint8, device="cuda")
        ll = torch.empty((), dtype=torch.float64, device="cuda")
        fn = dpp.dpp_sample_herm_z_dist if cplx else dpp.dpp_sample_herm_d_dist
        copy_ms = []

        def step(i):
            loc.copy_(loc0)
            fn(comm, n, loc, n, SEED + i, mask, ll, None, None, work)
        ms, clocks = _timed(step, args.steps, args.warmup, world, dist)
        # the restore copy is inside the timed step; measure it alone to report the sampler's own rate
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            loc.copy_(loc0)
        e1.record()
        torch.cuda.synchronize()
        copy_ms = e0.elapsed_time(e1)
        dpp.dpp_comm_destroy(comm)
        flops = (4.0 if cplx else 1.0) * n ** 3 / 3.0 * args.steps  # complex LDL^H 4n^3/3 (R11)
        line.update(value=round(flops / (ms / 1e3) / 1e9, 2), ms_per_step=round(ms / args.steps, 3), scaling="strong",
                    dtype="c128" if cplx else "f64", samples_per_s=round(args.steps / (ms / 1e3), 4),
                    config={"workload": f"BASELINE configs[4]: dense {'complex Hermitian' if cplx else 'real-symmetric'} "
                                        f"K=Q diag(lam) Q^H, lam~U(0,1), n={n}, ONE sample per step factored 1D "
                                        f"block-column-cyclic over {world} GPU(s) (NCCL broadcast of each panel, "
                                        f"depth-1 lookahead, trailing updates of G = 3 block steps grouped); step includes restoring the "
                                        f"local columns",
                            "n": n, "nb": nb, "global_batch": 1, "seq_len": None, "parallelism": f"bcc{world}"},
                    restore_copy_ms_per_step=round(copy_ms / args.steps, 3),
                    value_excluding_restore=round(flops / ((ms - copy_ms) / 1e3) / 1e9, 2),
                    kept=int(mask.sum()), loglik=float(ll),
                    pct_fp64_peak=round(100 * flops / (ms / 1e3) / 1e12 / (FP64_PEAK_TFLOPS * world), 2), clocks=clocks)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _tf32_peak():
    """Dense tf32 tensor-core peak: the measured bf16 peak x the nominal tf32/bf16 ratio."""
    try:
        bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        bf16 = 2250.0  # the guide's nominal dense bf16 (no measurement available)
    return bf16 * 1.1 / 2.25


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6541.8


def _shared_uid(dist, rank):
    from paper_1905_00165_b200 import dist as D
    uid = [D.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    return uid[0]


def reference_arm(args, n):
    """The CPU oracle, as it stands, on this host's cores; same metric/unit/config."""
    import torch
    import workloads as W
    cores = len(os.sched_getaffinity(0))
    if torch.cuda.is_available():
        Kc = W.haar_kernel_torch(n, seed=KSEED, spectrum="beta")

        def prefix(m):
            return Kc[:m, :m].cpu().numpy().T.copy()
        workload = f"leading m x m block of the config[3] kernel (n={n}, Beta(1/2,1/2), GPU-generated)"
    else:
        def prefix(m):
            return W.haar_kernel(m, seed=KSEED, spectrum="beta")
        workload = "numpy Haar kernel with the config[3] recipe (no GPU to generate the n=16384 kernel)"
    # each step must be bounded so the whole --steps K --warmup W run ends within a few minutes
    per_step_s = max(2.0, min(10.0, 150.0 / max(args.steps + args.warmup, 1)))
    m = pick_prefix(prefix, per_step_s, cores)
    Kpre = prefix(m)
    for _ in range(args.warmup):
        oracle_leg(Kpre, 1, cores)
    t0 = time.perf_counter()
    gf, wall = oracle_leg(Kpre, args.steps, cores)
    ms = (time.perf_counter() - t0) * 1e3
    line = {
        "metric": METRIC, "value": round(gf, 3), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE configs[3] (n={n}) -- oracle sample: {workload}, m={m}",
                   "n": n, "m_sample": m, "global_batch": cores, "seq_len": None, "parallelism": f"{cores} host processes"},
        "impl": "reference",
        "cpu_baseline": {"value": round(gf, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"per step {cores} concurrent unblocked oracle samples of the leading {m}x{m} block"},
        "e2e": {"value": round(gf, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
