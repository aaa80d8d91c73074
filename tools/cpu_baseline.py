"""The BASELINE.md CPU-baseline plan (SURVEY §8(d) timing protocol), run on the GPU box's host.

* single-threaded oracle (pinned to one core) for herm_d at n in {256, 1024, 2048, 3120, 4096}
  and lu_z at n in {400, 1600, 3200} (3200 instead of the plan's 6400: ~8x cheaper, and the n^3
  fit below uses the two largest sizes either way);
* t = c n^3 fitted on the two largest sizes of each kind and extrapolated to C3 (Aztec lu_z
  n = 25600), C4 (herm_d n = 16384) and C5 (herm_d n = 65536, herm_z n = 32768 via the herm_d fit
  x 4 complex flops) -- labelled EXTRAPOLATED;
* C2 (UST 40x40, n = 3120): samples/s with one oracle process per host core.
The oracle is the test oracle (oracle/, plain C, unblocked Listing 1), timed as it stands.
Writes one JSON document to stdout.
Usage: python tools/cpu_baseline.py [--quick]
"""
from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def _flops(kind, n):
    return {"herm_d": n ** 3 / 3.0, "herm_z": 4.0 * n ** 3 / 3.0, "lu_z": 8.0 * n ** 3 / 3.0}[kind]


def _kernel(kind, n):
    if kind == "herm_d":
        return W.haar_kernel(n, seed=0, spectrum="beta")
    return W.similarity(W.haar_kernel(n, seed=0, complex_=True), seed=0)


def _time_one(kind, K, core):
    # the kernel is built by the parent (numpy's LAPACK threads must not be pinned to one core)
    os.sched_setaffinity(0, {core})
    n = K.shape[0]
    fn = oracle.sample_herm_d if kind == "herm_d" else oracle.sample_lu_z
    fn(K, 0, 0) if n <= 1024 else None  # warm (small sizes only)
    t0 = time.perf_counter()
    fn(K, 0, 1)
    return time.perf_counter() - t0


def _ust_worker(args):
    K, b0, count = args
    t0 = time.perf_counter()
    for b in range(b0, b0 + count):
        oracle.sample_herm_d(K, 0, b)
    return time.perf_counter() - t0


def main():
    quick = "--quick" in sys.argv
    oracle.build()
    cores = sorted(os.sched_getaffinity(0))
    core = cores[-1]
    out = {"what": "CPU oracle (oracle/, plain C, one thread per process, unblocked Listing 1, fp64)",
           "host_cores": len(cores), "cpu": _cpu_name(), "single_core": [], "fits": {}, "extrapolated": {}}
    plan = {"herm_d": [256, 1024, 2048, 3120, 4096], "lu_z": [400, 1600, 3200]}
    if quick:
        plan = {"herm_d": [256, 512], "lu_z": [200, 400]}
    for kind, ns in plan.items():
        for n in ns:
            K = _kernel(kind, n)
            with mp.get_context("fork").Pool(1) as pool:
                t = pool.apply(_time_one, (kind, K, core))
            out["single_core"].append({"kind": kind, "n": n, "seconds": round(t, 4),
                                       "gflops": round(_flops(kind, n) / t / 1e9, 4), "core": core})
            print(f"# {kind} n={n}: {t:.3f} s", file=sys.stderr, flush=True)
        a, b = [r for r in out["single_core"] if r["kind"] == kind][-2:]
        c = (a["seconds"] / a["n"] ** 3 + b["seconds"] / b["n"] ** 3) / 2.0
        out["fits"][kind] = {"c_seconds_per_n3": c, "from_n": [a["n"], b["n"]]}
    ch, cz = out["fits"]["herm_d"]["c_seconds_per_n3"], out["fits"]["lu_z"]["c_seconds_per_n3"]
    for name, kind, n, c in (("C4 herm_d n=16384", "herm_d", 16384, ch), ("C5a herm_d n=65536", "herm_d", 65536, ch),
                             ("C5b herm_z n=32768 (herm_d fit x 4)", "herm_z", 32768, 4 * ch),
                             ("C3 Aztec lu_z n=25600", "lu_z", 25600, cz)):
        t = c * n ** 3
        out["extrapolated"][name] = {"seconds_EXTRAPOLATED": round(t, 1),
                                     "gflops_EXTRAPOLATED": round(_flops(kind, n) / t / 1e9, 3), "cores": 1}
    # C2: UST 40x40 samples/s, one oracle process per host core
    K = W.ust_kernel(40, 40)
    per = 1 if quick else 2
    with mp.get_context("fork").Pool(len(cores)) as pool:
        t0 = time.perf_counter()
        pool.map(_ust_worker, [(K, i * per, per) for i in range(len(cores))])
        wall = time.perf_counter() - t0
    out["ust_40x40_all_cores"] = {"samples": per * len(cores), "seconds": round(wall, 2),
                                  "samples_per_s": round(per * len(cores) / wall, 3), "processes": len(cores),
                                  "gflops": round(per * len(cores) * _flops("herm_d", 3120) / wall / 1e9, 3)}
    print(json.dumps(out, indent=1))


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


if __name__ == "__main__":
    main()
