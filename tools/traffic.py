"""DRAM traffic of the trailing-update launches (b) of ONE n x n sample, from an ncu CSV with
dram__bytes_read.sum and dram__bytes_write.sum per launch of update_ws_kernel (the launches of one
sample, in order: per block step  panel GEMM, lookahead column (a), trailing update (b)).

Algorithmic bytes of (b) at step k (m2 = n - nb (k + 1), jn = min(nb, m2)): one read and one write
of the lower triangle of the trailing region [jn, m2)^2 in fp64 -- the operand panels come from L2.
With paired updates (the default) an even step defers its trailing update to the next step, whose
lookahead update covers two block columns; pass the driver's DPP_PAIR_MIN_ROWS (pairing only while
the trailing size exceeds it; -1 = pairing off).
Usage: python tools/traffic.py launches.csv n nb [pair_min_rows] > profiles/..._update_traffic.json"""
import collections
import csv
import json
import sys

path, n, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
pmin = int(sys.argv[4]) if len(sys.argv) > 4 else 6144
rows = list(csv.reader(open(path)))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if "update_ws_kernel" not in d["Kernel Name"]:
        continue
    key = d["ID"]
    unit = d.get("Metric Unit", "byte")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * scale
launches = list(per.values())
steps = (n + nb - 1) // nb - 1
# replicate the driver's launch order: panel, (a), and (b) unless deferred (first step of a pair)
seq = []
pair_open = False
for k in range(steps):
    j1 = nb * (k + 1)
    m2 = n - j1
    jn0 = min(nb, m2)
    pfirst = pmin >= 0 and k % 2 == 0 and jn0 == nb and m2 - jn0 > 0 and m2 > pmin
    psecond = pmin >= 0 and k % 2 == 1 and pair_open
    jn = min(2 * nb if psecond else nb, m2)
    kinds = ["panel", "a"] + (["b"] if (m2 > jn and not pfirst) else [])
    for kd in kinds:
        seq.append((kd, k, m2, jn))
    pair_open = pfirst
launches = launches[-len(seq):]  # the last sample of the capture
meas = alg = 0.0
nb_launch = 0
for (kd, k, m2, jn), L in zip(seq, launches):
    if kd != "b":
        continue
    m = m2 - jn
    alg += 2 * 8.0 * m * (m + 1) / 2
    meas += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
    nb_launch += 1
print(json.dumps({
    "kernel": "update_ws_kernel<real, mask> trailing update (b), V1 layout (16 consumer warps), A = W21",
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, {path}",
    "n": n, "nb": nb, "launches": nb_launch,
    "measured_bytes_total": meas, "algorithmic_bytes_total": alg,
    "measured_bytes_per_launch": meas / max(nb_launch, 1),
    "ratio_measured_over_algorithmic": round(meas / alg, 4) if alg else None,
    "note": "algorithmic = one read + one write of the lower triangle of each step's trailing region (fp64); "
            "operand panels are L2-resident"}, indent=1))
