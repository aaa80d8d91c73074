"""DRAM traffic of the trailing-update launches (b) of ONE n x n sample, from an ncu CSV with
dram__bytes_read.sum and dram__bytes_write.sum per launch of update_ws_kernel (the launches of one
sample, in order: per block step  panel GEMM, lookahead column (a), trailing update (b)).

Algorithmic bytes of (b) at step k (m2 = n - nb (k + 1), jn = min(nb, m2)): one read and one write
of the lower triangle of the trailing region [jn, m2)^2 in fp64 -- the operand panels come from L2.
Usage: python tools/traffic.py launches.csv n nb > profiles/..._update_traffic.json"""
import collections
import csv
import json
import sys

path, n, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
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
# the last steps have no (b) launch once m2 <= nb; each step launches panel, (a), and (b) if m2 > jn
seq = []
i = 0
for k in range(steps):
    m2 = n - nb * (k + 1)
    jn = min(nb, m2)
    kinds = ["panel", "a"] + (["b"] if m2 > jn else [])
    for kd in kinds:
        seq.append((kd, k, m2, jn))
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
