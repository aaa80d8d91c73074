"""Per-source-line warp-stall samples of one kernel in an ncu report (captured with
--warp-sampling-interval 0 --import-source on and -lineinfo builds): top lines and per-file totals.
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = hdr = None
res, tot = [], 0
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or r[2] != "-":
        continue
    try:
        n = int(r[4])
    except ValueError:
        continue
    d = dict(zip(hdr[4:], r[4:]))
    st = {k.replace("stall_", ""): int(v) for k, v in d.items()
          if k.startswith("stall_") and "Not Issued" not in k and v not in ("-", "") and int(v) > 0}
    tot += n
    res.append((n, f, int(r[0]), r[1].strip()[:70], sorted(st.items(), key=lambda x: -x[1])[:3]))
print(f"# {rep}: {tot} warp-stall samples")
byfile = {}
for n, fn, *_ in res:
    byfile[fn] = byfile.get(fn, 0) + n
print("# per file:", {k: v for k, v in sorted(byfile.items(), key=lambda x: -x[1]) if v})
for n, fn, ln, src, st in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{n:6d} {100.0 * n / max(tot, 1):5.1f}%  {fn}:{ln:<4d} {src:70s} {st}")
