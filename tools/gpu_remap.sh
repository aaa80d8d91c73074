# update-kernel consumer loop changes: build, parity tests, probe, UST / C4 / complex benches
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for a in "15872 128" "15872 384" "15872 3072" "8192 384" "4096 384"; do python tools/probe.py $a; done 2>&1 | tee gpurun_out/probe_k_sweep2.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_lensemble.py tests/test_gpu_dist.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_remap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_remap.log
tail -4 gpurun_out/pytest_remap.log
timeout 900 python bench.py --workload ust --steps 5 --warmup 3 > gpurun_out/bench_ust_remap.json 2> gpurun_out/bench_ust_remap.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/bench_c4_remap.json 2> gpurun_out/bench_c4_remap.err
timeout 900 python bench.py --workload herm_z --steps 5 --warmup 3 > gpurun_out/bench_hz_remap.json 2> gpurun_out/bench_hz_remap.err
timeout 900 python bench.py --workload aztec --steps 3 --warmup 2 > gpurun_out/bench_az_remap.json 2> gpurun_out/bench_az_remap.err
python - <<'PY'
import json
for f in ("ust", "c4", "hz", "az"):
    f = "gpurun_out/bench_%s_remap.json" % f
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["ms_per_step"], d.get("samples_per_s"), d.get("pct_fp64_peak"),
          (d.get("latency_one_stream") or {}).get("ms_per_sample"), (d.get("roofline") or {}).get("frac"))
PY
