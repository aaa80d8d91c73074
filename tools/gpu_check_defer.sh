# deferred workspace copy: build, the batched / guard / workload parity tests, UST and C4 benches
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_defer.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_defer.log
tail -6 gpurun_out/pytest_defer.log
timeout 900 python bench.py --workload ust --steps 5 --warmup 3 > gpurun_out/bench_ust_defer.json 2> gpurun_out/bench_ust_defer.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/bench_c4_defer.json 2> gpurun_out/bench_c4_defer.err
python - <<'EOF'
import json
for f in ("gpurun_out/bench_ust_defer.json", "gpurun_out/bench_c4_defer.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["ms_per_step"], d.get("samples_per_s"), d.get("pct_fp64_peak"),
          (d.get("latency_one_stream") or {}).get("ms_per_sample"))
    for k, v in (d.get("stages") or {}).items(): print("  ", k, v)
EOF
