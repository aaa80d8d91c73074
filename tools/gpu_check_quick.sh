# panel W21 epilogue: build, the batched / guard / workload parity tests, UST and C4 benches
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
python tools/timeline.py > gpurun_out/timeline_new.json 2> gpurun_out/timeline_new.err
python tools/timeline.py 3120 0 1024 > gpurun_out/timeline_ust_new.json 2> gpurun_out/timeline_ust_new.err
python - <<'PY'
import json
for f in ("gpurun_out/timeline_new.json", "gpurun_out/timeline_ust_new.json"):
    d = json.load(open(f))
    print(f, "sample_ms", d["sample_ms"], d["sample_ms_no_events"], "no_trailing", round(d["no_trailing_ms"], 2))
    for k, v in d["stages"].items(): print("   ", k, v["launches"], round(v["ms"], 3), "top_ms", round(v["top_ms"], 4))
PY
