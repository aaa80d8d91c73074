# split-chain schedule: parity, timelines with and without it, the C4 latency
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py -m gpu -x -q 2>&1 | tail -3
python tools/timeline.py 16384 0 > gpurun_out/tl_split.json 2> gpurun_out/tl.err
python tools/timeline.py 16384 4 > gpurun_out/tl_nosplit.json 2>> gpurun_out/tl.err
python - <<'P'
import json
for f in ("gpurun_out/tl_split.json", "gpurun_out/tl_nosplit.json"):
    t = json.load(open(f))
    print(f, t["sample_ms_no_events"], t["sample_ms"], t["no_trailing_ms"], t["trailing_union_ms"])
    print("  tail steps", [(s["step"], s["step_ms"]) for s in t["steps"][-40::6]])
P
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['value'], d['ms_per_step'], d['latency_one_stream'])"
