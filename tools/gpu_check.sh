# after a kernel change: build, the full GPU suite, smoke, C4 (three in flight + one-stream latency), UST
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
v() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d.get('value'), d.get('ms_per_step'), d.get('samples_per_s'), (d.get('latency_one_stream') or {}).get('ms_per_sample'), d.get('pct_fp64_peak'))" $1; }
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/c4.json 2>/dev/null; v gpurun_out/c4.json
timeout 600 python bench.py --workload ust --steps 3 --warmup 2 > gpurun_out/ust.json 2>/dev/null; v gpurun_out/ust.json
