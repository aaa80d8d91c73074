# fp32 diag-tile change: diag A/B (fp64 bit-identity), fp32 + parity suites, herm_s and C4 bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
bash tools/gpu_diag_exp.sh 2>&1 | grep '^{'
timeout 1200 python -m pytest tests/test_gpu_fp32.py tests/test_gpu_parity.py tests/test_gpu_guard.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -3 gpurun_out/pytest_q.log
v() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d.get('value'), d.get('ms_per_step'), (d.get('latency_one_stream') or {}).get('ms_per_sample'), d.get('stages',{}).get('diag'))" $1; }
timeout 600 python bench.py --workload herm_s --steps 5 --warmup 3 > gpurun_out/hs.json 2>/dev/null; v gpurun_out/hs.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/c4.json 2>/dev/null; v gpurun_out/c4.json
