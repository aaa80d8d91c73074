# dist change: the dist GPU tests, guard tests, the dist / dist_z benches (and the default line's dist record)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guard.py -m gpu -q -x --timeout 900 > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -4 gpurun_out/pytest_q.log
for w in dist dist_z; do timeout 900 python bench.py --workload $w --steps 3 --warmup 2 > gpurun_out/b_$w.json 2>/dev/null
python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d.get('value'), d.get('ms_per_step'), d.get('pct_fp64_peak'))" gpurun_out/b_$w.json; done
