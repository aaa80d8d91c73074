python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_workloads.py tests/test_gpu_dist.py -m gpu -x -q 2>&1 | tail -2
python tools/host_time.py 0 | tail -3
for m in 4096 15872; do python tools/probe.py $m 384; done
timeout 900 python bench.py --workload ust --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ust', d['value'], d['samples_per_s'], d['pct_fp64_peak'])"
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['value'], d['ms_per_step'], d['roofline']['frac'], d['latency_one_stream']['ms_per_sample'])"
