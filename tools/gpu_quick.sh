# quick iteration: build, the parity tests, one-stream bench with every stage bracketed
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_map.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
tail -4 gpurun_out/pytest_q.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1 --prof all > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('value',d['value'],'ms',d['ms_per_step'],'lat',d['latency_one_stream']['ms_per_sample'])
for k,v in d['stages'].items(): print(k, v, 'us/launch', round(1000*v['ms']/max(v['launches'],1),1))
"
tail -3 gpurun_out/bench_q.err
