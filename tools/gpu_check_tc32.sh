# tc32 change: fp32 tests, herm_s and aztec_c benches
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_fp32.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -2 gpurun_out/pytest_q.log
for r in 1 2; do timeout 600 python bench.py --workload herm_s --steps 5 --warmup 3 > gpurun_out/hs.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/hs.json').read().strip().splitlines()[-1]);print('herm_s', d['value'], d['ms_per_step'], d['clocks'].get('reasons'))"; done
timeout 900 python bench.py --workload aztec_c --steps 2 --warmup 1 > gpurun_out/ac.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ac.json').read().strip().splitlines()[-1]);print('aztec_c', d['variants']['tensor_3xtf32']['value'], d['variants']['tensor_3xtf32']['perfect_tilings_last_step'])"
