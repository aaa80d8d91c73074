# split-chain / next-tile change: its bitwise test, the parity suite, C4 latency (two runs)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log; tail -3 gpurun_out/pytest_q.log
v() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[1], d.get('value'), d.get('ms_per_step'), (d.get('latency_one_stream') or {}).get('ms_per_sample'))" $1; }
for r in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/c4.json 2>/dev/null; v gpurun_out/c4.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv | grep -i "next_tile\|diag_rl"
