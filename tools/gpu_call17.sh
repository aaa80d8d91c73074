set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload ust > gpurun_out/bench_ust_la1.json 2> gpurun_out/bench_ust_la1.err
timeout 900 python bench.py --workload ust --lookahead 0 > gpurun_out/bench_ust_la0.json 2> gpurun_out/bench_ust_la0.err
timeout 900 python bench.py --workload ust --lookahead 0 --batch-chunk 1024 > gpurun_out/bench_ust_la0c.json 2> gpurun_out/bench_ust_la0c.err
echo done
