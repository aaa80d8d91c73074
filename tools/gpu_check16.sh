set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload ust --nb 64 > gpurun_out/bench_ust64.json 2> gpurun_out/bench_ust64.err
timeout 900 python bench.py --workload ust --nb 64 --batch-chunk 512 > gpurun_out/bench_ust64c.json 2> gpurun_out/bench_ust64c.err
timeout 900 python bench.py --workload ust --batch-chunk 512 > gpurun_out/bench_ust128c.json 2> gpurun_out/bench_ust128c.err
echo done
