set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
DPP_WS_VARIANT=2 timeout 900 python -m pytest tests -m gpu -q -x -k "herm_d or config3 or config1 or dist or map or lensemble" > gpurun_out/pytest_v2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v2.log
timeout 1500 python -m pytest tests -m gpu -q -x -k "alternate" > gpurun_out/pytest_alt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_alt.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
DPP_WS_VARIANT=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v2.json 2> gpurun_out/bench_v2.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v1b.json 2> gpurun_out/bench_v1b.err
DPP_WS_VARIANT=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v2b.json 2> gpurun_out/bench_v2b.err
DPP_WS_VARIANT=2 timeout 900 python bench.py --workload ust > gpurun_out/bench_ust_v2.json 2> gpurun_out/bench_ust_v2.err
DPP_WS_VARIANT=2 timeout 900 python bench.py --workload dist --n 32768 > gpurun_out/bench_dist_v2.json 2> gpurun_out/bench_dist_v2.err
timeout 900 python bench.py --workload dist --n 32768 > gpurun_out/bench_dist_v1.json 2> gpurun_out/bench_dist_v1.err
echo done
