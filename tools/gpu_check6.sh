set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pair.json 2> gpurun_out/bench_pair.err
DPP_PAIR=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_nopair.json 2> gpurun_out/bench_nopair.err
for w in herm_z ust dist; do timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_pair.json 2> gpurun_out/bench_${w}_pair.err; done
echo done
