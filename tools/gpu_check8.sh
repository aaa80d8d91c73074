set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r$i.json 2> gpurun_out/bench_r$i.err; done
for w in herm_z ust; do timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_r.json 2> gpurun_out/bench_${w}_r.err; done
echo done
