set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_d512.json 2> gpurun_out/bench_d512.err
DPP_DIAG_NT=256 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_d256.json 2> gpurun_out/bench_d256.err
for w in herm_z; do
  DPP_DIAG_NT=512 timeout 900 python bench.py --workload $w > gpurun_out/bench_${w}_d512.json 2> gpurun_out/bench_${w}_d512.err
done
timeout 900 python bench.py --workload ust > gpurun_out/bench_ust.json 2> gpurun_out/bench_ust.err
timeout 900 python bench.py --workload dist > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err
echo done
