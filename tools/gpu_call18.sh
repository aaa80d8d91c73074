set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_b1.json 2> gpurun_out/bench_c4_b1.err
DPP_DIAG_BLOCKED=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_b0.json 2> gpurun_out/bench_c4_b0.err
timeout 900 python bench.py --workload herm_z > gpurun_out/bench_herm_z_b1.json 2> gpurun_out/bench_herm_z_b1.err
DPP_DIAG_BLOCKED=0 timeout 900 python bench.py --workload herm_z > gpurun_out/bench_herm_z_b0.json 2> gpurun_out/bench_herm_z_b0.err
timeout 900 python bench.py --workload ust > gpurun_out/bench_ust_b1.json 2> gpurun_out/bench_ust_b1.err
echo done
