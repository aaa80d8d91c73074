set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --workload aztec > gpurun_out/bench_aztec.json 2> gpurun_out/bench_aztec.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"diag_kernel" -s 20 -c 1 -o gpurun_out/prof_diag3 $CMD > gpurun_out/ncu_diag.log 2>&1
echo done
