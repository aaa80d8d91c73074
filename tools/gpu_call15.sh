set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_fp32.py -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload herm_s > gpurun_out/bench_herm_s.json 2> gpurun_out/bench_herm_s.err
timeout 900 python bench.py --workload aztec_c --steps 2 --warmup 1 > gpurun_out/bench_aztec_c80.json 2> gpurun_out/bench_aztec_c80.err
CMD="python bench.py --workload herm_s --steps 1 --warmup 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_simt" -s 50 -c 1 -o gpurun_out/prof_simt $CMD > gpurun_out/ncu_simt.log 2>&1
echo done
