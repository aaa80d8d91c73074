set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fp32.py -x -q > gpurun_out/t_fp32.log 2>&1; tail -3 gpurun_out/t_fp32.log
timeout 900 python bench.py --workload herm_s > gpurun_out/bench_herm_s.json 2> gpurun_out/bench_herm_s.err
timeout 900 python bench.py --workload aztec_c > gpurun_out/bench_aztec_c.json 2> gpurun_out/bench_aztec_c.err
timeout 600 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"update_simt_kernel<float, \(bool\)1" -s 20 -c 1 -o gpurun_out/simt python bench.py --workload herm_s --steps 1 --warmup 1 > gpurun_out/ncu_simt.log 2>&1
echo done
