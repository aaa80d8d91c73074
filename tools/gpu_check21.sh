set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_c4q.json 2> gpurun_out/bench_c4q.err
timeout 600 ncu --set full --warp-sampling-interval 0 --import-source on --clock-control none --kernel-name-base demangled -k regex:"diag_kernel<double, \(bool\)1, \(int\)128, \(int\)256>" -s 30 -c 1 -o gpurun_out/diag4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_diag.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
echo done
