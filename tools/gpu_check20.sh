set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --warp-sampling-interval 0 --import-source on --clock-control none --kernel-name-base demangled -k regex:"diag_kernel<double, \(bool\)1, \(int\)128, \(int\)256>" -s 30 -c 1 -o gpurun_out/diag python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_diag.log 2>&1
echo done
