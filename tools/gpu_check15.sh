set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
CMD="python bench.py --workload herm_s --steps 1 --warmup 3"
timeout 900 ncu --set full --warp-sampling-interval 2 --clock-control none --import-source on --kernel-name-base demangled -k regex:"update_simt_kernel<float, \(bool\)1" -s 5 -c 1 -o gpurun_out/prof_simt2 $CMD > gpurun_out/ncu_simt.log 2>&1
echo done
