set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"diag_kernel" -s 20 -c 1 -o gpurun_out/prof_diag2 $CMD > gpurun_out/ncu_diag.log 2>&1
echo done
