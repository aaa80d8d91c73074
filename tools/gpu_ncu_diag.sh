# ncu --set full of one diag-tile launch (C4 bench, one stream) with source correlation
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --cache-control none -k regex:"diag_rl_kernel|diag_kernel" -s 40 -c 1 -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag.log 2>&1
tail -3 gpurun_out/ncu_diag.log
