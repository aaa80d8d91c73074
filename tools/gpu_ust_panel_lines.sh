# per-source-line warp stalls of one UST batched panel launch (update_ws_kernel MASK=0, 1024 samples)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
UCMD="python bench.py --workload ust --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.0' -s 7 -c 1 -o gpurun_out/prof_ust_panel_lines $UCMD > gpurun_out/ncu_ust_panel_lines.log 2>&1
tail -2 gpurun_out/ncu_ust_panel_lines.log
