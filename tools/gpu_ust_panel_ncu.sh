# ncu of UST batch panel launches (update_ws_kernel MASK=0, K = 128, 1024 samples) and one grouped trailing launch
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --workload ust --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.0' -s 6 -c 2 -o gpurun_out/prof_ust_panel $CMD > gpurun_out/ncu_ust_panel.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.1' -s 4 -c 2 -o gpurun_out/prof_ust_upd $CMD > gpurun_out/ncu_ust_upd.log 2>&1
tail -2 gpurun_out/ncu_ust_panel.log
