# per-source-line warp stalls of the roofline probe launch and of one UST batched trailing update
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/probe.py > gpurun_out/probe_plain.txt 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:'update_ws_kernel' -s 1 -c 1 -o gpurun_out/prof_probe_lines python tools/probe.py > gpurun_out/ncu_probe_lines.log 2>&1
UCMD="python bench.py --workload ust --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.1' -s 9 -c 1 -o gpurun_out/prof_ust_upd_lines $UCMD > gpurun_out/ncu_ust_upd_lines.log 2>&1
cat gpurun_out/probe_plain.txt; tail -2 gpurun_out/ncu_probe_lines.log gpurun_out/ncu_ust_upd_lines.log
