# stage-2 panel after the snaked fragments: launch timelines (C4 one sample, UST batch) and ncu of
# C4 / UST panel launches
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python tools/timeline.py > gpurun_out/timeline_new.json 2> gpurun_out/timeline_new.err
python tools/timeline.py 3120 0 1024 > gpurun_out/timeline_ust_new.json 2> gpurun_out/timeline_ust_new.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.0' -s 30 -c 3 -o gpurun_out/prof_panel_new $CMD > gpurun_out/ncu_panel_new.log 2>&1
UCMD="python bench.py --workload ust --steps 1 --warmup 1"
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.0' -s 6 -c 2 -o gpurun_out/prof_ust_panel_new $UCMD > gpurun_out/ncu_ust_panel_new.log 2>&1
echo done
