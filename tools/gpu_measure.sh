# round-2 measurement session: panel + probe-launch ncu captures, launch list, UST stage breakdown,
# elementary-vs-generic crossover, CPU-baseline plan
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
# stage-2 panel GEMMs (MASK = 0 launches of one sample, steps 10..12)
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:"update_ws_kernel<\(bool\)0, \(bool\)0, \(bool\)0" -s 10 -c 3 -o gpurun_out/prof_panel $CMD > gpurun_out/ncu_panel.log 2>&1
# the largest trailing-update launch (the roofline probe): masked launches (a)0 (a)1 (b)1 -> the 3rd
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k regex:"update_ws_kernel<\(bool\)0, \(bool\)0, \(bool\)1" -s 2 -c 1 -o gpurun_out/prof_probe $CMD > gpurun_out/ncu_probe.log 2>&1
# the launch list of the same command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 python bench.py --workload ust --steps 3 --warmup 2 --prof all > gpurun_out/bench_ust_prof.json 2>&1
timeout 1200 python bench.py --workload crossover > gpurun_out/bench_crossover.json 2>&1
timeout 1200 python tools/cpu_baseline.py > gpurun_out/cpu_baseline.json 2> gpurun_out/cpu_baseline.err
tail -c 400 gpurun_out/bench_crossover.json
