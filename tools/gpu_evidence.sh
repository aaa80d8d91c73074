# round evidence: GPU suite, smoke, the default bench line (as the driver runs it), every other
# workload, the reference arm, ncu launch list + diag / panel / tc32 captures, launch timelines,
# the diag-tile kernel alone (tools/diag_timing.cu)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in ust aztec herm_z lu_z herm_s lensemble dist dist_z; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for k in 10 100 500; do timeout 600 python bench.py --workload elementary --rank $k --steps 5 --warmup 3 > gpurun_out/bench_elem_$k.json 2>/dev/null; done
timeout 600 python bench.py --workload aztec_c --steps 3 --warmup 2 > gpurun_out/bench_aztec_c.json 2>/dev/null
timeout 600 python bench.py --workload crossover > gpurun_out/bench_crossover.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
python tools/timeline.py > gpurun_out/timeline.json 2> gpurun_out/timeline.err
python tools/timeline.py 3120 0 1024 > gpurun_out/timeline_ust.json 2> gpurun_out/timeline_ust.err
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include -I paper_1905_00165_b200/csrc tools/diag_timing.cu -o tools/diag_timing.bin > /dev/null 2>&1
{ timeout 60 tools/diag_timing.bin 1 50 128 128 0; for a in "1 20 128 131 0" "1 20 128 130 1" "1 20 64 64 0" "148 10 128 128 0" "1024 5 128 128 0"; do timeout 60 tools/diag_timing.bin $a | head -1; done; } > gpurun_out/diag_timing.txt 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --cache-control none -k regex:"diag_rl_kernel" -s 40 -c 1 -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --kernel-name-base demangled -k regex:'update_ws_kernel<.bool.0, .bool.0, .bool.0' -s 30 -c 3 -o gpurun_out/prof_panel $CMD > gpurun_out/ncu_panel.log 2>&1
HCMD="python bench.py --workload herm_s --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --cache-control none --kernel-name-base demangled -k regex:"update_tc32_kernel" -s 40 -c 1 -o gpurun_out/prof_tc32 $HCMD > gpurun_out/ncu_tc32.log 2>&1
echo done
