# round-2 evidence: GPU suite, smoke, the default bench line (as the driver runs it), every other
# workload, the ncu launch list + diag capture of the current code
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in ust aztec herm_z lu_z herm_s lensemble dist dist_z; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
for k in 10 100 500; do timeout 600 python bench.py --workload elementary --rank $k --steps 5 --warmup 3 > gpurun_out/bench_elem_$k.json 2>/dev/null; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
timeout 900 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 --cache-control none -k regex:"diag_rl_kernel" -s 40 -c 1 -o gpurun_out/prof_diag $CMD > gpurun_out/ncu_diag.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
python tools/timeline.py > gpurun_out/timeline.json 2> gpurun_out/timeline.err
timeout 600 python bench.py --workload aztec_c --steps 3 --warmup 2 > gpurun_out/bench_aztec_c.json 2>/dev/null
timeout 600 python bench.py --workload crossover > gpurun_out/bench_crossover.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
HCMD="python bench.py --workload herm_s --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_herm_s.csv $HCMD > gpurun_out/ncu_launch_hs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --cache-control none --kernel-name-base demangled -k regex:"update_tc32_kernel" -s 40 -c 1 -o gpurun_out/prof_tc32 $HCMD > gpurun_out/ncu_tc32.log 2>&1
echo done
