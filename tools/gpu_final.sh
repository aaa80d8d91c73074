# round-end evidence: full GPU suite, default bench (with e2e + cpu baseline), the ncu launch list of
# the same command, one --set full capture of a trailing-update launch, DRAM bytes of every (b)
# launch of one sample
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --streams 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
# the masked (trailing / lookahead) update launches: (a)0 (a)1 (b)1 (a)2 (a)3 (b)3 ... -> the 6th is the
# paired trailing update of step 3 (K = 256)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"update_ws_kernel<\(bool\)0, \(bool\)0, \(bool\)1" -s 5 -c 1 -o gpurun_out/prof_update $CMD > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"update_ws_kernel" --csv --log-file gpurun_out/traffic.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
echo done
