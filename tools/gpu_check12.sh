set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -k "elementary" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 10 100 500; do timeout 900 python bench.py --workload elementary --rank $r > gpurun_out/bench_elem_$r.json 2> gpurun_out/bench_elem_$r.err; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"update_ws_kernel<\(bool\)0, \(bool\)0, \(bool\)1" -s 5 -c 1 -o gpurun_out/prof_update $CMD > gpurun_out/ncu_full.log 2>&1
echo done
