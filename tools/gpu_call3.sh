set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload aztec > gpurun_out/bench_aztec.json 2> gpurun_out/bench_aztec.err
timeout 900 python bench.py --workload lu_z > gpurun_out/bench_lu_z.json 2> gpurun_out/bench_lu_z.err
for c in 512 1024; do timeout 900 python bench.py --workload ust --batch-chunk $c > gpurun_out/bench_ust_$c.json 2> gpurun_out/bench_ust_$c.err; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_ws_kernel" -s 40 -c 2 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
