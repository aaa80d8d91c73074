set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
DPP_WS_VARIANT=1 timeout 900 python -m pytest tests -m gpu -q -x -k "herm_d or config3 or dist or ust or map" > gpurun_out/pytest_v1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v1.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v0.json 2> gpurun_out/bench_v0.err
DPP_WS_VARIANT=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
timeout 600 python bench.py --workload dist --n 32768 > gpurun_out/bench_dist_v0.json 2> gpurun_out/bench_dist_v0.err
DPP_WS_VARIANT=1 timeout 600 python bench.py --workload dist --n 32768 > gpurun_out/bench_dist_v1.json 2> gpurun_out/bench_dist_v1.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
DPP_WS_VARIANT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"update_ws_kernel" -s 40 -c 2 -o gpurun_out/prof_c4_v1 $CMD > gpurun_out/ncu_full_v1.log 2>&1
echo done
