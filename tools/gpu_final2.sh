# confirmation of the committed HEAD: GPU suite, smoke, default bench, launch list, probe ncu
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-dist --streams 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on --warp-sampling-interval 0 --kernel-name-base demangled -k regex:update_ws_kernel -s 1 -c 1 -o gpurun_out/prof_probe_final python tools/probe.py > gpurun_out/ncu_probe_final.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
