set -x
python paper_1905_00165_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r01a.json 2> gpurun_out/bench_r01a.err
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"diag_kernel|panel_|update_kernel" --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo finished
