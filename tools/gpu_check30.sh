set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --workload ust --no-e2e --no-cpu-baseline > gpurun_out/ust_idle.json 2>/dev/null
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_idle.json 2>/dev/null
timeout 600 python bench.py --workload herm_z --no-e2e --no-cpu-baseline > gpurun_out/hz_idle.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
echo done
