set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for i in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_small$i.json 2>/dev/null
  DPP_WS_SMALL=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_nosmall$i.json 2>/dev/null
done
timeout 600 python bench.py --workload lensemble --no-e2e --no-cpu-baseline > gpurun_out/lens_small.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
echo done
