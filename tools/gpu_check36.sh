set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for i in 1 2; do
  timeout 900 python bench.py --no-e2e --no-cpu-baseline --streams 2 > gpurun_out/c4_s2_$i.json 2>gpurun_out/c4_s2_$i.err
  timeout 900 python bench.py --no-e2e --no-cpu-baseline --streams 1 > gpurun_out/c4_s1_$i.json 2>gpurun_out/c4_s1_$i.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
echo done
