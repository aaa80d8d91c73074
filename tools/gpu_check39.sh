set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/final2
for r in 10 100 500; do
  timeout 600 python bench.py --workload elementary --rank $r --no-e2e --no-cpu-baseline > gpurun_out/final2/bench_elem_$r.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_elementary.py -x -q > gpurun_out/t_elem.log 2>&1; tail -2 gpurun_out/t_elem.log
echo done
