set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_elementary.py -x -q > gpurun_out/t_elem.log 2>&1; tail -3 gpurun_out/t_elem.log
for r in 10 100 500; do
  timeout 600 python bench.py --workload elementary --rank $r --no-e2e --no-cpu-baseline > gpurun_out/el_$r.json 2>/dev/null
  DPP_ELEM_NT=1024 timeout 600 python bench.py --workload elementary --rank $r --no-e2e --no-cpu-baseline > gpurun_out/el_${r}_w.json 2>/dev/null
  timeout 600 python bench.py --workload elementary --rank $r --batch 1184 --no-e2e --no-cpu-baseline > gpurun_out/el_${r}_b.json 2>/dev/null
done
DPP_ELEM_NT=256 timeout 600 python -m pytest tests/test_gpu_elementary.py -x -q > gpurun_out/t_elem256.log 2>&1; tail -3 gpurun_out/t_elem256.log
echo done
