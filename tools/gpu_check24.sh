set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grouped or alternate" > gpurun_out/t_group.log 2>&1; tail -3 gpurun_out/t_group.log
for g in 2 3 4; do
  DPP_GROUP=$g timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_g$g.json 2>/dev/null
  DPP_GROUP=$g timeout 600 python bench.py --workload herm_z --no-e2e --no-cpu-baseline > gpurun_out/hz_g$g.json 2>/dev/null
  DPP_GROUP=$g timeout 600 python bench.py --workload ust --no-e2e --no-cpu-baseline > gpurun_out/ust_g$g.json 2>/dev/null
done
DPP_GROUP=3 DPP_PAIR_MIN_ROWS=8192 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_g3m8.json 2>/dev/null
DPP_GROUP=4 DPP_PAIR_MIN_ROWS=8192 timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_g4m8.json 2>/dev/null
echo done
