set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for t in 5 4 3 2.5; do
  DPP_DIAG_TILES=$t timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_dt$t.json 2>/dev/null
  DPP_DIAG_TILES=$t timeout 600 python bench.py --workload ust --no-e2e --no-cpu-baseline > gpurun_out/ust_dt$t.json 2>/dev/null
done
echo done
