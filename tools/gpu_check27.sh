set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in 512 1024; do
  timeout 900 python bench.py --workload ust --batch-chunk $c --no-e2e --no-cpu-baseline > gpurun_out/ust_c$c.json 2>/dev/null
done
for m in 3072 4096 8192; do
  DPP_PAIR_MIN_ROWS=$m timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_pm$m.json 2>/dev/null
done
echo done
