set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for s in 1 2; do
  timeout 900 python bench.py --workload ust --ust-streams $s --no-e2e --no-cpu-baseline > gpurun_out/ust_s$s.json 2>gpurun_out/ust_s$s.err
done
timeout 900 python bench.py --workload ust --ust-streams 2 --batch-chunk 512 --batch 512 --no-e2e --no-cpu-baseline > gpurun_out/ust_s2b512.json 2>/dev/null
echo done
