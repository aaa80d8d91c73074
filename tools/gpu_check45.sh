set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for s in 1 2 3; do
  timeout 900 python bench.py --workload aztec --aztec-streams $s --no-e2e --no-cpu-baseline > gpurun_out/az_s$s.json 2>gpurun_out/az_s$s.err
done
echo done
