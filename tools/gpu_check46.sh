set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for w in herm_z lu_z; do
  timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline > gpurun_out/${w}_s3.json 2>gpurun_out/${w}_s3.err
  timeout 900 python bench.py --workload $w --streams 1 --no-e2e --no-cpu-baseline > gpurun_out/${w}_s1.json 2>/dev/null
done
echo done
