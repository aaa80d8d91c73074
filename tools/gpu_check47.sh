set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload herm_s --no-e2e --no-cpu-baseline > gpurun_out/hs_s3.json 2>gpurun_out/hs_s3.err
timeout 900 python bench.py --workload herm_s --streams 1 --no-e2e --no-cpu-baseline > gpurun_out/hs_s1.json 2>/dev/null
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c4_last.json 2>/dev/null
echo done
