set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/c4_def.json 2>gpurun_out/c4_def.err
timeout 600 python bench.py --workload aztec > gpurun_out/az_def.json 2>gpurun_out/az_def.err
timeout 600 python bench.py --workload herm_s > gpurun_out/hs_def.json 2>gpurun_out/hs_def.err
echo done
