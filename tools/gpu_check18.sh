set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload aztec_c --steps 2 --warmup 1 > gpurun_out/az_new_21.json 2>/dev/null
cp tools/update_simt_prev.cu.txt paper_1905_00165_b200/csrc/update_simt.cu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1 || { cat gpurun_out/build2.log; exit 1; }
timeout 900 python bench.py --workload aztec_c > gpurun_out/az_old_53.json 2>/dev/null
echo done
