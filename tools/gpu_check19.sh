set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload aztec_c --aztec-d 60 --steps 3 --warmup 3 --tally 12 > gpurun_out/tally60.json 2>gpurun_out/tally60.err
timeout 900 python bench.py --workload aztec_c --aztec-d 70 --steps 3 --warmup 3 --tally 8 > gpurun_out/tally70.json 2>gpurun_out/tally70.err
timeout 1200 python bench.py --workload aztec_c --aztec-d 80 --steps 3 --warmup 3 --tally 8 > gpurun_out/tally80.json 2>gpurun_out/tally80.err
echo done
