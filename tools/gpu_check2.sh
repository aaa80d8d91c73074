set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -k "fp32 or elementary or lensemble" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload herm_s > gpurun_out/bench_herm_s.json 2> gpurun_out/bench_herm_s.err
timeout 900 python bench.py --workload aztec_c --steps 2 --warmup 1 > gpurun_out/bench_aztec_c80.json 2> gpurun_out/bench_aztec_c80.err
echo done
