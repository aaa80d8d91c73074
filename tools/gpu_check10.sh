set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -k "lensemble or parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for t in 0 4096 6144 8192; do DPP_PAIR_MIN_ROWS=$t timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_p$t.json 2> gpurun_out/bench_p$t.err; done
for t in 0 6144; do DPP_PAIR_MIN_ROWS=$t timeout 900 python bench.py --workload herm_z > gpurun_out/bench_z_p$t.json 2> gpurun_out/bench_z_p$t.err; done
echo done
