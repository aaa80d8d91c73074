set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
DPP_TAIL_ROWS=1000 timeout 900 python -m pytest tests -m gpu -q -x -k "config3 or herm_d" > gpurun_out/pytest_tail.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tail.log
for t in 0 2048 4096 6144; do DPP_TAIL_ROWS=$t timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t$t.json 2> gpurun_out/bench_t$t.err; done
echo done
