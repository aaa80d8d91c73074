set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -k "parity or host" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
DPP_COPY_GATED=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_ng.json 2> gpurun_out/bench_c4_ng.err
echo done
