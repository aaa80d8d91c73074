# round-2 GPU session: build, GPU tests, a short bench (args: extra bench flags)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 $BENCH_FLAGS > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
tail -c 1500 gpurun_out/bench_a.json; tail -5 gpurun_out/bench_a.err
