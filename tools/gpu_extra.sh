# build; GPU parity suite; the non-default bench workloads (configs 1, 2, 4) -- one JSON line each
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-aztec dist dist_z ust}; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
echo done
