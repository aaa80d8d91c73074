python paper_1905_00165_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
for tpc in 2 4 8 1000; do DPP_WS_TPC=$tpc timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_tpc$tpc.json 2> gpurun_out/bench_tpc$tpc.err; done
echo done
