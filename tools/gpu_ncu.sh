# build, parity tests, bench; then one ncu --set full capture of the kernels matching $NCU_K
python paper_1905_00165_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"diag_kernel|panel_|update_" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-update_}" -s ${NCU_S:-6} -c ${NCU_C:-3} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo done
