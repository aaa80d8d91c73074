# throughput of the other BASELINE configs + ncu DRAM traffic of the trailing-update launches
python paper_1905_00165_b200/build.py > /dev/null || exit 1
timeout 600 python bench.py --workload ust --steps 3 --warmup 1 > gpurun_out/bench_ust.json 2> gpurun_out/bench_ust.err
timeout 600 python bench.py --workload herm_z --steps 3 --warmup 2 > gpurun_out/bench_herm_z.json 2> gpurun_out/bench_herm_z.err
timeout 600 python bench.py --workload lu_z --steps 3 --warmup 2 > gpurun_out/bench_lu_z.json 2> gpurun_out/bench_lu_z.err
timeout 900 python bench.py --workload dist --n 32768 --steps 2 --warmup 1 > gpurun_out/bench_dist.json 2> gpurun_out/bench_dist.err
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/bench_small0.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:update_ws --csv --log-file gpurun_out/traffic.csv $CMD > gpurun_out/ncu_traffic.log 2>&1
echo done
