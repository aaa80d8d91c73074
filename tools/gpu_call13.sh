set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
for w in aztec ust herm_s; do timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
for d in 60 80; do timeout 900 python bench.py --workload aztec_c --aztec-d $d --steps 2 --warmup 1 > gpurun_out/bench_aztec_c$d.json 2> gpurun_out/bench_aztec_c$d.err; done
echo done
