# one-tile launch latency (probe) and the UST step's launch list (serialised kernel times)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for m in 128 256 1024 4096; do python tools/probe.py $m 128; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ust.csv python bench.py --workload ust --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ust.log 2>&1
python tools/launches.py gpurun_out/launches_ust.csv | head -20
