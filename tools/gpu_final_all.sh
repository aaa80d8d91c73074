# round-end evidence, part 2: every bench workload with the current code (one JSON line each)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
mkdir -p gpurun_out/final
for w in ust aztec herm_z lu_z herm_s aztec_c lensemble dist dist_z; do
  timeout 900 python bench.py --workload $w --no-e2e --no-cpu-baseline > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err
done
for r in 10 100 500; do
  timeout 600 python bench.py --workload elementary --rank $r --no-e2e --no-cpu-baseline > gpurun_out/final/bench_elem_$r.json 2> gpurun_out/final/bench_elem_$r.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final/bench_reference_arm.json 2> gpurun_out/final/bench_reference_arm.err
echo done
