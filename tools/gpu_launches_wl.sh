# per-kernel launch lists of other workloads (ncu --metrics gpu__time_duration.sum): herm_z, lu_z, herm_s
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in herm_z lu_z herm_s; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "== $w"; python tools/launches.py gpurun_out/launches_$w.csv | grep "dpp::" | head -8
done
