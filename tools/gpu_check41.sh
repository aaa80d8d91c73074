set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for s in 3 4; do
  timeout 900 python bench.py --no-e2e --no-cpu-baseline --streams $s > gpurun_out/c4_st$s.json 2>/dev/null
  timeout 900 python bench.py --no-e2e --no-cpu-baseline --streams $s --steps 8 > gpurun_out/c4_st${s}_k8.json 2>/dev/null
done
echo done
