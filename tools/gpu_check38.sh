set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for e in 2 3 4; do
  timeout 900 python bench.py --no-cpu-baseline --e2e-streams $e --steps 6 > gpurun_out/c4_e$e.json 2>gpurun_out/c4_e$e.err
done
timeout 900 python bench.py --no-cpu-baseline --streams 1 --e2e-streams 2 --steps 6 > gpurun_out/c4_s1e2.json 2>gpurun_out/c4_s1e2.err
echo done
