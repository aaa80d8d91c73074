set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/c4_s2u.json 2>gpurun_out/c4_s2u.err
timeout 900 python bench.py --no-e2e --no-cpu-baseline --streams 1 > gpurun_out/c4_s1u.json 2>gpurun_out/c4_s1u.err
echo done
