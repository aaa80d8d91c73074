set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for i in 1 2; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --prof all > gpurun_out/c4_pall$i.json 2>gpurun_out/c4_pall$i.err
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --prof trailing > gpurun_out/c4_ptr$i.json 2>gpurun_out/c4_ptr$i.err
done
timeout 600 python -m pytest tests/test_library.py -q > gpurun_out/t_lib.log 2>&1; tail -2 gpurun_out/t_lib.log
echo done
