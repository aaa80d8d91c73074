set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host" > gpurun_out/t_host.log 2>&1; tail -3 gpurun_out/t_host.log
timeout 900 python bench.py > gpurun_out/c4_e2e.json 2>gpurun_out/c4_e2e.err
echo done
