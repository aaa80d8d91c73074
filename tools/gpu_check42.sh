set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_default3.json 2>gpurun_out/bench_default3.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref3.json 2>gpurun_out/bench_ref3.err
echo done
