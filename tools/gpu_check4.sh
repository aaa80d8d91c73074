set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x -k "chunked or host or config3 or parity" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
DPP_CHUNK_COLS=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c4_nochunk.json 2> gpurun_out/bench_c4_nochunk.err
DPP_CHUNK_COLS=2048 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_ch2048.json 2> gpurun_out/bench_c4_ch2048.err
DPP_CHUNK_COLS=4096 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_ch4096.json 2> gpurun_out/bench_c4_ch4096.err
DPP_CHUNK_COLS=1024 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_ch1024.json 2> gpurun_out/bench_c4_ch1024.err
echo done
