# last check of the round: full GPU suite, smoke, default bench and the main workloads with the
# committed defaults; then the complex ring variant (-DDPP_WS_KCZ=16) on the suite and the complex workloads
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in ust aztec herm_z lu_z lensemble dist dist_z; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
python tools/probe.py > gpurun_out/probe_final.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
NCCL_INC=""; [ -f /usr/include/nccl.h ] && NCCL_INC="-I/usr/include"
(cd paper_1905_00165_b200 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include $NCCL_INC -DDPP_WS_KCZ=16 -DDPP_WS_STAGESZ=4 -c csrc/update_ws.cu -o _build/update_ws.o &&
 nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libdpp_b200.so _build/*.o -L/usr/lib/x86_64-linux-gnu -lnccl -Xlinker -rpath=/usr/lib/x86_64-linux-gnu) || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_kcz16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_kcz16.log
for w in aztec herm_z lu_z dist_z; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_${w}_kcz16.json 2> gpurun_out/bench_${w}_kcz16.err
done
tail -3 gpurun_out/pytest_gpu_kcz16.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_*.json')):
    if 'remap' in f or 'final' in f: continue
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: continue
    print(f.split('/')[-1], d.get('value'), 'ms', d.get('ms_per_step'), 'pct', d.get('pct_fp64_peak'), 'sps', d.get('samples_per_s'), 'lat', (d.get('latency_one_stream') or {}).get('ms_per_sample'), 'roof', (d.get('roofline') or {}).get('frac'))
PY
