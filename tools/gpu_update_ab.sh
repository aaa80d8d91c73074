# A/B of update_ws.cu compile-time variants (-D...): probe at three K, parity tests, UST, C4
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCCL_INC=""; [ -f /usr/include/nccl.h ] && NCCL_INC="-I/usr/include"
relink() {
  (cd paper_1905_00165_b200 && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include $NCCL_INC $1 -c csrc/update_ws.cu -o _build/update_ws.o &&
   nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libdpp_b200.so _build/*.o -L/usr/lib/x86_64-linux-gnu -lnccl -Xlinker -rpath=/usr/lib/x86_64-linux-gnu) || exit 1
}
v() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], 'value', d.get('value'), 'samples/s', d.get('samples_per_s'), 'lat', (d.get('latency_one_stream') or {}).get('ms_per_sample'))" $1 "$2"; }
for D in "$@"; do
  relink "$D"
  for a in "15872 128" "15872 384" "15872 3072"; do echo "$D $(timeout 120 python tools/probe.py $a)"; done
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lensemble.py -m gpu -q -x --timeout 300 2>&1 | tail -2
  timeout 600 python bench.py --workload ust --steps 4 --warmup 3 > gpurun_out/sw.json 2>/dev/null; v gpurun_out/sw.json "ust $D"
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/sw.json 2>/dev/null; v gpurun_out/sw.json "c4 $D"
done
