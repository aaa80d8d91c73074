# schedule-constant sweep: driver.cu and dist.cu rebuilt with -D overrides; C4 (one-stream latency + three in flight), UST (UST=1), the block-cyclic workloads (DIST=1 instead of C4)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cd paper_1905_00165_b200
NCCL_INC=""; [ -f /usr/include/nccl.h ] && NCCL_INC="-I/usr/include"
relink() {
  for f in driver dist; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../include $NCCL_INC $1 -c csrc/$f.cu -o _build/$f.o || exit 1
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libdpp_b200.so _build/*.o -L/usr/lib/x86_64-linux-gnu -lnccl -Xlinker -rpath=/usr/lib/x86_64-linux-gnu || exit 1
}
cd ..
v() { python -c "import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]);print(sys.argv[2], 'value', d.get('value'), 'samples/s', d.get('samples_per_s'), 'lat', (d.get('latency_one_stream') or {}).get('ms_per_sample'))" $1 "$2"; }
for D in "$@"; do
  (cd paper_1905_00165_b200 && relink "$D")
  [ -z "$DIST" ] && { timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dist > gpurun_out/sw.json 2>/dev/null; v gpurun_out/sw.json "c4 $D"; }
  [ -n "$DIST" ] && for w in dist dist_z; do timeout 600 python bench.py --workload $w --steps 3 --warmup 2 > gpurun_out/sw.json 2>/dev/null; v gpurun_out/sw.json "$w $D"; done
  [ -n "$UST" ] && { timeout 600 python bench.py --workload ust --steps 3 --warmup 2 > gpurun_out/sw.json 2>/dev/null; v gpurun_out/sw.json "ust $D"; }
done
