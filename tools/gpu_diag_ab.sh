nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DDIAG_OLD '-DOLD_FILE="_prev_diag_rl.cu"' -I include -I paper_1905_00165_b200/csrc tools/diag_timing.cu -o tools/diag_ab.bin > /dev/null 2>&1 || echo BUILD FAILED
for r in 1 2; do for a in "1 50 128 128 0" "1 50 128 130 1" "1024 5 128 128 0"; do timeout 60 tools/diag_ab.bin $a | head -1; done; done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --workload herm_s --steps 5 --warmup 3 > gpurun_out/hs.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/hs.json').read().strip().splitlines()[-1]);print('herm_s', d['value'], d['ms_per_step'], d['stages']['diag'])"
