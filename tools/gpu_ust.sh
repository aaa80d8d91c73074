# UST (configs[1]) variants, every stage bracketed
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for cfg in "--nb 128" "--nb 128 --lookahead 0" "--nb 128 --group 3"; do
  timeout 600 python bench.py --workload ust --steps 3 --warmup 2 --prof all $cfg > gpurun_out/ust.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ust.json').read().strip().splitlines()[-1])
print('$cfg', d['samples_per_s'], d['pct_fp64_peak'], {k:(v['ms'],v['ms_union']) for k,v in d['stages'].items()})"
done
