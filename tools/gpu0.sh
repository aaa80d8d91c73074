nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi0.txt 2>&1
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clk0.csv) & SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.jsonl 2>&1
python tools/dgemm_peak.py > gpurun_out/dgemm_peak.jsonl 2>&1
kill $SMI
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
