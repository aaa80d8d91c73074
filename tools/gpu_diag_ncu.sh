# ncu of the diag-tile kernel alone (tools/diag_timing.cu, one 128-tile): stall reasons per source line
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -I include -I paper_1905_00165_b200/csrc tools/diag_timing.cu -o tools/diag_timing.bin > /dev/null 2>&1 || echo BUILD FAILED
timeout 300 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:diag_rl_kernel -s 5 -c 1 -o gpurun_out/prof_diag_new tools/diag_timing.bin 1 8 128 128 0 > gpurun_out/ncu_diag_new.log 2>&1
tail -3 gpurun_out/ncu_diag_new.log
