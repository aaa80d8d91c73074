# the diag-tile kernel alone: new vs old (tools/_old_diag_rl.cu, a saved copy of the previous kernel) -- time and bitwise outputs; phase stamps
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -DDIAG_OLD -I include -I paper_1905_00165_b200/csrc tools/diag_timing.cu -o tools/diag_timing.bin > /dev/null 2>&1 || echo BUILD FAILED
timeout 60 tools/diag_timing.bin 1 50 128 128 0
timeout 60 tools/diag_timing.bin 1 20 128 131 0 | head -1
timeout 60 tools/diag_timing.bin 1 20 128 130 1 | head -1
timeout 60 tools/diag_timing.bin 1 20 64 64 0 | head -1
timeout 60 tools/diag_timing.bin 148 10 128 128 0 | head -1
timeout 60 tools/diag_timing.bin 1024 5 128 128 0 | head -1
