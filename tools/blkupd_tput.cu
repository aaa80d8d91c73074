// Diagnostic: throughput of the diag kernel's block-update task (rl_block_updates<2>: two 16x16
// blocks of one block column, K = 16, DMMA.8x8x4) with 1..8 warps of one CTA, each warp on its own
// blocks; cycles per DMMA per SM sub-partition against the pipe's 16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include \
//        -I paper_1905_00165_b200/csrc tools/blkupd_tput.cu -o tools/blkupd_tput.bin
#include <cuda_runtime.h>
#include <cstdio>
#include "kernels.h"
#include "../paper_1905_00165_b200/csrc/diag_rl.cu"

constexpr int REPS = 64;
__global__ void k(long long* cyc, int nwarps) {
  extern __shared__ __align__(16) double Lb[];
  __shared__ double pv[128];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 36 * dpp::BLK_SZ * 2; e += blockDim.x) Lb[e] = 1e-3 * (e % 97);
  for (int e = tid; e < 128; e += blockDim.x) pv[e] = 0.5;
  __syncthreads();
  // warp w updates blocks (I, J) = (2 + ... ) of its own 8-row band of the packed tile: use blocks
  // of block column J = 1 + (w % 7), rows I = J, J+1 (wrapping into valid rows), sub-panel P = 0
  const int J = 1 + (warp % 6), I = J;
  long long t0 = clock64();
  if (warp < nwarps)
    for (int r = 0; r < REPS; ++r) dpp::rl_block_updates<2>(Lb, I, J, 0, pv, lane);
  long long t1 = clock64();
  __syncthreads();
  if (lane == 0 && warp < nwarps) cyc[warp] = t1 - t0;
}
int main() {
  long long* cyc;
  cudaMalloc(&cyc, 64 * 8);
  const size_t smem = 36 * dpp::BLK_SZ * 2 * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int w : {1, 2, 4, 8}) {
    k<<<1, 256, smem>>>(cyc, w); cudaDeviceSynchronize();
    k<<<1, 256, smem>>>(cyc, w); cudaError_t e = cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
    const double dm = (double)REPS * 32;  // DMMAs per warp
    printf("%s warps %d: %.1f cycles per DMMA per warp, %.1f per DMMA per SMSP\n", cudaGetErrorString(e), w, mx / dm,
           mx / dm / (w > 4 ? 2.0 : 1.0));
  }
  return 0;
}
