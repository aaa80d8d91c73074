// Diagnostic: DMMA.8x8x4 throughput of ONE CTA (one SM) with 1..16 warps, each warp issuing
// independent accumulator chains (8 chains), cycles per DMMA per SM and per warp.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_tput.cu -o tools/dmma_tput.bin
#include <cuda_runtime.h>
#include <cstdio>
constexpr int N = 512;
__global__ void k(double* out, long long* cyc) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < N; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  __syncthreads();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 2, 3, 4, 8, 12, 16}) {
    k<<<1, 32 * w>>>(out, cyc); cudaDeviceSynchronize();
    k<<<1, 32 * w>>>(out, cyc); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double dm = (double)N * 8 * w;
    printf("warps %2d: %.2f cycles per DMMA per SM, %.1f per DMMA per warp\n", w, h / dm, h / (dm / w));
  }
  return 0;
}
