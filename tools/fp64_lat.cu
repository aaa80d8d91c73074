// Diagnostic: dependent-chain latencies (cycles) of the FP64 instructions on the diag tile's
// critical path -- DFMA, DMUL, DADD, DSETP+FSEL, MUFU.RCP64H, a full recip (RCP64H + 2 Newton
// steps), DMMA.8x8x4 (accumulator chain), SHFL of a double, LDS, named barrier -- one warp alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_lat.cu -o tools/fp64_lat.bin
#include <cuda_runtime.h>

#include <cstdio>

constexpr int N = 256;

__global__ void lat(double* out, long long* cyc, double x0) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = x0 + lane;
  __syncwarp();
  double x = x0 + lane * 1e-3, y = 1.0 + lane * 1e-6;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (lane == 0) cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64();
  if (lane == 0) cyc[1] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64();
  if (lane == 0) cyc[2] = t1 - t0;
  // DSETP + select chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = (x <= y) ? x + 1e-300 : x - 1e-300;
  t1 = clock64();
  if (lane == 0) cyc[3] = t1 - t0;
  // MUFU.RCP64H chain (approximate reciprocal of the high word)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double r;
    asm volatile("{ .reg .f64 t; rcp.approx.ftz.f64 t, %1; mov.f64 %0, t; }" : "=d"(r) : "d"(x));
    x = r;
  }
  t1 = clock64();
  if (lane == 0) cyc[4] = t1 - t0;
  // full reciprocal (RCP64H + 2 Newton steps, as common.cuh recip)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double r;
    asm volatile("{ .reg .f64 t; rcp.approx.ftz.f64 t, %1; mov.f64 %0, t; }" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    x = fma(r, e, r);
  }
  t1 = clock64();
  if (lane == 0) cyc[5] = t1 - t0;
  // DMMA accumulator chain
  double c0 = 0.0, c1 = 0.0;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(x), "d"(y));
  t1 = clock64();
  if (lane == 0) cyc[6] = t1 - t0;
  // SHFL of a double chain
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64();
  if (lane == 0) cyc[7] = t1 - t0;
  // LDS chain (dependent address)
  int idx = lane;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) idx = ((int)sm[idx & 63]) & 31;
  t1 = clock64();
  if (lane == 0) cyc[8] = t1 - t0;
  // named barrier (one warp)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) asm volatile("bar.sync 1, 32;\n" ::: "memory");
  t1 = clock64();
  if (lane == 0) cyc[9] = t1 - t0;
  // STS -> bar.sync -> LDS round trip (the panel's publish)
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    if (lane < 16) sm[lane] = x;
    asm volatile("bar.sync 1, 32;\n" ::: "memory");
    x = sm[(lane + 1) & 15] + 1e-300;
  }
  t1 = clock64();
  if (lane == 0) cyc[10] = t1 - t0;
  out[lane] = x + c0 + c1 + idx;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 16 * 8);
  cudaMemset(cyc, 0, 16 * 8);
  for (int r = 0; r < 3; ++r) lat<<<1, 32>>>(out, cyc, 0.5);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"DFMA", "DMUL", "DADD", "DSETP+FSEL+DADD", "MUFU.RCP64H", "recip(RCP64H+2 Newton)",
                         "DMMA.8x8x4 acc chain", "SHFL double", "LDS (dep addr, +cvt)", "BAR.SYNC 1 warp",
                         "STS->BAR->LDS(+DADD)"};
  for (int i = 0; i < 11; ++i) printf("%-28s %6.1f cycles per link\n", names[i], (double)h[i] / N);
  return 0;
}
