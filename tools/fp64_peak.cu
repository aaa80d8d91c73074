// FP64 peak microbenchmark for the roofline denominator.
// Measures: DMMA (mma.sync m8n8k4 f64) throughput, DFMA throughput, both with many
// independent accumulators per warp, over a grid of blocks x warps.  Prints JSON lines.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("{\"error\":\"%s line %d\"}\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template<int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// half of the warps of every block run the DMMA loop, the other half the DFMA loop: if the two
// pipes were separate, the combined rate would exceed either alone
template<int NACC>
__global__ void mixed_loop(double* out, int iters, int dfma_scale) {
  const int warp = threadIdx.x >> 5;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double s = 0;
  if (warp & 1) {
    double c[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = i;
    for (int it = 0; it < iters * dfma_scale; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i];
  } else {
    double c[NACC][2];
#pragma unroll
    for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      }
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int warps_list[] = {4, 8, 16};
  for (int wi = 0; wi < 3; ++wi) {
    int warps = warps_list[wi];
    int iters = 4000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<16><<<sms * 2, warps * 32>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 16.0 * iters * (double)warps * sms * 2;
      if (rep) printf("{\"kind\":\"dmma_m8n8k4\",\"warps_per_block\":%d,\"blocks\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", warps, sms*2, ms, flops / ms / 1e9);
    }
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      dfma_loop<16><<<sms * 2, warps * 32>>>(out, iters * 8);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16.0 * iters * 8 * (double)warps * 32 * sms * 2;
      if (rep) printf("{\"kind\":\"dfma\",\"warps_per_block\":%d,\"blocks\":%d,\"ms\":%.4f,\"tflops\":%.3f}\n", warps, sms*2, ms, flops / ms / 1e9);
    }
  }
  for (int scale : {4, 8, 16}) {
    const int warps = 8, iters = 4000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      mixed_loop<16><<<sms * 2, warps * 32>>>(out, iters, scale);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl_dmma = 2.0 * 8 * 8 * 4 * 16.0 * iters * (warps / 2) * sms * 2;
      double fl_dfma = 2.0 * 16.0 * iters * scale * (warps / 2) * 32 * sms * 2;
      if (rep) printf("{\"kind\":\"mixed_dmma_dfma\",\"dfma_scale\":%d,\"ms\":%.4f,\"tflops_total\":%.3f,\"dmma_share\":%.3f}\n",
                      scale, ms, (fl_dmma + fl_dfma) / ms / 1e9, fl_dmma / (fl_dmma + fl_dfma));
    }
  }
  CK(cudaGetLastError());
  return 0;
}
