// Diagnostic: the 3xTF32 tcgen05 update kernel (update_tc32.cu) alone on small matrices against a
// double-precision host reference, C -= A B^T with A (M x K), B (N x K) column-major.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 [-DTC32_DEBUG] -I include \
//        -I paper_1905_00165_b200/csrc tools/tc32_test.cu -o tools/tc32_test.bin
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.h"
#include "../paper_1905_00165_b200/csrc/update_tc32.cu"

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 128, N = argc > 2 ? atoi(argv[2]) : 128, K = argc > 3 ? atoi(argv[3]) : 32;
  const int mode = argc > 4 ? atoi(argv[4]) : 0;  // 0 random, 1 A = e_i e_k pattern probe
  std::vector<float> A((size_t)M * K), B((size_t)N * K), C((size_t)M * N, 0.f);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : B) x = (float)rand() / RAND_MAX - 0.5f;
  if (mode == 1) {  // A(i, k) = i + 1000 k, B(j, k) = (k == 0 && j == 0) -> C(i, 0) = -(i)
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < M; ++i) A[i + (size_t)k * M] = (float)(i + 1000 * k);
    std::fill(B.begin(), B.end(), 0.f);
    B[0] = 1.f;
  }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C.data(), C.size() * 4, cudaMemcpyHostToDevice);
  dpp::UpdateArgs u{};
  u.Aop = dA; u.lda = M; u.Bop = dB; u.ldb = N; u.C = dC; u.ldc = M;
  u.a_rows = M; u.b_rows = N; u.K = K; u.rows = M; u.cols = N; u.batch = 1; u.vec = 1;
  u.tcs_bytes = (int64_t)dpp::tc32_scratch_bytes(M, N, K, false);
  cudaMalloc(&u.tcs, (size_t)u.tcs_bytes);
  cudaError_t e = dpp::launch_update_tc32(u, 0, false);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("launch %s sync %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
  std::vector<float> G(C.size());
  cudaMemcpy(G.data(), dC, G.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  int bi = -1, bj = -1;
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < M; ++i) {
      double r = 0;
      for (int k = 0; k < K; ++k) r -= (double)A[i + (size_t)k * M] * B[j + (size_t)k * N];
      const double d = fabs(r - G[i + (size_t)j * M]);
      maxref = fmax(maxref, fabs(r));
      if (d > maxerr) { maxerr = d; bi = i; bj = j; }
    }
  printf("M %d N %d K %d: max |err| %.3e (max |ref| %.3e) at (%d, %d)\n", M, N, K, maxerr, maxref, bi, bj);
  if (mode == 1)
    for (int i = 0; i < 12; ++i) printf("C(%d,0) = %.1f (want %.1f)   C(%d,1) = %.1f\n", i, G[i], -(double)i, i, G[i + M]);
  if (mode == 0) {
    printf("row errors (col 0): ");
    for (int i = 0; i < 16; ++i) {
      double r = 0;
      for (int k = 0; k < K; ++k) r -= (double)A[i + (size_t)k * M] * B[0 + (size_t)k * N];
      printf("%.2e ", fabs(r - G[i]));
    }
    printf("\n");
  }
  return 0;
}
