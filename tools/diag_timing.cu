// Diagnostic: one diag-tile kernel (stage 1, real 128-tile) alone -- its CUDA-event time per launch
// and, from a second build with per-warp clock64 stamps, where the time goes inside the tile
// (sub-panel pivots vs the other warps' block updates / inverse rows vs the CTA barriers).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include \
//        -I paper_1905_00165_b200/csrc tools/diag_timing.cu -o tools/diag_timing.bin
// Run:   tools/diag_timing.bin [batch=1] [reps=50]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

__device__ long long g_stamps[16][64];
#define DIAG_STAMP(slot)                                                                          \
  do {                                                                                            \
    if (blockIdx.y == 0 && (threadIdx.x & 31) == 0) g_stamps[threadIdx.x >> 5][(slot)] = clock64(); \
  } while (0)

#include "kernels.h"
#include "../paper_1905_00165_b200/csrc/diag_rl.cu"
#ifdef DIAG_OLD
#ifndef OLD_FILE
#define OLD_FILE "_old_diag_rl.cu"
#endif
#include OLD_FILE  // the previous kernel (a saved copy): bitwise A/B of every output
#endif

template <class F>
static float time_launch(F launch, double* dA, const double* dA0, size_t bytes, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps + 3; ++r) {
    cudaMemcpy(dA, dA0, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    cudaError_t le = launch();
    cudaEventRecord(e1);
    cudaError_t se = cudaEventSynchronize(e1);
    if (le != cudaSuccess || se != cudaSuccess) {
      printf("error %s %s\n", cudaGetErrorString(le), cudaGetErrorString(se));
      exit(1);
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 3 && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const int batch = argc > 1 ? atoi(argv[1]) : 1, reps = argc > 2 ? atoi(argv[2]) : 50;
  const int nb = argc > 3 ? atoi(argv[3]) : 128, ld = argc > 4 ? atoi(argv[4]) : nb, n = nb;
  const int forced = argc > 5 ? atoi(argv[5]) : 0;
  const bool fp32 = argc > 6 && atoi(argv[6]) != 0;  // the single-precision instantiation (no A/B)
  // A = 0.5 I + 0.3/sqrt(n) * symmetric noise: pivots in (0, 1), roughly half kept
  std::vector<double> A((size_t)ld * n * batch, 0.0);
  srand(7);
  for (int s = 0; s < batch; ++s)
    for (int j = 0; j < n; ++j)
      for (int i = j; i < n; ++i) {
        const double v = (i == j) ? 0.5 : 0.3 / 11.3 * ((double)rand() / RAND_MAX - 0.5);
        A[(size_t)s * ld * n + i + (size_t)j * ld] = v;
        A[(size_t)s * ld * n + j + (size_t)i * ld] = 77.0;  // poisoned upper triangle
      }
  std::vector<uint8_t> F((size_t)n * batch);
  for (auto& f : F) f = rand() & 1;
  double *dA0, *dA, *Bm, *dvec, *ll;
  uint8_t *mask, *dF;
  void* state;
  const size_t bytes = A.size() * 8;
  cudaMalloc(&dA0, bytes); cudaMalloc(&dA, bytes);
  cudaMalloc(&Bm, (size_t)nb * nb * 8 * batch); cudaMalloc(&dvec, (size_t)nb * 8 * batch);
  cudaMalloc(&ll, 8 * batch); cudaMalloc(&mask, (size_t)n * batch); cudaMalloc(&state, 64 * (size_t)batch);
  cudaMalloc(&dF, F.size());
  if (fp32) {  // the tile in fp32, in the first half of the buffers
    std::vector<float> Af(A.begin(), A.end());
    cudaMemcpy(dA0, Af.data(), Af.size() * 4, cudaMemcpyHostToDevice);
  } else {
    cudaMemcpy(dA0, A.data(), bytes, cudaMemcpyHostToDevice);
  }
  cudaMemcpy(dF, F.data(), F.size(), cudaMemcpyHostToDevice);
  dpp::DiagArgs d{};
  d.A = dA; d.ld = ld; d.strideA = (int64_t)ld * n; d.n = n + 1;  // n + 1: not the last tile (ops formed)
  d.j0 = 0; d.tcol = 0; d.jb = nb; d.seed = 1; d.b0 = 0; d.mask = mask; d.forced = forced ? dF : nullptr;
  d.state = state; d.loglik = ll; d.info = nullptr; d.tie_tol = 1e-9; d.range_tol = 1e-8; d.batch = batch; d.map = 0;
  d.need_ops = 1; d.Bm = Bm; d.Am = nullptr; d.dvec = dvec; d.ldm = nb; d.strideM = (int64_t)nb * nb;
  auto outputs = [&]() {
    std::vector<double> o(A.size() + (size_t)nb * nb * batch + (size_t)nb * batch + 8 * batch);
    std::vector<uint8_t> m((size_t)n * batch);
    cudaMemcpy(o.data(), dA, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data() + A.size(), Bm, (size_t)nb * nb * 8 * batch, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data() + A.size() + (size_t)nb * nb * batch, dvec, (size_t)nb * 8 * batch, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data() + A.size() + (size_t)nb * nb * batch + (size_t)nb * batch, state, 64 * batch,
               cudaMemcpyDeviceToHost);
    cudaMemcpy(m.data(), mask, m.size(), cudaMemcpyDeviceToHost);
    return std::make_pair(o, m);
  };
  const float t_new = time_launch([&] { return dpp::launch_diag_rl(nb, d, 0, fp32); }, dA, dA0, bytes, reps);
  auto out_new = outputs();
  long long st[16][64];
  cudaMemcpyFromSymbol(st, g_stamps, sizeof st);
  printf("{\"batch\": %d, \"nb\": %d, \"ld\": %d, \"forced\": %d, \"us_new\": %.2f", batch, nb, ld, forced, 1000 * t_new);
#ifdef DIAG_OLD
  if (!fp32) {
  const float t_old = time_launch([&] { return dpp_old::launch_diag_rl(nb, d, 0); }, dA, dA0, bytes, reps);
  auto out_old = outputs();
  size_t ndiff = 0;
  for (size_t i = 0; i < out_new.first.size(); ++i)
    if (memcmp(&out_new.first[i], &out_old.first[i], 8) != 0) ++ndiff;
  const bool mask_eq = out_new.second == out_old.second;
  printf(", \"us_old\": %.2f, \"words_differing_from_old\": %zu, \"mask_equal\": %s", 1000 * t_old, ndiff,
         mask_eq ? "true" : "false");
  }
#endif
  printf("}\n");
  if (batch > 1) return 0;
  const int NW = dpp::RL_NWARP;
  const long long t0 = st[0][30];
  printf("# clocks from kernel entry (warp 0); slots: 0 copies issued, 1 tile loaded, per sub-panel P: 2+3P S1 done, "
         "3+3P after barrier, 4+3P S2/S3 done; 28 end\n");
  for (int P = 0; P < nb / 16; ++P) {
    const long long start = P == 0 ? st[0][1] : st[0][4 + 3 * (P - 1)];
    long long oth = 0;
    for (int w = 1; w < NW; ++w) {
      const long long t = st[w][2 + 3 * P] - start;
      oth = t > oth ? t : oth;
    }
    long long upd = 0, s2 = 0;
    for (int w = 1; w < NW; ++w) {
      const long long t = st[w][40 + P] - start;
      upd = t > upd ? t : upd;
    }
    for (int w = 0; w < NW; ++w) {
      const long long t = st[w][48 + P] - st[0][3 + 3 * P];
      s2 = t > s2 ? t : s2;
    }
    if (P >= 1) {
      printf("   workers (from phase start): ");
      for (int w = 1; w < NW; ++w)
        printf(" w%d: updates %5lld end %5lld |", w, st[w][40 + P] - start, st[w][2 + 3 * P] - start);
      printf("\n");
    }
    printf("P=%d  F(warp0) %6lld  others %6lld (block updates %6lld)  S2 %6lld (w0 %5lld)  S3 %6lld  total %6lld\n", P,
           st[0][2 + 3 * P] - start, oth, P ? upd : 0, s2, st[0][48 + P] - st[0][3 + 3 * P],
           st[0][4 + 3 * P] - st[0][32 + P], st[0][4 + 3 * P] - start);
  }
  long long endmax = 0;
  for (int w = 0; w < NW; ++w) endmax = st[w][28] - t0 > endmax ? st[w][28] - t0 : endmax;
  printf("load %lld  end stage %lld (per warp:", st[0][1] - t0, endmax - (st[0][4 + 3 * (nb / 16 - 1)] - t0));
  for (int w = 0; w < NW; ++w) printf(" %lld", st[w][28] - st[0][4 + 3 * (nb / 16 - 1)]);
  printf(")  total %lld cycles\n", endmax);
  return 0;
}
