// next_tile.cu -- the chain's two one-tile GEMMs of a split step fused into one CTA (real fp64,
// nb = 128): the first row tile of the panel and the lookahead update of the next diagonal tile.
//
// Listing 3, for the rows of the NEXT block only (reading R17: the panel solve as
// a GEMM with the diag kernel's tile operator Bm):
//   P0:  L21_0 = A21_0 - A21_0 Bm^T               (rows j1 .. j1+127 of block column j0; in place)
//        W21_0 = L21_0 D1                          (the pre-scaled copy, into its panel slot)
//   LT:  A22_00 -= W21_0 L21_0^T                   (lower triangle of the next diagonal tile)
// In the split schedule (driver.cu, run_blocked) these two launches are all the next diag tile
// waits for; as two update-kernel launches they cost ~30 us each on one SM (launch, ring fill,
// C round trip, epilogue), here L21_0 stays in shared memory between the two products.
//
// Bitwise contract: every output equals the unfused launches' (update_ws_kernel): the same DMMA.8x8x4
// sequence per 32x32 warp tile (k-quads in increasing order; the panel's warp column wn stops at
// chunk 4 wn + 4 like the triangular-operator cut `btri` of the update kernel), the same
// "C - acc" subtraction and the same W = L d products (LT's A operand is formed in registers by the
// same multiply the panel epilogue stores).
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpp {
namespace {

constexpr int NB = 128, LDS = NB + 4, KCH = 32, NTH = 512;
constexpr size_t NT_SMEM = (size_t)(NB * LDS + 2 * KCH * LDS) * 8;

__global__ void __launch_bounds__(NTH, 1) next_tile_kernel(const NextTileArgs a) {
  extern __shared__ __align__(16) double sm[];
  double* Ls = sm;               // [k][LDS]: A21_0 (k-major), then L21_0 in place
  double* Bb = sm + NB * LDS;    // 2 x [KCH][LDS]: chunks of Bm
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;  // 4 x 4 warp tiles of 32 x 32 (update kernel: wm = warp % WM)

  // ---- loads: A21_0 whole (group 0), Bm chunk 0 (group 1), chunk c+1 while chunk c is used
  for (int idx = tid; idx < NB * (NB / 2); idx += NTH) {
    const int k = idx / (NB / 2), r2 = idx % (NB / 2);
    cp_async16(&Ls[k * LDS + 2 * r2], a.A21 + (int64_t)k * a.ld + 2 * r2, 16);
  }
  cp_async_commit();
  auto load_b = [&](int c) {
    double* dst = Bb + (c & 1) * KCH * LDS;
    for (int idx = tid; idx < KCH * (NB / 2); idx += NTH) {
      const int kk = idx / (NB / 2), n2 = idx % (NB / 2);
      cp_async16(&dst[kk * LDS + 2 * n2], a.Bm + (int64_t)(c * KCH + kk) * a.ldm + 2 * n2, 16);
    }
    cp_async_commit();
  };
  load_b(0);

  // ---- P0: acc = A21_0 Bm^T, warp column wn over the chunks kc8 < 4 wn + 4 (of 8 k)
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kend = 32 * wn + 32;  // k < kend
  for (int c = 0; c < NB / KCH; ++c) {
    if (c + 1 < NB / KCH) {
      load_b(c + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* Bc = Bb + (c & 1) * KCH * LDS;
    if (c * KCH < kend) {
#pragma unroll
      for (int q = 0; q < KCH / 4; ++q) {
        const int kl = q * 4 + (lane & 3), k = c * KCH + kl;
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = Ls[k * LDS + wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = Bc[kl * LDS + wn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncthreads();  // chunk c's buffer is reloaded by the next iteration's prefetch
  }
  // L21_0 = A21_0 - acc in place (every warp has finished reading Ls as its A operand)
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wn * 32 + j * 8 + 2 * (lane & 3) + e;
        Ls[c * LDS + r] = Ls[c * LDS + r] - acc[i][j][e];
      }
  }
  __syncthreads();
  // L21_0 -> A21 (in place) and W21_0 = L21_0 D1 -> its panel slot (coalesced along the rows)
  for (int idx = tid; idx < NB * NB; idx += NTH) {
    const int c = idx / NB, r = idx % NB;
    const double l = Ls[c * LDS + r];
    a.A21[r + (int64_t)c * a.ld] = l;
    a.W21[r + (int64_t)c * a.ldw] = scal(l, __ldg(a.d + c));
  }

  // ---- LT: the next diagonal tile's lower triangle -= W21_0 L21_0^T: its 10 warp tiles on or below
  // the diagonal (the update kernel idles the 6 above it) spread 3/3/2/2 over the four SM
  // sub-partitions (warp w runs on sub-partition w % 4) -- which warp computes a tile does not
  // change its arithmetic
  if (warp >= 10) return;
  int tm = 0, tn = warp;  // warp -> (tm, tn), tn <= tm, row-major over the lower triangle
  while (tn > tm) { tn -= tm + 1; ++tm; }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int q = 0; q < NB / 4; ++q) {
    const int k = q * 4 + (lane & 3);
    const double dk = __ldg(a.d + k);
    double af[4], bf[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = scal(Ls[k * LDS + tm * 32 + i * 8 + (lane >> 2)], dk);
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = Ls[k * LDS + tn * 32 + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  // C -= acc on the lower triangle: every load issued before the first store (the stores could
  // alias the loads as far as the compiler knows, which would serialize 32 global round trips)
  double cv[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = tm * 32 + i * 8 + (lane >> 2), c = tn * 32 + j * 8 + 2 * (lane & 3) + e;
        cv[i][j][e] = r >= c ? a.C[r + (int64_t)c * a.ld] : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = tm * 32 + i * 8 + (lane >> 2), c = tn * 32 + j * 8 + 2 * (lane & 3) + e;
        if (r >= c) a.C[r + (int64_t)c * a.ld] = cv[i][j][e] - acc[i][j][e];
      }
}

}  // namespace

cudaError_t launch_next_tile(const NextTileArgs& a, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(next_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT_SMEM);
  if (e != cudaSuccess) return e;
  next_tile_kernel<<<1, NTH, NT_SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace dpp
