// next_tile.cu -- the chain's two one-tile GEMMs of a split step fused into one CTA (real fp64,
// nb = 128): the first row tile of the panel and the lookahead update of the next diagonal tile.
//
// Listing 3, for the rows of the NEXT block only (reading R17: the panel solve as
// a GEMM with the diag kernel's tile operator Bm):
//   P0:  L21_0 = A21_0 - A21_0 Bm^T               (rows j1 .. j1+127 of block column j0; in place)
//        W21_0 = L21_0 D1                          (the pre-scaled copy, into its panel slot)
//   LT:  A22_00 -= W21_0 L21_0^T                   (lower triangle of the next diagonal tile)
// In the split schedule (driver.cu, run_blocked) these two products are all the next diag tile
// waits for; as two update-kernel launches they cost ~30 us each on one SM (launch, ring fill,
// C round trip, epilogue), and fused in one CTA ~40 us (round 2, first version).  Here they run on
// a cluster of 4 CTAs (4 SMs): each computes P0 for 32 rows, the CTAs exchange their rows of L21_0
// through distributed shared memory, and each computes a share of LT's lower-triangle tiles.
//
// Bitwise contract: every output equals the unfused launches' (update_ws_kernel): the same DMMA.8x8x4
// sequence per output element (k-quads in increasing order; the panel's 32-wide column group wn
// stops at k = 32 wn + 32 like the triangular-operator cut `btri` of the update kernel), the same
// "C - acc" subtraction and the same W = L d products (LT's A operand is formed in registers by the
// same multiply the panel epilogue stores).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace dpp {
namespace {

constexpr int NB = 128, LDS = NB + 4;

// ---- the same two products on a cluster of 4 CTAs (4 SMs), one 32-row block of the tile each.
// CTA q: P0 for rows 32q .. 32q+31 (8 warps, 32 x 16 warp tiles, warp w's columns 16w .. 16w+15 use
// k < 32 (w/2 + 1) like the 32-wide warp column w/2 of the one-CTA kernel), then, after a cluster
// barrier, every CTA copies the whole L21_0 (4 x 32 rows) from its peers' shared memory (DSMEM)
// and computes LT tiles t = q, q+4, q+8 of the 10 lower-triangle 32 x 32 tiles (row-major), each
// by two warps of 32 x 16.  Per output element the k-quads are accumulated in the same increasing
// order with the same DMMA.8x8x4 and the same operand products as the one-CTA kernel: bit-identical.
constexpr int CL = 4, RB = NB / CL, LDR = RB + 4, CNT = 256;
constexpr size_t CL_SMEM = (size_t)(NB * LDR + NB * LDS) * 8;

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CNT, 1) next_tile_cluster_kernel(const NextTileArgs a) {
  namespace cgx = cooperative_groups;
  cgx::cluster_group cluster = cgx::this_cluster();
  extern __shared__ __align__(16) double sm[];
  double* Lr = sm;               // [k][LDR]: this CTA's 32 rows of A21_0, then of L21_0 in place
  double* Bf = sm + NB * LDR;    // [k][LDS]: Bm (P0), then the whole L21_0 (LT)
  const int q = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- loads: my rows of A21_0 (k-major) and all of Bm
  for (int idx = tid; idx < NB * (RB / 2); idx += CNT) {
    const int k = idx / (RB / 2), r2 = idx % (RB / 2);
    cp_async16(&Lr[k * LDR + 2 * r2], a.A21 + (int64_t)k * a.ld + RB * q + 2 * r2, 16);
  }
  for (int idx = tid; idx < NB * (NB / 2); idx += CNT) {
    const int k = idx / (NB / 2), n2 = idx % (NB / 2);
    cp_async16(&Bf[k * LDS + 2 * n2], a.Bm + (int64_t)k * a.ldm + 2 * n2, 16);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // ---- P0 on my rows: warp w, columns 16w .. 16w+15, k < 32 (w/2 + 1)
  {
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int kq_end = 8 * (warp / 2 + 1);  // k-quads
    for (int kq = 0; kq < kq_end; ++kq) {
      const int k = kq * 4 + (lane & 3);
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Lr[k * LDR + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bf[k * LDS + 16 * warp + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();  // every warp has read Lr as its A operand
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = 16 * warp + j * 8 + 2 * (lane & 3) + e;
          Lr[c * LDR + r] = Lr[c * LDR + r] - acc[i][j][e];
        }
    }
  }
  __syncthreads();
  // L21_0 rows -> A21 (in place) and W21_0 = L21_0 D1 -> its panel slot
  for (int idx = tid; idx < NB * RB; idx += CNT) {
    const int c = idx / RB, r = idx % RB;
    const double l = Lr[c * LDR + r];
    a.A21[RB * q + r + (int64_t)c * a.ld] = l;
    a.W21[RB * q + r + (int64_t)c * a.ldw] = scal(l, __ldg(a.d + c));
  }
  // ---- every CTA's L21_0 rows are final: gather the whole L21_0 into Bf (Bm is no longer needed)
  cluster.sync();
  for (int p = 0; p < CL; ++p) {
    const double* src = cluster.map_shared_rank(Lr, p);
    for (int idx = tid; idx < NB * (RB / 2); idx += CNT) {
      const int k = idx / (RB / 2), r2 = idx % (RB / 2);
      *reinterpret_cast<double2*>(&Bf[k * LDS + RB * p + 2 * r2]) =
          *reinterpret_cast<const double2*>(&src[k * LDR + 2 * r2]);
    }
  }
  cluster.sync();  // (no CTA leaves while a peer still reads its shared memory)

  // ---- LT: tile t = q + 4 (warp / 2) (if < 10), columns 16 (warp & 1) .. of the tile
  const int t = q + CL * (warp >> 1);
  if (t >= 10) return;
  int tm = 0, tn = t;
  while (tn > tm) { tn -= tm + 1; ++tm; }
  const int h = warp & 1;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int kq = 0; kq < NB / 4; ++kq) {
    const int k = kq * 4 + (lane & 3);
    const double dk = __ldg(a.d + k);
    double af[4], bf[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = scal(Bf[k * LDS + tm * 32 + i * 8 + (lane >> 2)], dk);
#pragma unroll
    for (int j = 0; j < 2; ++j) bf[j] = Bf[k * LDS + tn * 32 + 16 * h + j * 8 + (lane >> 2)];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  double cv[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = tm * 32 + i * 8 + (lane >> 2), c = tn * 32 + 16 * h + j * 8 + 2 * (lane & 3) + e;
        cv[i][j][e] = r >= c ? a.C[r + (int64_t)c * a.ld] : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = tm * 32 + i * 8 + (lane >> 2), c = tn * 32 + 16 * h + j * 8 + 2 * (lane & 3) + e;
        if (r >= c) a.C[r + (int64_t)c * a.ld] = cv[i][j][e] - acc[i][j][e];
      }
}

}  // namespace

cudaError_t launch_next_tile(const NextTileArgs& a, cudaStream_t s) {
  cudaError_t e = cudaFuncSetAttribute(next_tile_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)CL_SMEM);
  if (e != cudaSuccess) return e;
  next_tile_cluster_kernel<<<CL, CNT, CL_SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace dpp
