// linear.cuh — plan of the stream-K weight-streaming GEMM and the fixed-order
// partial reduction shared by every row epilogue.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afdk {

struct LinearPlan {
  int m_tok;    // decode tokens (rows of X / Y), <= 512
  int n_mma;    // m_tok rounded up to the MMA N granularity (16)
  int n_out;    // output features (rows of W)
  int k;        // reduction dim, multiple of 64
  int tiles;    // ceil(n_out / mtile)
  int kblocks;  // k / 64
  int mtile;    // weight rows per work tile: 128, or 256 (two MMA panels sharing the
                // token panel) once the token panel is wide (L2->smem bytes per FLOP)
};

namespace lin {
constexpr int kBM = 128;
constexpr int kMaxSegs = 16;    // CTAs that may share one tile (linear_grid caps G)
constexpr int kMaxTiles = 128;  // tiles a row epilogue may span (n_out <= 16384)

// Which partial slots hold tile t: CTAs c_lo[t] .. c_lo[t]+n[t]-1 (the grid
// never has empty CTAs), slot = t + c.  Built once per epilogue CTA in smem.
struct SlotTable {
  int c_lo[kMaxTiles];
  int n[kMaxTiles];
  __device__ __forceinline__ float sum(const LinearPlan& P, const float* __restrict__ part, int row,
                                       int f) const {
    const int t = f / P.mtile, c0 = c_lo[t], nn = n[t];
    const float* base = part + ((size_t)(t + c0) * P.m_tok + row) * P.mtile + (f % P.mtile);
    const size_t stride = (size_t)P.m_tok * P.mtile;
    float acc = 0.0f;
#pragma unroll 4
    for (int k = 0; k < nn; ++k) acc += __ldcg(base + (size_t)k * stride);
    return acc;
  }
  // features f..f+3 (f % 4 == 0, one tile): one 16-byte load per segment
  __device__ __forceinline__ float4 sum4(const LinearPlan& P, const float* __restrict__ part, int row,
                                         int f) const {
    const int t = f / P.mtile, c0 = c_lo[t], nn = n[t];
    const float4* base =
        reinterpret_cast<const float4*>(part + ((size_t)(t + c0) * P.m_tok + row) * P.mtile + (f % P.mtile));
    const size_t stride = (size_t)P.m_tok * P.mtile / 4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int k = 0; k < nn; ++k) {
      const float4 v = __ldcg(base + (size_t)k * stride);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    return acc;
  }
};

__device__ __forceinline__ void build_slot_table(const LinearPlan& P, int G, SlotTable& tab) {
  const long long U = (long long)P.tiles * P.kblocks;
  for (int t = threadIdx.x; t < P.tiles; t += blockDim.x) {
    const long long u0 = (long long)t * P.kblocks, u1 = u0 + P.kblocks;  // [u0, u1)
    const int c_lo = (int)((u0 * G) / U);   // CTA c owns [cU/G, (c+1)U/G): floor-based
    int lo = c_lo;
    while (lo > 0 && ((long long)lo * U) / G > u0) --lo;
    while (((long long)(lo + 1) * U) / G <= u0) ++lo;
    int hi = (int)(((u1 - 1) * G) / U);
    while (hi > 0 && ((long long)hi * U) / G > u1 - 1) --hi;
    while (((long long)(hi + 1) * U) / G <= u1 - 1) ++hi;
    tab.c_lo[t] = lo;
    tab.n[t] = hi - lo + 1;
  }
  __syncthreads();
}
}  // namespace lin

}  // namespace afdk
