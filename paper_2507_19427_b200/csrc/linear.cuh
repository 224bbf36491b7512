// linear.cuh — plan of the stream-K weight-streaming GEMM and the fixed-order
// partial reduction shared by every row epilogue.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afdk {

struct LinearPlan {
  int m_tok;    // decode tokens (rows of X / Y), <= 256
  int n_mma;    // m_tok rounded up to the MMA N granularity (16)
  int n_out;    // output features (rows of W)
  int k;        // reduction dim, multiple of 64
  int tiles;    // ceil(n_out / 128)
  int kblocks;  // k / 64
};

namespace lin {
constexpr int kBM = 128;

// Sum, in CTA order, of the partials covering (row, feature f).  CTA c owns the
// unit range [c*U/G, (c+1)*U/G) of U = tiles*kblocks units; the partial of the
// (tile, c) segment lives in slot tile + c (layout [slot][m_tok][128]).
__device__ __forceinline__ float linear_partial_sum(const LinearPlan& P, const float* __restrict__ part,
                                                    int G, int row, int f) {
  const int tile = f / kBM;
  const long long U = (long long)P.tiles * P.kblocks;
  const long long u0 = (long long)tile * P.kblocks, u1 = u0 + P.kblocks - 1;
  int c = (int)((u0 * G) / U);
  while (c > 0 && ((long long)c * U) / G > u0) --c;
  while (((long long)(c + 1) * U) / G <= u0) ++c;
  float acc = 0.0f;
  for (;; ++c) {
    const long long lo = ((long long)c * U) / G, hi = ((long long)(c + 1) * U) / G;
    if (lo > u1) break;
    if (hi > lo) acc += __ldg(part + ((size_t)(tile + c) * P.m_tok + row) * kBM + (f % kBM));
  }
  return acc;
}
}  // namespace lin

}  // namespace afdk
