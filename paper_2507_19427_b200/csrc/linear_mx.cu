// linear_mx.cu — decode-shaped weight-streaming GEMM with MXFP8 operands
// (afdk_linear_mx): the attention projections in the FP8 GEMM form the paper
// measures (the Step-3 card is FP8 everywhere).
//
// Y[m_tok, n_out] = dequant(Xq)[m_tok, K] . dequant(Wq)[n_out, K]^T, e4m3
// codes with one UE8M0 scale per 32 elements along K (OCP MX) on both
// operands, fp32 accumulation in TMEM through the hardware block-scaled MMA
// (tcgen05.mma kind::mxf8f6f4.block_scale): half the weight bytes of the bf16
// projections and twice the tensor rate.  The schedule is linear.cu's: swap-AB
// (128 weight rows = MMA M, the <= 256 tokens = N), the (tile, 128-wide
// k-block) units cut stream-K over all SMs, fp32 segment partials in the same
// layout, so linear.cu's store kernel and the layer's row epilogues consume
// them unchanged.  Scale factors reach the tensor core through TMEM: per
// pipeline stage the four stager warps write one 32-bit word (the 4 k-steps'
// UE8M0 bytes) per weight row and per token row — column j, lane i of every
// subpartition = row 32j + i — read from smem, where the producer's TMA put
// each stage's 16-byte scale boxes (the 4-k-block group holding the stage's
// word: 16 B x 128 weight rows, 16 B x N token rows) with its operand tiles.
//
// Roles (320 threads): w0 TMA producer, w1 MMA issuer + TMEM owner, w2-5
// epilogue, w6-9 scale stagers.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "afdk_internal.h"
#include "linear.cuh"
#include "sm100.cuh"

namespace afdk {
namespace linmx {

using namespace sm100;

constexpr int kThreads = 320;
constexpr int kA = 128 * 128;          // one 128-row x 128-element e4m3 weight k-block
// scale ring after the accumulators: per stage 4 weight columns + one column
// per 32 token rows (N <= 256: 8, or 12 in the two-MMA form for N <= 384)
template <bool kW> struct SfRing;
template <> struct SfRing<false> { static constexpr uint32_t col0 = 256; static constexpr int cols = 12; };
// (the two-MMA form keeps each half's token columns at a 4-aligned offset: 4.. and 12..)
template <> struct SfRing<true> { static constexpr uint32_t col0 = 384; static constexpr int cols = 20; };

struct KParams {
  LinearPlan plan;        // kblocks = K / 128
  float* part;            // [(tiles + G)][m_tok][128] fp32 segment partials
  const uint8_t* w_sf;    // UE8M0 [n_out, K/32]
  const uint8_t* x_sf;    // UE8M0 [m_tok, K/32]
  int k_words;            // K / 128: 32-bit scale words per row
  int stage_bytes, stages;
  int w_dep;              // the weights are a predecessor's output: no PDL prefill
};

__device__ __forceinline__ void unit_range(int c, int G, int U, int& lo, int& hi) {
  lo = (int)(((long long)c * U) / G);
  hi = (int)(((long long)(c + 1) * U) / G);
}

// kW: 257-384 tokens as two MMAs of N/2 (N a multiple of 64) sharing each
// weight k-block, the accumulator single-buffered in TMEM columns [0, N)
template <bool kW>
__global__ void __launch_bounds__(kThreads, 1)
linear_mx_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                 const __grid_constant__ CUtensorMap tm_wsf, const __grid_constant__ CUtensorMap tm_xsf,
                 const KParams kp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const LinearPlan& P = kp.plan;
  const int S = kp.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kp.stage_bytes);
  uint64_t* sf_full = full + S;
  uint64_t* empty = sf_full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int U = P.tiles * P.kblocks;
  int u_lo, u_hi;
  unit_range(cta, G, U, u_lo, u_hi);
  const int n_mma = P.n_mma;
  const bool dbuf = n_mma <= 128;  // double-buffered accumulators while 2 x N columns fit before the scales
  constexpr uint32_t kSfCol0 = SfRing<kW>::col0;
  constexpr int kSfCols = SfRing<kW>::cols;
  const int nh = kW ? n_mma / 2 : n_mma;  // token rows per MMA

  const int xb = n_mma * 128;        // token panel bytes per stage
  const int sfw_off = kA + xb;       // stage layout: W | X | W scales (2 KB) | X scales (16 B per row)
  const int sfx_off = sfw_off + 128 * 16;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wsf);
    tma_prefetch_desc(&tm_xsf);
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&sf_full[i], 4); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_launch();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const uint32_t bytes = kA + xb + 128 * 16 + n_mma * 16;
      // weights (and their scales) never depend on the previous kernel: fill
      // the first stages' weight panels before waiting for the predecessor
      const int pro = min(S, u_hi - u_lo);
      if (kp.w_dep) griddep_wait();
      for (int i = 0; i < pro; ++i) {
        const int u = u_lo + i, tile = u / P.kblocks, kb = u % P.kblocks;
        uint8_t* st = smem + i * kp.stage_bytes;
        mbar_expect_tx(&full[i], bytes);
        tma_load_2d(st, &tm_w, &full[i], kb * 128, tile * 128, pol_w);
        tma_load_2d(st + sfw_off, &tm_wsf, &full[i], (kb >> 2) * 16, tile * 128, pol_w);
      }
      if (!kp.w_dep) griddep_wait();
      for (int i = 0; i < pro; ++i) {
        const int u = u_lo + i, kb = u % P.kblocks;
        uint8_t* st = smem + i * kp.stage_bytes;
        tma_load_2d(st + kA, &tm_x, &full[i], kb * 128, 0, pol_x);
        tma_load_2d(st + sfx_off, &tm_xsf, &full[i], (kb >> 2) * 16, 0, pol_x);
        if (kW) {
          tma_load_2d(st + kA + nh * 128, &tm_x, &full[i], kb * 128, nh, pol_x);
          tma_load_2d(st + sfx_off + nh * 16, &tm_xsf, &full[i], (kb >> 2) * 16, nh, pol_x);
        }
      }
      for (int u = u_lo + pro, i = pro; u < u_hi; ++u, ++i) {
        const int s = i % S, n = i / S;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        const int tile = u / P.kblocks, kb = u % P.kblocks;
        uint8_t* st = smem + s * kp.stage_bytes;
        mbar_expect_tx(&full[s], bytes);
        tma_load_2d(st, &tm_w, &full[s], kb * 128, tile * 128, pol_w);
        tma_load_2d(st + kA, &tm_x, &full[s], kb * 128, 0, pol_x);
        tma_load_2d(st + sfw_off, &tm_wsf, &full[s], (kb >> 2) * 16, tile * 128, pol_w);
        tma_load_2d(st + sfx_off, &tm_xsf, &full[s], (kb >> 2) * 16, 0, pol_x);
        if (kW) {
          tma_load_2d(st + kA + nh * 128, &tm_x, &full[s], kb * 128, nh, pol_x);
          tma_load_2d(st + sfx_off + nh * 16, &tm_xsf, &full[s], (kb >> 2) * 16, nh, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      griddep_wait();
      const uint32_t idesc = idesc_mxf8(128, (uint32_t)nh);
      int seg = 0;
      for (int u = u_lo, i = 0; u < u_hi; ++seg) {
        const int tile = u / P.kblocks;
        const int seg_end = min(u_hi, (tile + 1) * P.kblocks);
        const int ab = dbuf ? (seg & 1) : 0, na = dbuf ? (seg >> 1) : seg;
        if (dbuf ? seg >= 2 : seg >= 1) mbar_wait(&acc_empty[ab], (na & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * 128;
        for (bool first = true; u < seg_end; ++u, ++i, first = false) {
          const int s = i % S, n = i / S;
          mbar_wait(&full[s], n & 1);
          mbar_wait(&sf_full[s], n & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * kp.stage_bytes);
          const uint32_t b_base = a_base + kA;
          const uint32_t sf = tmem + kSfCol0 + (uint32_t)(s * kSfCols);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = sdesc_sw128(a_base + kk * 32, 0, 1024);
            const uint64_t db = sdesc_sw128(b_base + kk * 32, 0, 1024);
            const uint32_t sel = (uint32_t)kk << 30;
            mma_mxf8(d, da, db, idesc | idesc_sf_ids(kk, kk), sf | sel, (sf + 4) | sel, (first && kk == 0) ? 0u : 1u);
            if (kW) {  // tokens [N/2, N): the panel's second half, accumulator columns N/2.., scale columns 12..
              const uint64_t db2 = sdesc_sw128(b_base + nh * 128 + kk * 32, 0, 1024);
              mma_mxf8(d + nh, da, db2, idesc | idesc_sf_ids(kk, kk), sf | sel, (sf + 12) | sel,
                       (first && kk == 0) ? 0u : 1u);
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[ab]);
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------------ scale stagers
    // every subpartition holds the same words: column j, lane i = row 32j + i
    const int sp = warp & 3;
    const uint32_t t_lane = tmem + ((uint32_t)(sp * 32) << 16);
    const int nx = (n_mma + 31) >> 5;  // token columns
    for (int u = u_lo, i = 0; u < u_hi; ++u, ++i) {
      const int s = i % S, n = i / S;
      const int kb = u % P.kblocks;
      mbar_wait(&full[s], n & 1);  // the stage's tiles and scale boxes have landed
      if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);  // the TMEM scale slot's previous MMAs are done
      // row r's 4 group words sit at r * 16 bytes of its box; this stage's word is (kb & 3)
      const uint32_t* gw = reinterpret_cast<const uint32_t*>(smem + s * kp.stage_bytes + sfw_off) + (kb & 3);
      const uint32_t* gx = reinterpret_cast<const uint32_t*>(smem + s * kp.stage_bytes + sfx_off) + (kb & 3);
      uint32_t wv[4], xv[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = gw[(32 * j + lane) * 4];
      const int nxh = kW ? nx / 2 : nx;  // token columns per MMA
#pragma unroll
      for (int j = 0; j < 8; ++j) xv[j] = j < nxh ? gx[(32 * j + lane) * 4] : 0u;
      const uint32_t col = t_lane + kSfCol0 + (uint32_t)(s * kSfCols);
      tmem_st4(col, wv[0], wv[1], wv[2], wv[3]);
      tmem_st4(col + 4, xv[0], xv[1], xv[2], xv[3]);
      if (nxh > 4) tmem_st4(col + 8, xv[4], xv[5], xv[6], xv[7]);
      if (kW) {  // the second MMA's token rows [N/2, N) at columns 12..
#pragma unroll
        for (int j = 0; j < 8; ++j) xv[j] = j < nxh ? gx[(nh + 32 * j + lane) * 4] : 0u;
        tmem_st4(col + 12, xv[0], xv[1], xv[2], xv[3]);
        if (nxh > 4) tmem_st4(col + 16, xv[4], xv[5], xv[6], xv[7]);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sf_full[s]);
    }
  } else {
    // ---------------------------------------------------------- epilogue
    // TMEM lane = weight row = output feature, column = token; each (tile,
    // k-range) segment writes its fp32 partial to slot tile + cta
    const int sub = warp & 3;
    const int feat = sub * 32 + lane;
    int seg = 0;
    for (int u = u_lo; u < u_hi; ++seg) {
      const int tile = u / P.kblocks;
      const int seg_end = min(u_hi, (tile + 1) * P.kblocks);
      u = seg_end;
      const int ab = dbuf ? (seg & 1) : 0, na = dbuf ? (seg >> 1) : seg;
      mbar_wait(&acc_full[ab], na & 1);
      tc_fence_after();
      float* dst = kp.part + ((size_t)(tile + cta) * P.m_tok) * lin::kBM + feat;
      const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16) + ab * 128;
      for (int c = 0; c < n_mma; c += 32) {
        uint32_t v[32];
        tmem_ld32(t_row + c, v);
        tmem_wait_ld();
        float* d = dst + (size_t)c * lin::kBM;
        const int nv = P.m_tok - c;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) d[j * lin::kBM] = __uint_as_float(v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace linmx

// Plan of the MXFP8 linear: 128-row tiles, 128-element k-blocks.
LinearPlan make_linear_mx_plan(int m_tok, int n_out, int k) {
  LinearPlan p = make_linear_plan(m_tok, n_out, k);
  if (p.n_mma > 256) p.n_mma = ((m_tok + 63) / 64) * 64;  // two MMAs of N/2, each a multiple of 32 rows
  p.mtile = lin::kBM;
  p.tiles = (n_out + lin::kBM - 1) / lin::kBM;
  p.kblocks = k / 128;
  return p;
}

cudaError_t linear_mx_launch(Ctx& ctx, const LinearPlan& p, const void* xq, const uint8_t* xsf, const void* wq,
                             const uint8_t* wsf, float* part, cudaStream_t stream, bool w_dep) {
  using namespace linmx;
  const bool wide = p.n_mma > 256;
  if (p.n_mma > 384 || (wide && p.n_mma % 64) || p.k % 128) return cudaErrorInvalidValue;
  CUtensorMap tw, tx, twsf, txsf;
  {
    const uint64_t dims[2] = {(uint64_t)(p.k / 32), (uint64_t)p.n_out};
    const uint64_t strides[1] = {(uint64_t)(p.k / 32)};
    const uint32_t box[2] = {16, 128};
    if (!encode_tma(ctx, &twsf, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(wsf), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)(p.k / 32), (uint64_t)p.m_tok};
    const uint64_t strides[1] = {(uint64_t)(p.k / 32)};
    const uint32_t box[2] = {16, (uint32_t)(wide ? p.n_mma / 2 : p.n_mma)};
    if (!encode_tma(ctx, &txsf, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(xsf), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.n_out};
    const uint64_t strides[1] = {(uint64_t)p.k};
    const uint32_t box[2] = {128, 128};
    if (!encode_tma(ctx, &tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(wq), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.m_tok};
    const uint64_t strides[1] = {(uint64_t)p.k};
    const uint32_t box[2] = {128, (uint32_t)(wide ? p.n_mma / 2 : p.n_mma)};
    if (!encode_tma(ctx, &tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(xq), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  KParams kp{};
  kp.plan = p;
  kp.part = part;
  kp.w_sf = wsf;
  kp.x_sf = xsf;
  kp.k_words = p.k / 128;
  kp.w_dep = w_dep ? 1 : 0;
  kp.stage_bytes = (int)align_up((size_t)kA + p.n_mma * 128 + 128 * 16 + p.n_mma * 16, 1024);
  kp.stages = (200 * 1024) / kp.stage_bytes;
  if (kp.stages > (wide ? 8 : 10)) kp.stages = wide ? 8 : 10;
  const size_t smem = (size_t)kp.stages * kp.stage_bytes + 1024 + 512;
  const int grid = linear_grid(ctx, p);
  auto go = [&](auto kernel) -> cudaError_t {
    if (const cudaError_t e = ensure_smem(kernel, smem); e != cudaSuccess) return e;
    return launch_k(ctx.pdl, kernel, dim3(grid), dim3(kThreads), smem, stream, tw, tx, twsf, txsf, kp);
  };
  return wide ? go(linear_mx_kernel<true>) : go(linear_mx_kernel<false>);
}

}  // namespace afdk
