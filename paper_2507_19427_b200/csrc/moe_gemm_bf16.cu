// moe_gemm_bf16.cu — K7/K8 with 16-bit expert weights: grouped bf16 expert
// GEMMs on tcgen05.mma kind::f16.
//
// The reference models the FFN's compute format as a first-class quant
// setting (QuantScheme.weight_bytes / compute_kind, types.hpp:34-40;
// effective_kind, types.hpp:93-95); the paper runs BF16 where FP8 is not
// available.  Same two GEMMs per gated expert as the FP8
// kernels (builtin_catalog.cpp:248-251) and the same swap-AB orientation: a
// 128-row weight tile is MMA M, up to 128 dispatched token rows are N, K
// streams in 64-element (128-byte) k-blocks through a TMA ring.  No scale
// factors: the accumulator spans the whole K loop in TMEM.
//
// W13 (kGLU): gate and up tiles of the same 128 intermediate features land in
// one stage, two accumulators (gate | up) in TMEM columns [0,256); the
// epilogue writes h = SiLU(gate) * up in bf16.  W2: two 128-column
// accumulators so the epilogue of item i overlaps the MMAs of item i+1; fp32
// outputs for the combine.
//
// Items are ordered (expert, m-tile, chunk) (moe.cuh item_of), so an expert's
// chunks share each weight tile while it is in L2.
//
// Items carry up to 128 token rows, or 256 once experts average >= 128 rows
// (MMA N = 256 halves the L2->smem bytes per FLOP, the limit of the 128-row
// form at large batches; gate | up then fill all 512 TMEM columns).
//
// Roles (192 threads): w0 TMA producer, w1 MMA issuer + TMEM owner, w2-5
// epilogue (one TMEM subpartition each).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "afdk_internal.h"
#include "moe.cuh"
#include "sm100.cuh"

namespace afdk {
namespace moe {

using namespace sm100;

constexpr int kBfThreads = 192;

struct BfGemmParams {
  const Work* work;
  const int* n_work;
  int m_tiles;    // output features / 128 (W13: per half)
  int kblocks;    // K / 64
  int w_rows;     // weight rows per expert (W13: 2I, W2: H)
  int up_offset;  // W13: row offset of the up half (= I)
  int E, expert_lo, n_local;
  int out_cols;          // W13: I, W2: H
  __nv_bfloat16* h;      // W13 out: [rows_pad, I] bf16
  float* y;              // W2 out:  [rows_pad, H] fp32
  int stage_bytes, stages;
  int chunk;             // token rows per item: 128, or 256 at large batches (MMA N = 256:
                         // half the L2->smem bytes per FLOP; accumulators use all 512 TMEM columns)
};

template <bool kGLU>
__global__ void __launch_bounds__(kBfThreads, 1)
moe_gemm_bf16_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                     const BfGemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kA = 128 * 128;  // 128 weight rows x 64 bf16
  constexpr int kAOps = kGLU ? 2 : 1;
  const int kB = p.chunk * 128;
  const int acc_cols = p.chunk;  // one accumulator's TMEM columns
  const int S = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * p.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_items = *p.n_work * p.m_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // weights stream through L2 (read by one expert's chunks, adjacent
      // items); activation panels stay for the m-tiles that re-read them
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int i = 0;
      for (int it = cta; it < n_items; it += G) {
        const ItemRef ir = item_of(p.work, it, p.m_tiles);
        const Work wk = p.work[ir.chunk];
        const int wi = wk.group == p.E ? p.n_local : wk.group - p.expert_lo;
        const int wrow = wi * p.w_rows + ir.mt * 128;
        const int xrow = kGLU ? wk.xrow0 : wk.row0;
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
          if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
          uint8_t* st = smem + s * p.stage_bytes;
          mbar_expect_tx(&full[s], kAOps * kA + kB);
          tma_load_2d(st, &tm_w, &full[s], kb * 64, wrow, pol_w);
          if (kGLU) tma_load_2d(st + kA, &tm_w, &full[s], kb * 64, wrow + p.up_offset, pol_w);
          tma_load_2d(st + kAOps * kA, &tm_x, &full[s], kb * 64, xrow, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int i = 0, li = 0;
      for (int it = cta; it < n_items; it += G, ++li) {
        const Work wk = p.work[item_of(p.work, it, p.m_tiles).chunk];
        const int b = kGLU ? 0 : (li & 1);
        const int nb = kGLU ? li : (li >> 1);
        if (nb > 0) mbar_wait(&acc_empty[b], (nb & 1) ^ 1);
        tc_fence_after();
        const uint32_t idesc = idesc_bf16(128, (uint32_t)((wk.rows + 15) & ~15), false, false);
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
          mbar_wait(&full[s], n & 1);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * p.stage_bytes);
          const uint32_t b_base = base + kAOps * kA;
#pragma unroll
          for (int op = 0; op < kAOps; ++op) {
            const uint32_t d = tmem + (uint32_t)((kGLU ? op : b) * acc_cols);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K = 16 bf16 = 32 bytes per MMA
              mma_bf16(d, sdesc_sw128(base + op * kA + kk * 32, 0, 1024), sdesc_sw128(b_base + kk * 32, 0, 1024),
                       idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[s]);
          if (kb == p.kblocks - 1) mma_commit(&acc_full[b]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int sub = warp & 3, feat = sub * 32 + lane;  // feature row within the tile
    const uint32_t t_lane = tmem + ((uint32_t)(sub * 32) << 16);
    int li = 0;
    for (int it = cta; it < n_items; it += G, ++li) {
      const ItemRef ir = item_of(p.work, it, p.m_tiles);
      const Work wk = p.work[ir.chunk];
      const int b = kGLU ? 0 : (li & 1);
      const int nb = kGLU ? li : (li >> 1);
      mbar_wait(&acc_full[b], nb & 1);
      tc_fence_after();
      const int col = ir.mt * 128 + feat;
#pragma unroll 1
      for (int c = 0; c < p.chunk / 32; ++c) {
        if (c * 32 >= wk.rows) break;
        uint32_t v[32];
        tmem_ld32(t_lane + b * acc_cols + c * 32, v);
        if (kGLU) {
          uint32_t u[32];
          tmem_ld32(t_lane + acc_cols + c * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int r = c * 32 + j;
            if (r < wk.rows) {
              const float g = __uint_as_float(v[j]);
              const float hv = silu_fast(g) * __uint_as_float(u[j]);
              p.h[((size_t)wk.row0 + r) * p.out_cols + col] = __float2bfloat16_rn(hv);
            }
          }
        } else {
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int r = c * 32 + j;
            if (r < wk.rows) p.y[((size_t)wk.row0 + r) * p.out_cols + col] = __uint_as_float(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace moe

cudaError_t moe_gemm_bf16_launch(Ctx& ctx, bool glu, const MoeGemmBf16Args& a, cudaStream_t stream) {
  using namespace moe;
  const int K = glu ? a.H : a.I;
  const int w_rows = glu ? 2 * a.I : a.H;
  CUtensorMap tw, tx;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(a.n_local + 1) * w_rows};
    const uint64_t strides[1] = {(uint64_t)K * 2};
    const uint32_t box[2] = {64, 128};
    if (!encode_tma(ctx, &tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.w), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)a.rows_pad};
    const uint64_t strides[1] = {(uint64_t)K * 2};
    const uint32_t box[2] = {64, (uint32_t)a.chunk};
    if (!encode_tma(ctx, &tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.x), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  BfGemmParams p{};
  p.work = a.work;
  p.n_work = a.n_work;
  p.m_tiles = glu ? a.I / 128 : a.H / 128;
  p.kblocks = K / 64;
  p.w_rows = w_rows;
  p.up_offset = glu ? a.I : 0;
  p.E = a.E;
  p.expert_lo = a.expert_lo;
  p.n_local = a.n_local;
  p.out_cols = glu ? a.I : a.H;
  p.h = a.h;
  p.y = a.y;
  p.chunk = a.chunk;
  p.stage_bytes = (glu ? 2 : 1) * 128 * 128 + a.chunk * 128;
  p.stages = (200 * 1024) / p.stage_bytes;
  if (p.stages > 8) p.stages = 8;
  const size_t smem = (size_t)p.stages * p.stage_bytes + 1024 + 256;
  cudaError_t e;
  if (glu) {
    if ((e = ensure_smem(moe_gemm_bf16_kernel<true>, smem)) != cudaSuccess) return e;
    return launch_k(ctx.pdl, moe_gemm_bf16_kernel<true>, dim3(ctx.num_sms), dim3(kBfThreads), smem, stream, tw, tx, p);
  }
  if ((e = ensure_smem(moe_gemm_bf16_kernel<false>, smem)) != cudaSuccess) return e;
  return launch_k(ctx.pdl, moe_gemm_bf16_kernel<false>, dim3(ctx.num_sms), dim3(kBfThreads), smem, stream, tw, tx, p);
}

}  // namespace afdk
