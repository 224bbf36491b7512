// moe_gemm_mx.cu — K7/K8 for large FFN batches: grouped MXFP8 expert GEMMs on
// the hardware block-scaled tensor-core path (tcgen05.mma kind::mxf8f6f4
// .block_scale).
//
// Same two GEMMs per gated expert as moe_gemm.cu (builtin_catalog.cpp:248-251,
// 3*h*inter params per expert) and the same swap-AB orientation (a 128-row
// weight tile is MMA M, up to 128 dispatched rows are N), but the operands carry
// one UE8M0 scale per 32 K elements (OCP MX) and the tensor core applies them
// inside the MMA.  The accumulator therefore spans the whole K loop in TMEM:
// no per-k-block promotion by the epilogue warps, which is what bounds the
// 1x128/128x128 software-scaled kernel once batches are large (PAPER.md:651,
// the FFN side at hundreds of tokens per expert).
//
// Scale factors reach the tensor core through TMEM.  Per pipeline stage (one
// 128-wide k-block) a ring slot holds 4 columns per operand; column j, lane i
// of every 32-lane subpartition holds the 4 packed UE8M0 bytes (k sub-blocks
// 0..3) of row 32j+i, and the k-step kk of the MMA selects byte kk through
// the instruction descriptor's sf ids.  The producer TMA-loads the packed
// scales of 4 k-blocks at a time (one 16 B x 128-row box per operand, from the
// row-major [rows, K/32] UE8M0 arrays) into a 2-slot smem ring; four stager
// warps (one per TMEM subpartition) read them from smem and write the TMEM
// slot with tcgen05.st.
//
// Items are ordered chunk-major (all m-tiles of a chunk, then the next chunk;
// an expert's chunks are adjacent), so the ~148 concurrently running items
// cover a few chunks of one or two experts: each weight tile is fetched from
// HBM about once and shared in L2 by the expert's chunks, each activation
// panel by the m-tiles of its chunk.
//
// Roles (320 threads): w0 TMA producer, w1 MMA issuer + TMEM owner, w2-5
// epilogue, w6-9 scale stagers.  TMEM: accumulators in columns [0,256) (W13:
// gate | up of one item; W2: two 128-column buffers so the epilogue of item i
// overlaps the MMAs of item i+1), scale ring from column 256.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "afdk_internal.h"
#include "moe.cuh"
#include "sm100.cuh"

namespace afdk {
namespace moe {

using namespace sm100;

constexpr int kMxThreads = 320;
constexpr uint32_t kSfCol0 = 256;

struct MxGemmParams {
  const Work* work;
  const int* n_work;
  int m_tiles;          // output features / 128 (W13: per half)
  int kblocks;          // K / 128 (multiple of 4)
  int w_rows;           // weight rows per expert (W13: 2I, W2: H)
  int up_offset;        // W13: row offset of the up half (= I)
  const uint8_t* w_sf;  // [(n_local+1) * w_rows, K/32]
  const uint8_t* x_sf;  // [rows_pad, K/32]
  int E, expert_lo, n_local;
  int out_cols;         // W13: I, W2: H
  uint8_t* hq;          // W13 out: [rows_pad, I] e4m3
  uint8_t* hsf;         // W13 out: [rows_pad, I/32] UE8M0
  float* y;             // W2 out:  [rows_pad, H] fp32
  int stage_bytes, stages;
  int prefetch;         // L2-prefetch the first item's weights before the PDL wait
};

__device__ __forceinline__ int mx_weight_index(const MxGemmParams& p, int group) {
  return group == p.E ? p.n_local : group - p.expert_lo;
}

__device__ __forceinline__ int mx_exp(float amax) {
  const uint32_t u = __float_as_uint(amax);
  const int E = (int)((u >> 23) & 0xff);
  if (!(amax > 0.0f) || E == 0) return -127;
  const int e = ((u & 0x7fffffu) <= 6291456u) ? E - 135 : E - 134;
  return max(-127, min(127, e));
}

__device__ __forceinline__ uint32_t u4_get(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

template <bool kGLU>
__global__ void __launch_bounds__(kMxThreads, 1)
moe_gemm_mx_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_wsf, const __grid_constant__ CUtensorMap tm_xsf,
                   const MxGemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kA = 128 * 128;
  constexpr int kAOps = kGLU ? 2 : 1;
  constexpr int kB = kChunkMX * 128;
  constexpr int kSfCols = 4 * kAOps + 4;       // scale columns per ring slot
  constexpr int kSfOp = 128 * 16;              // one operand's scales for 4 k-blocks
  constexpr int kSfGrp = (kAOps + 1) * kSfOp;  // smem scale group (4 k-blocks)
  const int S = p.stages;
  uint8_t* sfbuf = smem + S * p.stage_bytes;   // 2 x kSfGrp
  uint64_t* full = reinterpret_cast<uint64_t*>(sfbuf + 2 * kSfGrp);
  uint64_t* sf_full = full + S;
  uint64_t* empty = sf_full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* sfg_full = acc_empty + 2;
  uint64_t* sfg_empty = sfg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfg_empty + 2);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wsf);
    tma_prefetch_desc(&tm_xsf);
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&sf_full[i], 4); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
      mbar_init(&sfg_full[i], 1);
      mbar_init(&sfg_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (p.prefetch && warp == 0 && lane == 0) {
    // Before the PDL wait: weights never depend on the predecessor, and the
    // work list was written by the permute kernel, which completed before
    // this grid could launch (the predecessor launches us only after its own
    // griddepcontrol.wait).  CTAs that start on SMs the predecessor's last,
    // partial wave left idle stream their first item's weight tile into L2
    // while HBM is under-used, instead of idling at the wait.
    const int n0 = *p.n_work * p.m_tiles;
    if (cta < n0) {
      const ItemRef ir = item_of(p.work, cta, p.m_tiles);
      const Work wk = p.work[ir.chunk];
      const int wrow = mx_weight_index(p, wk.group) * p.w_rows + ir.mt * 128;
      for (int kb = 0; kb < p.kblocks; ++kb) {
        tma_prefetch_l2_2d(&tm_w, kb * 128, wrow);
        if (kGLU) tma_prefetch_l2_2d(&tm_w, kb * 128, wrow + p.up_offset);
      }
    }
  }
  griddep_wait();
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_work = *p.n_work;
  const int n_items = n_work * p.m_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // this kernel runs at decode batches: every weight tile is read by about
      // one item, so weights stream through L2 (evict_first) and leave it to
      // the activation panels shared by a chunk's m-tiles and to the y / hq
      // outputs the next kernel reads
      const uint64_t pol = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int i = 0, gi = 0;
      for (int it = cta; it < n_items; it += G) {
        const ItemRef ir = item_of(p.work, it, p.m_tiles);
        const int mt = ir.mt;
        const Work wk = p.work[ir.chunk];
        const int wrow = mx_weight_index(p, wk.group) * p.w_rows + mt * 128;
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          if ((kb & 3) == 0) {  // scale group of k-blocks kb..kb+3
            const int g = gi & 1, ng = gi >> 1;
            ++gi;
            if (ng > 0) mbar_wait(&sfg_empty[g], (ng & 1) ^ 1);
            uint8_t* dst = sfbuf + g * kSfGrp;
            mbar_expect_tx(&sfg_full[g], kSfGrp);
            tma_load_2d(dst, &tm_wsf, &sfg_full[g], kb * 4, wrow, pol);
            if (kGLU) tma_load_2d(dst + kSfOp, &tm_wsf, &sfg_full[g], kb * 4, wrow + p.up_offset, pol);
            tma_load_2d(dst + kAOps * kSfOp, &tm_xsf, &sfg_full[g], kb * 4, kGLU ? wk.xrow0 : wk.row0, pol_x);
          }
          const int s = i % S, n = i / S;
          if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
          uint8_t* st = smem + s * p.stage_bytes;
          mbar_expect_tx(&full[s], kAOps * kA + kB);
          tma_load_2d(st, &tm_w, &full[s], kb * 128, wrow, pol);
          if (kGLU) tma_load_2d(st + kA, &tm_w, &full[s], kb * 128, wrow + p.up_offset, pol);
          tma_load_2d(st + kAOps * kA, &tm_x, &full[s], kb * 128, kGLU ? wk.xrow0 : wk.row0, pol_x);
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
        const uint32_t n_mma = (uint32_t)((wk.rows + 15) & ~15);
        const uint32_t idesc = idesc_mxf8(128, n_mma);
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
          mbar_wait(&full[s], n & 1);
          mbar_wait(&sf_full[s], n & 1);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * p.stage_bytes);
          const uint32_t b_base = base + kAOps * kA;
          const uint32_t sf = tmem + kSfCol0 + (uint32_t)(s * kSfCols);
#pragma unroll
          for (int op = 0; op < kAOps; ++op) {
            const uint32_t d = tmem + (kGLU ? op * 128 : b * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = sdesc_sw128(base + op * kA + kk * 32, 0, 1024);
              const uint64_t db = sdesc_sw128(b_base + kk * 32, 0, 1024);
              const uint32_t sel = (uint32_t)kk << 30;
              mma_mxf8(d, da, db, idesc | idesc_sf_ids(kk, kk), (sf + op * 4) | sel, (sf + kAOps * 4) | sel,
                       (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (kb == p.kblocks - 1) mma_commit(&acc_full[b]);
        }
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------------ scale stagers
    const int sp = warp & 3;
    const uint32_t t_lane = tmem + ((uint32_t)(sp * 32) << 16);
    int i = 0, gi = 0;
    for (int it = cta; it < n_items; it += G) {
      for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
        const int g = gi & 1;
        if ((kb & 3) == 0) mbar_wait(&sfg_full[g], (gi >> 1) & 1);
        const int s = i % S, n = i / S;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        // row r's 4 packed k-block scales sit at r*16 bytes of the operand's box
        const uint32_t* grp = reinterpret_cast<const uint32_t*>(sfbuf + g * kSfGrp) + (kb & 3) + lane * 4;
        const uint32_t col = t_lane + kSfCol0 + (uint32_t)(s * kSfCols);
        tmem_st4(col, grp[0], grp[128], grp[256], grp[384]);
        if (kGLU) tmem_st4(col + 4, grp[512], grp[512 + 128], grp[512 + 256], grp[512 + 384]);
        const uint32_t* gb = grp + kAOps * 512;
        tmem_st4(col + kAOps * 4, gb[0], gb[128], gb[256], gb[384]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sf_full[s]);
          if ((kb & 3) == 3 || kb == p.kblocks - 1) mbar_arrive(&sfg_empty[g]);
        }
        if ((kb & 3) == 3 || kb == p.kblocks - 1) ++gi;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int sub = warp & 3, feat = sub * 32 + lane;  // feature row within the tile
    const uint32_t t_lane = tmem + ((uint32_t)(sub * 32) << 16);
    int li = 0;
    for (int it = cta; it < n_items; it += G, ++li) {
      const ItemRef ir = item_of(p.work, it, p.m_tiles);
      const int mt = ir.mt;
      const Work wk = p.work[ir.chunk];
      const int b = kGLU ? 0 : (li & 1);
      const int nb = kGLU ? li : (li >> 1);
      mbar_wait(&acc_full[b], nb & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kChunkMX / 32; ++c) {
        if (c * 32 >= wk.rows) break;
        uint32_t v[32];
        tmem_ld32(t_lane + b * 128 + c * 32, v);
        if (kGLU) {
          uint32_t u[32];
          tmem_ld32(t_lane + 128 + c * 32, u);
          tmem_wait_ld();
          // h = SiLU(gate) * up, re-quantised to MXFP8 over 32-feature blocks
          // (this warp's 32 lanes = one block of the tile)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float g = __uint_as_float(v[j]);
            const float h = silu_fast(g) * __uint_as_float(u[j]);
            float m = fabsf(h);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
            const int e = mx_exp(m);
            const float inv = e < 127 ? __uint_as_float((uint32_t)(127 - e) << 23) : __uint_as_float(1u << 22);
            const int r = c * 32 + j;
            if (r < wk.rows) {
              const size_t row = (size_t)wk.row0 + r;
              p.hq[row * p.out_cols + mt * 128 + feat] =
                  (uint8_t)__nv_cvt_float_to_fp8(h * inv, __NV_SATFINITE, __NV_E4M3);
              if (lane == 0) p.hsf[row * (p.out_cols / 32) + mt * 4 + sub] = (uint8_t)(e + 127);
            }
          }
        } else {
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int r = c * 32 + j;
            if (r < wk.rows) p.y[((size_t)wk.row0 + r) * p.out_cols + mt * 128 + feat] = __uint_as_float(v[j]);
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

cudaError_t moe_gemm_mx_launch(Ctx& ctx, bool glu, const MoeGemmMxArgs& a, cudaStream_t stream) {
  using namespace moe;
  CUtensorMap tw, tx;
  const int K = glu ? a.H : a.I;
  const int w_rows = glu ? 2 * a.I : a.H;
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)(a.n_local + 1) * w_rows};
    const uint64_t strides[1] = {(uint64_t)K};
    const uint32_t box[2] = {128, 128};
    if (!encode_tma(ctx, &tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(a.w), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)K, (uint64_t)a.rows_pad};
    const uint64_t strides[1] = {(uint64_t)K};
    const uint32_t box[2] = {128, kChunkMX};
    if (!encode_tma(ctx, &tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(a.x), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  CUtensorMap twsf, txsf;
  {
    const uint64_t dims[2] = {(uint64_t)(K / 32), (uint64_t)(a.n_local + 1) * w_rows};
    const uint64_t strides[1] = {(uint64_t)(K / 32)};
    const uint32_t box[2] = {16, 128};
    if (!encode_tma(ctx, &twsf, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.w_sf), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)(K / 32), (uint64_t)a.rows_pad};
    const uint64_t strides[1] = {(uint64_t)(K / 32)};
    const uint32_t box[2] = {16, 128};
    if (!encode_tma(ctx, &txsf, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.x_sf), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  MxGemmParams p{};
  p.work = a.work;
  p.n_work = a.n_work;
  p.m_tiles = glu ? a.I / 128 : a.H / 128;
  p.kblocks = K / 128;
  p.w_rows = w_rows;
  p.up_offset = glu ? a.I : 0;
  p.w_sf = a.w_sf;
  p.x_sf = a.x_sf;
  p.E = a.E;
  p.expert_lo = a.expert_lo;
  p.n_local = a.n_local;
  p.out_cols = glu ? a.I : a.H;
  p.hq = a.hq;
  p.hsf = a.hsf;
  p.y = a.y;
  p.stage_bytes = (glu ? 2 : 1) * 128 * 128 + kChunkMX * 128;
  // off by default: 48 local experts 0.969 vs 0.987 ms, but expert shards
  // (16 / 8 experts, the AFD FFN GPUs) 0.381 vs 0.374 and 0.238 vs 0.228 ms
  static const int prefetch = [] { const char* e = std::getenv("AFDK_MX_PREFETCH"); return e ? std::atoi(e) : 0; }();
  p.prefetch = ctx.pdl ? prefetch : 0;
  p.stages = (196 * 1024) / p.stage_bytes;
  if (p.stages > 6) p.stages = 6;
  const size_t smem = (size_t)p.stages * p.stage_bytes + 2 * (glu ? 3 : 2) * 2048 + 1024 + 512;
  cudaError_t e;
  if (glu) {
    if ((e = ensure_smem(moe_gemm_mx_kernel<true>, smem)) != cudaSuccess) return e;
    return launch_k(ctx.pdl, moe_gemm_mx_kernel<true>, dim3(ctx.num_sms), dim3(kMxThreads), smem, stream, tw, tx, twsf, txsf, p);
  }
  if ((e = ensure_smem(moe_gemm_mx_kernel<false>, smem)) != cudaSuccess) return e;
  return launch_k(ctx.pdl, moe_gemm_mx_kernel<false>, dim3(ctx.num_sms), dim3(kMxThreads), smem, stream, tw, tx, twsf, txsf, p);
}

}  // namespace afdk
