// moe_gemm.cu — K7/K8: grouped FP8 expert GEMMs with 128x128 weight scales and
// 1x128 activation scales on sm_100a tensor cores.
//
// Each gated expert (builtin_catalog.cpp:248-251: 3*h*inter params, Step-3
// h=7168, inter=5120) is two GEMMs over its dispatched rows:
//   W13: [gate|up] = x . W13^T   (2I x H)   epilogue SiLU(gate)*up, re-quantised
//                                          to e4m3 with 1x128 scales
//   W2:  y = h . W2^T            (H x I)    epilogue fp32 rows
// The shared expert is group E, run over every token.  Decode batches give
// each expert only ~T*k/E rows, so the kernel is swap-AB like linear.cu: a
// 128-row weight tile is the MMA M side and up to 64 dispatched rows are N:
//
//   D[128 x N] = Wq[128 x 128k] . Xq[N x 128k]^T   tcgen05.mma kind::f8f6f4
//
// one TMEM accumulator slot per 128-wide k-block; the 4 epilogue warps promote
// it into fp32 registers with sw[tile,kb] * sx[row,kb] (DeepSeek-style block
// scaling in software, exact fp8 products, fp32 sums) while the tensor core
// fills the next slot.  Work items = (group chunk, m-tile); consecutive CTAs
// take chunks of the same group for one m-tile so a weight tile re-read by
// several chunks hits L2.
//
// Roles (224 threads): w0 TMA producer, w1 MMA issuer + TMEM owner, w2-5 epilogue,
// w6 activation-scale stager.
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

constexpr int kThreads = 224;  // w0 TMA, w1 MMA, w2-5 epilogue, w6 scale stager
constexpr int kAccSlots = 4;  // TMEM ring: 4 x 128 columns

struct GemmParams {
  const Work* work;
  const int* n_work;
  int m_tiles;       // output features / 128 (GLU: per half)
  int kblocks;       // K / 128
  int w_rows;        // weight rows per expert in the 2D weight map (GLU 2I, W2 H)
  int up_offset;     // GLU: row offset of the up half (= I)
  const float* w_scale;  // [(n_local+1)][w_rows/128][kblocks]
  int E, expert_lo, n_local;
  int rows_pad;
  int out_cols;      // GLU: I (hq row stride), W2: H (y row stride)
  uint8_t* hq;       // GLU out: [rows_pad, I] e4m3
  float* hs_t;       // GLU out: [I/128, rows_pad]
  float* y;          // W2 out:  [rows_pad, H] fp32
  const float* xs_t;  // [K/128][rows_pad] activation row scales
  int stage_bytes, stages;
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ int weight_index(const GemmParams& p, int group) {
  return group == p.E ? p.n_local : group - p.expert_lo;
}

template <bool kGLU>
__global__ void __launch_bounds__(kThreads, 1)
moe_gemm_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                const GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kA = 128 * 128;                 // 16 KB weight panel
  constexpr int kAOps = kGLU ? 2 : 1;
  constexpr int kB = kChunk * 128;              // 8 KB activation panel
  const int S = p.stages;
  // per stage: the chunk's kChunk activation row scales + the weight tile's
  // gate/up block scales of this k-block (staged by warp 6, read by the epilogue)
  constexpr int kRing = kChunk + 4;
  float* xs_ring = reinterpret_cast<float*>(smem + S * p.stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(xs_ring + S * kRing);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + kAccSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAccSlots);
  __shared__ float s_red[4][kChunk];

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1 + 32); mbar_init(&empty[i], 1 + 4); }  // TMA + stager lanes; MMA + epilogue warps
    for (int i = 0; i < kAccSlots; ++i) { mbar_init(&acc_full[i], 1); mbar_init(&acc_empty[i], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();  // work list, dispatch rows and scales come from the predecessors
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_work = *p.n_work;
  const int n_items = n_work * p.m_tiles;

  if (warp == 0) {
    // TMA producer: weight panel(s) + activation panel of every k-block
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int i = 0;
      for (int it = cta; it < n_items; it += G) {
        const int mt = it / n_work, gc = it % n_work;
        const Work wk = p.work[gc];
        const int wrow = weight_index(p, wk.group) * p.w_rows + mt * 128;
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
          if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
          uint8_t* st = smem + s * p.stage_bytes;
          mbar_expect_tx(&full[s], kAOps * kA + kB);
          tma_load_2d(st, &tm_w, &full[s], kb * 128, wrow, pol_w);
          if (kGLU) tma_load_2d(st + kA, &tm_w, &full[s], kb * 128, wrow + p.up_offset, pol_w);
          tma_load_2d(st + kAOps * kA, &tm_x, &full[s], kb * 128, kGLU ? wk.xrow0 : wk.row0, pol_x);
        }
      }
    }
  } else if (warp == 6) {
    // row-scale stager: the chunk's activation scales of each k-block (plain
    // loads: dispatch rows start at arbitrary offsets), off the TMA issue path
    int i = 0;
    const int nb_rows = p.w_rows / 128;
    for (int it = cta; it < n_items; it += G) {
      const int mt = it / n_work;
      const Work wk = p.work[it % n_work];
      const float* sw = p.w_scale + (size_t)weight_index(p, wk.group) * nb_rows * p.kblocks;
      for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
        const int s = i % S, n = i / S;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        const float* src = p.xs_t + (size_t)kb * p.rows_pad + (kGLU ? wk.xrow0 : wk.row0);
        float* dst = xs_ring + s * kRing;
        dst[lane] = (lane < wk.rows) ? __ldg(src + lane) : 0.0f;
        dst[lane + 32] = (lane + 32 < wk.rows) ? __ldg(src + lane + 32) : 0.0f;
        if (lane == 0) dst[kChunk] = __ldg(sw + (size_t)mt * p.kblocks + kb);
        if (lane == 1 && kGLU) dst[kChunk + 1] = __ldg(sw + (size_t)(mt + p.up_offset / 128) * p.kblocks + kb);
        mbar_arrive(&full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int i = 0;
      for (int it = cta; it < n_items; it += G) {
        const Work wk = p.work[it % n_work];
        const uint32_t n_mma = (uint32_t)((wk.rows + 15) & ~15);
        const uint32_t idesc = idesc_e4m3(128, n_mma);
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
          const int a = i % kAccSlots, na = i / kAccSlots;
          mbar_wait(&full[s], n & 1);
          if (na > 0) mbar_wait(&acc_empty[a], (na & 1) ^ 1);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * p.stage_bytes);
          const uint32_t b_base = base + kAOps * kA;
#pragma unroll
          for (int op = 0; op < kAOps; ++op) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = sdesc_sw128(base + op * kA + kk * 32, 0, 1024);
              const uint64_t db = sdesc_sw128(b_base + kk * 32, 0, 1024);
              mma_e4m3(tmem + a * 128 + op * 64, da, db, idesc, kk > 0 ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          mma_commit(&acc_full[a]);
        }
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ----------------------------------------------------------- epilogue
    const int sub = warp & 3, et = sub * 32 + lane;  // et = feature row in the tile
    const uint32_t t_lane = tmem + ((uint32_t)(sub * 32) << 16);
    int i = 0;
    for (int it = cta; it < n_items; it += G) {
      const int mt = it / n_work;
      const Work wk = p.work[it % n_work];
      float accg[kChunk], accu[kGLU ? kChunk : 1];
#pragma unroll
      for (int n = 0; n < kChunk; ++n) accg[n] = 0.0f;
      if (kGLU) {
#pragma unroll
        for (int n = 0; n < kChunk; ++n) accu[kGLU ? n : 0] = 0.0f;
      }
      const int n_ld = (wk.rows + 31) >> 5;  // 32-column TMEM loads needed
      for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
        const int a = i % kAccSlots, na = i / kAccSlots;
        const int s = i % S;
        mbar_wait(&acc_full[a], na & 1);
        mbar_wait(&full[s], (i / S) & 1);  // row scales staged (complete; stage held until we arrive)
        tc_fence_after();
        const float* xs = xs_ring + s * kRing;
        const float swg = xs[kChunk];
        const float swu = kGLU ? xs[kChunk + 1] : 0.0f;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < n_ld) {
            uint32_t v[32];
            tmem_ld32(t_lane + a * 128 + c * 32, v);
            uint32_t u[32];
            if (kGLU) tmem_ld32(t_lane + a * 128 + 64 + c * 32, u);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float sx = xs[c * 32 + j];
              accg[c * 32 + j] = fmaf(__uint_as_float(v[j]), swg * sx, accg[c * 32 + j]);
              if (kGLU) accu[kGLU ? c * 32 + j : 0] = fmaf(__uint_as_float(u[j]), swu * sx, accu[kGLU ? c * 32 + j : 0]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&acc_empty[a]);
          mbar_arrive(&empty[s]);
        }
      }
      if (kGLU) {
        // h = SiLU(gate) * up; per dispatched row, quantise the tile's 128
        // features (one 1x128 block) to e4m3.  Work in groups of 16 rows and
        // skip the groups beyond this chunk's rows (warp-uniform).
        float h[kChunk];
#pragma unroll
        for (int g16 = 0; g16 < kChunk / 16; ++g16) {
          if (g16 * 16 < wk.rows) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = g16 * 16 + j;
              const float g = accg[n];
              h[n] = sm100::silu_fast(g) * accu[kGLU ? n : 0];
              float m = fabsf(h[n]);
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
              if (lane == 0) s_red[sub][n] = m;
            }
          }
        }
        named_bar(1, 128);
#pragma unroll
        for (int g16 = 0; g16 < kChunk / 16; ++g16) {
          if (g16 * 16 < wk.rows) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int n = g16 * 16 + j;
              if (n < wk.rows) {
                const float amax = fmaxf(fmaxf(s_red[0][n], s_red[1][n]), fmaxf(s_red[2][n], s_red[3][n]));
                const float sc = __fdiv_rn(fmaxf(amax, 1e-10f), 448.0f);
                const size_t row = (size_t)wk.row0 + n;
                p.hq[row * p.out_cols + mt * 128 + et] =
                    (uint8_t)__nv_cvt_float_to_fp8(__fdiv_rn(h[n], sc), __NV_SATFINITE, __NV_E4M3);
                if (et == 0) p.hs_t[(size_t)mt * p.rows_pad + row] = sc;
              }
            }
          }
        }
        named_bar(1, 128);
      } else {
#pragma unroll
        for (int n = 0; n < kChunk; ++n)
          if (n < wk.rows) p.y[((size_t)wk.row0 + n) * p.out_cols + mt * 128 + et] = accg[n];
      }
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

// W13 (kGLU) or W2 over the work list built by permute_launch.
cudaError_t moe_gemm_launch(Ctx& ctx, bool glu, const MoeGemmArgs& a, cudaStream_t stream) {
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
    const uint32_t box[2] = {128, kChunk};
    if (!encode_tma(ctx, &tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(a.x), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  GemmParams p{};
  p.work = a.work;
  p.n_work = a.n_work;
  p.m_tiles = glu ? a.I / 128 : a.H / 128;
  p.kblocks = K / 128;
  p.w_rows = w_rows;
  p.up_offset = glu ? a.I : 0;
  p.w_scale = a.w_scale;
  p.E = a.E;
  p.expert_lo = a.expert_lo;
  p.n_local = a.n_local;
  p.rows_pad = a.rows_pad;
  p.out_cols = glu ? a.I : a.H;
  p.hq = a.hq;
  p.hs_t = a.hs_t;
  p.y = a.y;
  p.xs_t = a.xs_t;
  const int a_bytes = (glu ? 2 : 1) * 128 * 128;
  p.stage_bytes = (int)align_up((size_t)a_bytes + kChunk * 128, 1024);
  p.stages = (200 * 1024) / p.stage_bytes;
  if (p.stages > 8) p.stages = 8;
  const size_t smem = (size_t)p.stages * (p.stage_bytes + (kChunk + 4) * 4) + 1024 + 512;
  cudaError_t e;
  if (glu) {
    if ((e = ensure_smem(moe_gemm_kernel<true>, smem)) != cudaSuccess) return e;
    return launch_k(ctx.pdl, moe_gemm_kernel<true>, dim3(ctx.num_sms), dim3(kThreads), smem, stream, tw, tx, p);
  } else {
    if ((e = ensure_smem(moe_gemm_kernel<false>, smem)) != cudaSuccess) return e;
    return launch_k(ctx.pdl, moe_gemm_kernel<false>, dim3(ctx.num_sms), dim3(kThreads), smem, stream, tw, tx, p);
  }
  return cudaGetLastError();
}

}  // namespace afdk
