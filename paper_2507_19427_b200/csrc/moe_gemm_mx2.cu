// moe_gemm_mx2.cu — K7/K8 MXFP8 expert GEMMs on CTA pairs (tcgen05 cta_group::2).
//
// The large-batch form of moe_gemm_mx.cu.  At hundreds of dispatched rows per
// expert the single-CTA kernel (128 weight rows x 128 tokens per item) is
// bound by L2->SM traffic: each k-block moves 48 KB per 8.4 MFLOP.  A CTA pair
// (two SMs of one TPC, launched as a 2-CTA cluster) issues one M=256 MMA over
// both CTAs' shared memory: each CTA stages 128 weight rows and HALF of the
// token panel, the tensor core reads the other half from the peer, and each CTA
// accumulates its 128 rows x N tokens (N <= 256) in its own TMEM.  Per SM a
// k-block is now 32 KB per 8.4 MFLOP, and an expert with <= 256 rows fetches
// its weights once per item instead of once per 128-row chunk.
//
// Item = (dispatch chunk, pair m-tile).  Chunks are 256 rows, or 384 rows in
// the two-accumulator form (kTwo, chosen when routed experts average 200-352
// rows): one MMA covers at most N=256 tokens, so a chunk's first 256 rows
// accumulate in TMEM columns [0,256) and the rest (<= 128) in [384,512) from
// a second B panel; both MMAs of a k-step read the same weight panel, so an
// expert with 257-384 rows streams its weights once instead of twice.  kTwo
// costs one pipeline stage (40 KB stages), so it is not used elsewhere.
//   W13: the pair covers 128 intermediate features; CTA r stages gate rows
//        [f0+64r, +64) and the matching up rows as one 128-row A panel, so
//        TMEM lanes 0-63 hold gate and 64-127 hold up for the same features;
//        the epilogue parks both in smem, and each thread applies SiLU(gate)*up
//        to one (token, 32-feature block) and re-quantises it to MXFP8.
//   W2:  the pair covers 256 output features, 128 per CTA.
// Scale factors: SFA = the CTA's own 128 rows (4 TMEM columns), SFB = all
// tokens replicated in both CTAs (8 + 4 columns), written per stage by four stager
// warps per CTA from TMA-loaded smem groups (see moe_gemm_mx.cu for the TMEM
// scale layout).
//
// Synchronisation across the pair: the leader (rank 0) owns full[], sf_full[]
// and acc_empty[]; the peer's TMA signals the leader's full barrier
// (cp.async.bulk.tensor .cta_group::2), its stager and epilogue warps arrive
// remotely; the leader's tcgen05.commit multicasts empty[] / acc_full[] to
// both CTAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "afdk_internal.h"
#include "moe.cuh"
#include "sm100.cuh"

namespace afdk {
namespace moe {

using namespace sm100;

constexpr int kPairThreads = 448;  // w0 TMA, w1 MMA (leader) + TMEM, w2-5 + w10-13 epilogue, w6-9 scale stagers
constexpr uint32_t kPSfCol0 = 256;
constexpr uint32_t kPAcc1Col = 384;     // kTwo: second accumulator, chunk rows 256..383
// per form: SF columns per stage (SFA 4 + SFB 8 [+ SFB1 4]), stage bytes
// (A 16 KB + B 16 KB [+ B1 8 KB]), scale-group bytes, stages (W13 / W2; the
// W13 epilogue exchange takes 35 KB of smem)
template <bool kTwo> struct PairCfg {
  static constexpr int kSfCols = kTwo ? 16 : 12;
  static constexpr int kStage = kTwo ? 40960 : 32768;
  static constexpr int kSfGrp = kTwo ? 2048 + 4096 + 2048 : 2048 + 4096;
  static constexpr int kStagesW13 = kTwo ? 4 : 5;
  static constexpr int kStagesW2 = kTwo ? 5 : 6;
};
static_assert(kPSfCol0 + PairCfg<true>::kStagesW2 * PairCfg<true>::kSfCols <= kPAcc1Col,
              "TMEM scale ring overlaps the second accumulator");
static_assert(kChunkMX2Two <= 384, "two accumulators cover at most 384 rows");
constexpr int kXRow = 68;          // padded smem row (floats) of the W13 epilogue exchange

struct Mx2Params {
  const Work* work;
  const int* n_work;
  int m_tiles;    // items per chunk: W13 I/128, W2 H/256
  int kblocks;    // K / 128 (multiple of 4)
  int w_rows;     // weight rows per expert (W13 2I, W2 H)
  int up_offset;  // W13: I
  int E, expert_lo, n_local;
  int out_cols;   // W13 I, W2 H
  uint8_t* hq;
  uint8_t* hsf;
  float* y;
};

__device__ __forceinline__ int mx2_exp(float amax) {
  const uint32_t u = __float_as_uint(amax);
  const int E = (int)((u >> 23) & 0xff);
  if (!(amax > 0.0f) || E == 0) return -127;
  const int e = ((u & 0x7fffffu) <= 6291456u) ? E - 135 : E - 134;
  return max(-127, min(127, e));
}

// TMEM column of chunk row t (t % 32 == 0): rows 0-255 in the first
// accumulator, 256-383 in the second
__device__ __forceinline__ uint32_t acc_col(int t) { return t < 256 ? (uint32_t)t : kPAcc1Col + (uint32_t)(t - 256); }

__device__ __forceinline__ void pair_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <bool kGLU, bool kTwo>
__global__ void __launch_bounds__(kPairThreads, 1)
moe_gemm_mx2_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                    const __grid_constant__ CUtensorMap tm_x1, const __grid_constant__ CUtensorMap tm_wsf,
                    const __grid_constant__ CUtensorMap tm_xsf, const __grid_constant__ CUtensorMap tm_xsf1,
                    const Mx2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  using Cfg = PairCfg<kTwo>;
  constexpr int S = kGLU ? Cfg::kStagesW13 : Cfg::kStagesW2;
  constexpr int kPStage = Cfg::kStage, kPSfGrp = Cfg::kSfGrp, kPSfCols = Cfg::kSfCols;
  uint8_t* sfbuf = smem + S * kPStage;
  float* xchg = reinterpret_cast<float*>(sfbuf + 2 * kPSfGrp);  // W13: gate, up [64 tokens][kXRow]
  uint64_t* full = reinterpret_cast<uint64_t*>(xchg + (kGLU ? 2 * 64 * kXRow : 0));
  uint64_t* sf_full = full + S;
  uint64_t* empty = sf_full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* sfg_full = acc_empty + 1;
  uint64_t* sfg_empty = sfg_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfg_empty + 2);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_x1);
    tma_prefetch_desc(&tm_wsf);
    tma_prefetch_desc(&tm_xsf);
    tma_prefetch_desc(&tm_xsf1);
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&sf_full[i], 8); mbar_init(&empty[i], 1); }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 16);
    for (int i = 0; i < 2; ++i) { mbar_init(&sfg_full[i], 1); mbar_init(&sfg_empty[i], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  griddep_wait();
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_work = *p.n_work;
  const int n_items = n_work * p.m_tiles;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal();
      const uint32_t full_l = mapa_shared(full, 0);
      int i = 0, gi = 0;
      for (int it = pair; it < n_items; it += n_pairs) {
        const ItemRef ir = item_of(p.work, it, p.m_tiles);
        const int mt = ir.mt;
        const Work wk = p.work[ir.chunk];
        const int n0 = min((wk.rows + 31) & ~31, 256), n1 = kTwo ? max(((wk.rows + 31) & ~31) - 256, 0) : 0;
        const int half = n0 >> 1, half1 = n1 >> 1;
        const int widx = (wk.group == p.E ? p.n_local : wk.group - p.expert_lo) * p.w_rows;
        const int arow = kGLU ? widx + mt * 128 + 64 * (int)rank : widx + mt * 256 + 128 * (int)rank;
        const int in_row0 = kGLU ? wk.xrow0 : wk.row0;  // W13 reads the token rows, W2 the intermediate
        const int brow = in_row0 + (int)rank * half;
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          if ((kb & 3) == 0) {
            const int g = gi & 1, ng = gi >> 1;
            ++gi;
            if (ng > 0) mbar_wait(&sfg_empty[g], (ng & 1) ^ 1);
            uint8_t* dst = sfbuf + g * kPSfGrp;
            mbar_expect_tx(&sfg_full[g], 2048 + 4096 + (n1 ? 2048 : 0));  // SFA + SFB [+ SFB1]
            tma_load_2d(dst, &tm_wsf, &sfg_full[g], kb * 4, arow, pol);
            if (kGLU) tma_load_2d(dst + 1024, &tm_wsf, &sfg_full[g], kb * 4, arow + p.up_offset, pol);
            tma_load_2d(dst + 2048, &tm_xsf, &sfg_full[g], kb * 4, in_row0, pol);
            if (n1) tma_load_2d(dst + 6144, &tm_xsf1, &sfg_full[g], kb * 4, in_row0 + 256, pol);
          }
          const int s = i % S, n = i / S;
          if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
          uint8_t* st = smem + s * kPStage;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * (32768 + (n1 ? 8192 : 0)));  // A + B [+ B1], both CTAs
          const uint32_t fb = full_l + 8u * s;
          tma_load_2d_pair(st, &tm_w, fb, kb * 128, arow, pol);
          if (kGLU) tma_load_2d_pair(st + 8192, &tm_w, fb, kb * 128, arow + p.up_offset, pol);
          tma_load_2d_pair(st + 16384, &tm_x, fb, kb * 128, brow, pol);
          if (n1) tma_load_2d_pair(st + 32768, &tm_x1, fb, kb * 128, in_row0 + 256 + (int)rank * half1, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int i = 0, li = 0;
#ifdef AFDK_MX2_PROF
      long long t_acc = 0, t_full = 0, t_sf = 0, t0 = clock64(), tq;
#define MX2_T(x) (tq = clock64(), x += tq - t0, t0 = tq)
#else
#define MX2_T(x)
#endif
      for (int it = pair; it < n_items; it += n_pairs, ++li) {
        const Work wk = p.work[item_of(p.work, it, p.m_tiles).chunk];
        const uint32_t npad = (uint32_t)((wk.rows + 31) & ~31);
        const uint32_t n0 = npad < 256u ? npad : 256u, n1 = (kTwo && npad > 256u) ? npad - 256u : 0u;
        const uint32_t idesc = idesc_mxf8(256, n0), idesc1 = idesc_mxf8(256, n1 ? n1 : 32u);
#ifdef AFDK_MX2_PROF
        t0 = clock64();
#endif
        if (li > 0) mbar_wait(acc_empty, (li & 1) ^ 1);
        MX2_T(t_acc);
        tc_fence_after();
        for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
          const int s = i % S, n = i / S;
#ifdef AFDK_MX2_PROF
          t0 = clock64();
#endif
          mbar_wait(&full[s], n & 1);
          MX2_T(t_full);
          mbar_wait(&sf_full[s], n & 1);
          MX2_T(t_sf);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * kPStage);
          const uint32_t sf = tmem + kPSfCol0 + (uint32_t)(s * kPSfCols);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = sdesc_sw128(base + kk * 32, 0, 1024);
            const uint64_t db = sdesc_sw128(base + 16384 + kk * 32, 0, 1024);
            const uint32_t sel = (uint32_t)kk << 30;
            mma_mxf8_pair(tmem, da, db, idesc | idesc_sf_ids(kk, kk), sf | sel, (sf + 4) | sel,
                          (kb > 0 || kk > 0) ? 1u : 0u);
            if (n1) {
              const uint64_t db1 = sdesc_sw128(base + 32768 + kk * 32, 0, 1024);
              mma_mxf8_pair(tmem + kPAcc1Col, da, db1, idesc1 | idesc_sf_ids(kk, kk), sf | sel, (sf + 12) | sel,
                            (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit_pair(&empty[s], 0x3);
          if (kb == p.kblocks - 1) mma_commit_pair(acc_full, 0x3);
        }
      }
#ifdef AFDK_MX2_PROF
      if (pair % 16 == 0)
        printf("mx2 glu=%d pair %d items %d wait_acc %lld wait_full %lld wait_sf %lld (cycles)\n", (int)kGLU, pair, li,
               t_acc, t_full, t_sf);
#endif
    }
  } else if (warp >= 6 && warp <= 9) {
    // ------------------------------------------------------ scale stagers
    const int sp = warp & 3;
    const uint32_t t_lane = tmem + ((uint32_t)(sp * 32) << 16);
    const uint32_t sf_full_l = mapa_shared(sf_full, 0);
    int i = 0, gi = 0;
    for (int it = pair; it < n_items; it += n_pairs) {
      for (int kb = 0; kb < p.kblocks; ++kb, ++i) {
        const int g = gi & 1;
        if ((kb & 3) == 0) mbar_wait(&sfg_full[g], (gi >> 1) & 1);
        const int s = i % S, n = i / S;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        const uint32_t* ga = reinterpret_cast<const uint32_t*>(sfbuf + g * kPSfGrp) + (kb & 3) + lane * 4;
        const uint32_t* gb = ga + 512;
        const uint32_t col = t_lane + kPSfCol0 + (uint32_t)(s * kPSfCols);
        tmem_st4(col, ga[0], ga[128], ga[256], ga[384]);
        tmem_st4(col + 4, gb[0], gb[128], gb[256], gb[384]);
        tmem_st4(col + 8, gb[512], gb[640], gb[768], gb[896]);
        if (kTwo) tmem_st4(col + 12, gb[1024], gb[1152], gb[1280], gb[1408]);  // rows 256-383 (stale when unused)
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_remote(sf_full_l + 8u * s);
          if ((kb & 3) == 3) mbar_arrive(&sfg_empty[g]);
        }
        if ((kb & 3) == 3) ++gi;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // 8 warps: two per TMEM subpartition (warps 2-5 and 10-13), splitting the
    // item's 32-token chunks between them
    const int sub = warp & 3, ehalf = warp >= 10 ? 1 : 0;
    const int etid = ehalf * 128 + (warp - (ehalf ? 10 : 2)) * 32 + lane;  // 0..255
    const uint32_t t_lane = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t acc_empty_l = mapa_shared(acc_empty, 0);
    int li = 0;
    for (int it = pair; it < n_items; it += n_pairs, ++li) {
      const ItemRef ir = item_of(p.work, it, p.m_tiles);
      const int mt = ir.mt;
      const Work wk = p.work[ir.chunk];
      const int n_chunks = (wk.rows + 31) >> 5;
      mbar_wait(acc_full, li & 1);
      tc_fence_after();
      if (kGLU) {
        // 64-token groups: each warp parks one 32-token chunk of its TMEM rows
        // (gate: subpartitions 0,1; up: 2,3) in smem [token][kXRow]; then two
        // threads per (token, 32-feature MX block) apply SiLU(gate)*up to 16
        // features each and re-quantise the block to MXFP8.
        float* xg = xchg;
        float* xu = xchg + 64 * kXRow;
        for (int g0 = 0; g0 < n_chunks * 32; g0 += 64) {
          if (g0 + ehalf * 32 < n_chunks * 32) {
            uint32_t v[32];
            tmem_ld32(t_lane + acc_col(g0 + ehalf * 32), v);
            tmem_wait_ld();
            float* dst = (sub < 2 ? xg : xu) + (ehalf * 32) * kXRow + (sub & 1) * 32 + lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) dst[j * kXRow] = __uint_as_float(v[j]);
          }
          pair_bar(1, 256);
          const int unit = etid >> 1, hf = etid & 1;
          const int tt = unit & 63, blk = unit >> 6;
          const float4* gp = reinterpret_cast<const float4*>(xg + tt * kXRow + blk * 32 + hf * 16);
          const float4* up = reinterpret_cast<const float4*>(xu + tt * kXRow + blk * 32 + hf * 16);
          float h[16];
          float amax = 0.0f;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 a = gp[q], b = up[q];
            const float ga[4] = {a.x, a.y, a.z, a.w}, ub[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              h[q * 4 + z] = silu_fast(ga[z]) * ub[z];
              amax = fmaxf(amax, fabsf(h[q * 4 + z]));
            }
          }
          amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 1));
          const int e = mx2_exp(amax);
          const float inv = e < 127 ? __uint_as_float((uint32_t)(127 - e) << 23) : __uint_as_float(1u << 22);
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t x = 0;
#pragma unroll
            for (int z = 0; z < 4; ++z)
              x |= (uint32_t)__nv_cvt_float_to_fp8(h[q * 4 + z] * inv, __NV_SATFINITE, __NV_E4M3) << (8 * z);
            w[q] = x;
          }
          const int r = g0 + tt;
          if (r < wk.rows) {
            const size_t row = (size_t)wk.row0 + r;
            const int f0 = mt * 128 + 64 * (int)rank + 32 * blk;
            *reinterpret_cast<uint4*>(p.hq + row * p.out_cols + f0 + hf * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            if (hf == 0) p.hsf[row * (p.out_cols / 32) + f0 / 32] = (uint8_t)(e + 127);
          }
          pair_bar(1, 256);
        }
      } else {
        for (int c = ehalf; c < n_chunks; c += 2) {
          uint32_t v[32];
          tmem_ld32(t_lane + acc_col(c * 32), v);
          tmem_wait_ld();
          const int feat = mt * 256 + 128 * (int)rank + sub * 32 + lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int r = c * 32 + j;
            if (r < wk.rows) p.y[((size_t)wk.row0 + r) * p.out_cols + feat] = __uint_as_float(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc_empty_l);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem);
  }
}

}  // namespace moe

cudaError_t moe_gemm_mx2_launch(Ctx& ctx, bool glu, const MoeGemmMxArgs& a, cudaStream_t stream) {
  using namespace moe;
  const int K = glu ? a.H : a.I;
  const int w_rows = glu ? 2 * a.I : a.H;
  const uint64_t wr = (uint64_t)(a.n_local + 1) * w_rows;
  CUtensorMap tw, tx, tx1, twsf, txsf, txsf1;
  auto enc = [&](CUtensorMap* m, const void* base, uint64_t inner, uint64_t rows, uint32_t bi, uint32_t br,
                 CUtensorMapSwizzle sw) {
    const uint64_t dims[2] = {inner, rows};
    const uint64_t strides[1] = {inner};
    const uint32_t box[2] = {bi, br};
    return encode_tma(ctx, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, sw);
  };
  if (!enc(&tw, a.w, K, wr, 128, glu ? 64 : 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !enc(&tx, a.x, K, a.rows_pad, 128, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !enc(&tx1, a.x, K, a.rows_pad, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !enc(&twsf, a.w_sf, K / 32, wr, 16, glu ? 64 : 128, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !enc(&txsf, a.x_sf, K / 32, a.rows_pad, 16, 256, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !enc(&txsf1, a.x_sf, K / 32, a.rows_pad, 16, 128, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  Mx2Params p{};
  p.work = a.work;
  p.n_work = a.n_work;
  p.m_tiles = glu ? a.I / 128 : a.H / 256;
  p.kblocks = K / 128;
  p.w_rows = w_rows;
  p.up_offset = glu ? a.I : 0;
  p.E = a.E;
  p.expert_lo = a.expert_lo;
  p.n_local = a.n_local;
  p.out_cols = glu ? a.I : a.H;
  p.hq = a.hq;
  p.hsf = a.hsf;
  p.y = a.y;
  const int grid = (ctx.num_sms / 2) * 2;
  auto go = [&](auto kernel, auto cfg) {
    using Cfg = decltype(cfg);
    const size_t smem = (size_t)(glu ? Cfg::kStagesW13 : Cfg::kStagesW2) * Cfg::kStage + 2 * Cfg::kSfGrp +
                        (glu ? 2 * 64 * kXRow * 4 : 0) + 1024 + 512;
    if (const cudaError_t e = ensure_smem(kernel, smem); e != cudaSuccess) return e;
    return launch_cluster_k(ctx.pdl, 2, kernel, dim3(grid), dim3(kPairThreads), smem, stream, tw, tx, tx1, twsf, txsf,
                            txsf1, p);
  };
  const bool two = a.chunk > kChunkMX2;
  if (glu) return two ? go(moe_gemm_mx2_kernel<true, true>, PairCfg<true>{})
                      : go(moe_gemm_mx2_kernel<true, false>, PairCfg<false>{});
  return two ? go(moe_gemm_mx2_kernel<false, true>, PairCfg<true>{})
             : go(moe_gemm_mx2_kernel<false, false>, PairCfg<false>{});
}

}  // namespace afdk
