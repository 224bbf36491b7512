// moe_ffn_mx_fused.cu — K7 + K8 of the MXFP8 MoE FFN at decode batches in ONE
// persistent launch with a dynamic item queue.
//
// At decode (a few dozen rows per routed expert, the AFD FFN GPUs of
// PAPER.md:651) the MoE layer is a stream of expert weights: 3*H*I bytes per
// expert (builtin_catalog.cpp:248-251).  Run as two launches (gate|up GEMM,
// then down GEMM) each grid pays a partial last wave: a shard of 16 experts +
// the shared one has 17*40 gate|up items for 148 CTAs (4.59 waves: CTAs run 4
// or 5 items, so the launch lasts 5) and 17*56 down items (6.43 waves), and
// the down GEMM cannot start before every gate|up item has finished.  Here
// both GEMMs share one queue: items are dequeued in order (all gate|up items,
// chunk-major, then all down items) by the CTA whose producer frees up first,
// so the only partial wave is the final one, of the smaller down items.  A
// down item of chunk c needs the whole SiLU(gate)*up intermediate of chunk c:
// the gate|up epilogue publishes each finished item (release add on a
// per-chunk counter), and the producer of a down item waits for the count
// (acquire) before its TMA reads the intermediate.  Items are dequeued only
// after all earlier ones, every one of which completes without waiting, so the
// waits cannot deadlock; in practice they never wait (the down items of a
// chunk come ~1 wave after its gate|up items).
//
// Per item the kernel is moe_gemm_mx.cu's single-CTA block-scaled GEMM (swap
// AB: 128 weight rows = MMA M, the chunk's rows = N; UE8M0 scales staged into
// TMEM).  The accumulator is a two-slot ring of 128 TMEM columns: a down item
// takes one slot, a gate|up item two (gate, up), so a down item's MMAs overlap
// the previous item's epilogue.  Roles (320 threads): w0 queue + TMA producer,
// w1 MMA issuer + TMEM owner, w2-5 epilogue, w6-9 scale stagers; a 4-deep smem
// ring hands each dequeued item index to the consumers.
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

namespace fused {
constexpr int kThreads = 320;
constexpr int kStages = 4;
constexpr int kA = 128 * 128;            // one 128-row weight k-block (e4m3)
constexpr int kB = kChunkMX * 128;       // one token-panel k-block
constexpr int kStage = 2 * kA + kB;      // gate | up | panel (down items use one A)
constexpr int kSfOp = 128 * 16;          // one operand's scales for 4 k-blocks
constexpr int kSfGrp = 3 * kSfOp;        // gate | up | panel scales
constexpr int kSfCols = 12;              // TMEM scale columns per stage
constexpr uint32_t kSfCol0 = 256;
constexpr int kRing = 4;                 // dequeued items in flight per CTA
constexpr int kRingConsumers = 1 + 4 + 4;  // MMA lane + epilogue warps + stager warps
}  // namespace fused

struct FusedMxParams {
  const Work* work;
  const int* n_work;
  int mt13, mt2;      // output tiles per chunk: I/128 (gate|up), H/128 (down)
  int kb13, kb2;      // k-blocks: H/128, I/128
  int I, H;
  int E, expert_lo, n_local;
  uint8_t* hq;        // [rows_pad, I] e4m3 intermediate
  uint8_t* hsf;       // [rows_pad, I/32] UE8M0
  float* y;           // [rows_pad, H] expert outputs
  int* sched;         // [0] queue head, [1 + chunk] finished gate|up items (zeroed by the permute kernel)
};

__device__ __forceinline__ int fmx_exp(float amax) {
  const uint32_t u = __float_as_uint(amax);
  const int E = (int)((u >> 23) & 0xff);
  if (!(amax > 0.0f) || E == 0) return -127;
  const int e = ((u & 0x7fffffu) <= 6291456u) ? E - 135 : E - 134;
  return max(-127, min(127, e));
}

__device__ __forceinline__ void red_release_gpu_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct FItem {
  bool glu;
  int mt, chunk;
};
__device__ __forceinline__ FItem fitem(const FusedMxParams& p, int n13, int it) {
  if (it < n13) {
    const ItemRef r = item_of(p.work, it, p.mt13);
    return {true, r.mt, r.chunk};
  }
  const ItemRef r = item_of(p.work, it - n13, p.mt2);
  return {false, r.mt, r.chunk};
}

__global__ void __launch_bounds__(fused::kThreads, 1)
moe_ffn_mx_fused_kernel(const __grid_constant__ CUtensorMap tm_w13, const __grid_constant__ CUtensorMap tm_x,
                        const __grid_constant__ CUtensorMap tm_w13sf, const __grid_constant__ CUtensorMap tm_xsf,
                        const __grid_constant__ CUtensorMap tm_w2, const __grid_constant__ CUtensorMap tm_h,
                        const __grid_constant__ CUtensorMap tm_w2sf, const __grid_constant__ CUtensorMap tm_hsf,
                        const FusedMxParams p) {
  using namespace fused;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sfbuf = smem + kStages * kStage;  // 2 scale groups
  uint64_t* full = reinterpret_cast<uint64_t*>(sfbuf + 2 * kSfGrp);
  uint64_t* sf_full = full + kStages;
  uint64_t* empty = sf_full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* sfg_full = acc_empty + 2;
  uint64_t* sfg_empty = sfg_full + 2;
  uint64_t* item_full = sfg_empty + 2;
  uint64_t* item_empty = item_full + kRing;
  int* s_item = reinterpret_cast<int*>(item_empty + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_item + kRing);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_w13);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w13sf);
    tma_prefetch_desc(&tm_xsf);
    tma_prefetch_desc(&tm_w2);
    tma_prefetch_desc(&tm_h);
    tma_prefetch_desc(&tm_w2sf);
    tma_prefetch_desc(&tm_hsf);
    for (int i = 0; i < kStages; ++i) { mbar_init(&full[i], 1); mbar_init(&sf_full[i], 4); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
      mbar_init(&sfg_full[i], 1);
      mbar_init(&sfg_empty[i], 4);
    }
    for (int i = 0; i < kRing; ++i) { mbar_init(&item_full[i], 1); mbar_init(&item_empty[i], kRingConsumers); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  griddep_wait();
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_work = *p.n_work;
  const int n13 = n_work * p.mt13;
  const int n_items = n13 + n_work * p.mt2;

  // every consumer: next dequeued item index (-1 = queue drained)
  // (warp_wide: all 32 lanes read the slot before lane 0 releases it)
  auto next_item = [&](int li, bool warp_wide) -> int {
    const int rs = li % kRing;
    mbar_wait(&item_full[rs], (li / kRing) & 1);
    const int it = s_item[rs];
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane == 0) mbar_arrive(&item_empty[rs]);
    return it;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------ queue + TMA producer
      const uint64_t pol = policy_evict_first();   // weights stream through L2 once
      const uint64_t pol_x = policy_evict_last();  // panels / intermediate are re-read
      int i = 0, gi = 0;
      for (int li = 0;; ++li) {
        int it = atomicAdd(p.sched, 1);
        if (it >= n_items) it = -1;
        const int rs = li % kRing, rn = li / kRing;
        if (rn > 0) mbar_wait(&item_empty[rs], (rn & 1) ^ 1);
        s_item[rs] = it;
        mbar_arrive(&item_full[rs]);
        if (it < 0) break;
        const FItem f = fitem(p, n13, it);
        const Work wk = p.work[f.chunk];
        const int widx = wk.group == p.E ? p.n_local : wk.group - p.expert_lo;
        const CUtensorMap* tw = f.glu ? &tm_w13 : &tm_w2;
        const CUtensorMap* tx = f.glu ? &tm_x : &tm_h;
        const CUtensorMap* twsf = f.glu ? &tm_w13sf : &tm_w2sf;
        const CUtensorMap* txsf = f.glu ? &tm_xsf : &tm_hsf;
        const int wrow = widx * (f.glu ? 2 * p.I : p.H) + f.mt * 128;
        const int xrow = f.glu ? wk.xrow0 : wk.row0;
        const int kblocks = f.glu ? p.kb13 : p.kb2;
        const int nA = f.glu ? 2 : 1;
        if (!f.glu) {  // the chunk's whole intermediate must be written
          unsigned ns = 64;
          long long spins = 0;
          while (ld_acquire_gpu(p.sched + 1 + f.chunk) < p.mt13) {
            __nanosleep(ns);
            if (ns < 512) ns <<= 1;
            if (++spins > (1ll << 24)) __trap();  // seconds: a lost publish fails the launch instead of hanging
          }
          fence_proxy_async_global();  // generic-proxy writes -> this thread's TMA reads
        }
        for (int kb = 0; kb < kblocks; ++kb, ++i) {
          if ((kb & 3) == 0) {
            const int g = gi & 1, ng = gi >> 1;
            ++gi;
            if (ng > 0) mbar_wait(&sfg_empty[g], (ng & 1) ^ 1);
            uint8_t* dst = sfbuf + g * kSfGrp;
            mbar_expect_tx(&sfg_full[g], (nA + 1) * kSfOp);
            tma_load_2d(dst, twsf, &sfg_full[g], kb * 4, wrow, pol);
            if (f.glu) tma_load_2d(dst + kSfOp, twsf, &sfg_full[g], kb * 4, wrow + p.I, pol);
            tma_load_2d(dst + 2 * kSfOp, txsf, &sfg_full[g], kb * 4, xrow, pol_x);
          }
          const int s = i % kStages, n = i / kStages;
          if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
          uint8_t* st = smem + s * kStage;
          mbar_expect_tx(&full[s], nA * kA + kB);
          tma_load_2d(st, tw, &full[s], kb * 128, wrow, pol);
          if (f.glu) tma_load_2d(st + kA, tw, &full[s], kb * 128, wrow + p.I, pol);
          tma_load_2d(st + 2 * kA, tx, &full[s], kb * 128, xrow, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------- MMA issuer
      int i = 0, r = 0;
      int nu[2] = {0, 0};
      for (int li = 0;; ++li) {
        const int it = next_item(li, false);
        if (it < 0) break;
        const FItem f = fitem(p, n13, it);
        const Work wk = p.work[f.chunk];
        const int nA = f.glu ? 2 : 1;
        int slot[2];
        for (int op = 0; op < nA; ++op) {
          const int sl = (r + op) & 1;
          slot[op] = sl;
          if (nu[sl] > 0) mbar_wait(&acc_empty[sl], (nu[sl] & 1) ^ 1);
          ++nu[sl];
        }
        r += nA;
        const uint32_t idesc = idesc_mxf8(128, (uint32_t)((wk.rows + 15) & ~15));
        const int kblocks = f.glu ? p.kb13 : p.kb2;
        for (int kb = 0; kb < kblocks; ++kb, ++i) {
          const int s = i % kStages, n = i / kStages;
          mbar_wait(&full[s], n & 1);
          mbar_wait(&sf_full[s], n & 1);
          tc_fence_after();
          const uint32_t base = smem_u32(smem + s * kStage);
          const uint32_t b_base = base + 2 * kA;
          const uint32_t sf = tmem + kSfCol0 + (uint32_t)(s * kSfCols);
          for (int op = 0; op < nA; ++op) {
            const uint32_t d = tmem + slot[op] * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t da = sdesc_sw128(base + op * kA + kk * 32, 0, 1024);
              const uint64_t db = sdesc_sw128(b_base + kk * 32, 0, 1024);
              const uint32_t sel = (uint32_t)kk << 30;
              mma_mxf8(d, da, db, idesc | idesc_sf_ids(kk, kk), (sf + op * 4) | sel, (sf + 8) | sel,
                       (kb > 0 || kk > 0) ? 1u : 0u);
            }
          }
          mma_commit(&empty[s]);
          if (kb == kblocks - 1)
            for (int op = 0; op < nA; ++op) mma_commit(&acc_full[slot[op]]);
        }
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------------------ scale stagers
    const int sp = warp & 3;
    const uint32_t t_lane = tmem + ((uint32_t)(sp * 32) << 16);
    int i = 0, gi = 0;
    for (int li = 0;; ++li) {
      const int it = next_item(li, true);
      if (it < 0) break;
      const bool glu = it < n13;
      const int kblocks = glu ? p.kb13 : p.kb2;
      for (int kb = 0; kb < kblocks; ++kb, ++i) {
        const int g = gi & 1;
        if ((kb & 3) == 0) mbar_wait(&sfg_full[g], (gi >> 1) & 1);
        const int s = i % kStages, n = i / kStages;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        const uint32_t* grp = reinterpret_cast<const uint32_t*>(sfbuf + g * kSfGrp) + (kb & 3) + lane * 4;
        const uint32_t col = t_lane + kSfCol0 + (uint32_t)(s * kSfCols);
        tmem_st4(col, grp[0], grp[128], grp[256], grp[384]);
        if (glu) tmem_st4(col + 4, grp[512], grp[512 + 128], grp[512 + 256], grp[512 + 384]);
        const uint32_t* gb = grp + 1024;
        tmem_st4(col + 8, gb[0], gb[128], gb[256], gb[384]);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&sf_full[s]);
          if ((kb & 3) == 3 || kb == kblocks - 1) mbar_arrive(&sfg_empty[g]);
        }
        if ((kb & 3) == 3 || kb == kblocks - 1) ++gi;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int sub = warp & 3, feat = sub * 32 + lane;
    const uint32_t t_lane = tmem + ((uint32_t)(sub * 32) << 16);
    int r = 0;
    int nu[2] = {0, 0};
    for (int li = 0;; ++li) {
      const int it = next_item(li, true);
      if (it < 0) break;
      const FItem f = fitem(p, n13, it);
      const Work wk = p.work[f.chunk];
      const int nA = f.glu ? 2 : 1;
      int slot[2] = {0, 0};
      for (int op = 0; op < nA; ++op) {
        const int sl = (r + op) & 1;
        slot[op] = sl;
        mbar_wait(&acc_full[sl], nu[sl] & 1);
        ++nu[sl];
      }
      r += nA;
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < kChunkMX / 32; ++c) {
        if (c * 32 >= wk.rows) break;
        uint32_t v[32];
        tmem_ld32(t_lane + slot[0] * 128 + c * 32, v);
        if (f.glu) {
          uint32_t u[32];
          tmem_ld32(t_lane + slot[1] * 128 + c * 32, u);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float hval = silu_fast(__uint_as_float(v[j])) * __uint_as_float(u[j]);
            float m = fabsf(hval);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffff, m, o));
            const int e = fmx_exp(m);
            const float inv = e < 127 ? __uint_as_float((uint32_t)(127 - e) << 23) : __uint_as_float(1u << 22);
            const int rr = c * 32 + j;
            if (rr < wk.rows) {
              const size_t row = (size_t)wk.row0 + rr;
              p.hq[row * p.I + f.mt * 128 + feat] =
                  (uint8_t)__nv_cvt_float_to_fp8(hval * inv, __NV_SATFINITE, __NV_E4M3);
              if (lane == 0) p.hsf[row * (p.I / 32) + f.mt * 4 + sub] = (uint8_t)(e + 127);
            }
          }
        } else {
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int rr = c * 32 + j;
            if (rr < wk.rows) p.y[((size_t)wk.row0 + rr) * p.H + f.mt * 128 + feat] = __uint_as_float(v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        for (int op = 0; op < nA; ++op) mbar_arrive(&acc_empty[slot[op]]);
      if (f.glu) {  // publish: this item's part of the chunk's intermediate is written
        __threadfence();
        epi_bar();
        if (warp == 2 && lane == 0) red_release_gpu_add(p.sched + 1 + f.chunk, 1);
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

size_t moe_ffn_mx_fused_smem() {
  using namespace moe::fused;
  return (size_t)kStages * kStage + 2 * kSfGrp + (4 * kStages + 8 + 2 * kRing) * 8 + kRing * 4 + 16 + 1024;
}

cudaError_t moe_ffn_mx_fused_launch(Ctx& ctx, const MoeGemmMxArgs& g13, const MoeGemmMxArgs& g2, int* sched,
                                    cudaStream_t stream) {
  using namespace moe;
  const int H = g13.H, I = g13.I, rows_w = g13.n_local + 1;
  CUtensorMap tw13, tx, tw13sf, txsf, tw2, th, tw2sf, thsf;
  auto map = [&](CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_c, uint32_t box_r,
                 bool swz) {
    const uint64_t dims[2] = {cols, rows};
    const uint64_t strides[1] = {cols};
    const uint32_t box[2] = {box_c, box_r};
    return encode_tma(ctx, m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                      swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  };
  if (!map(&tw13, g13.w, H, (uint64_t)rows_w * 2 * I, 128, 128, true) ||
      !map(&tx, g13.x, H, g13.rows_pad, 128, kChunkMX, true) ||
      !map(&tw13sf, g13.w_sf, H / 32, (uint64_t)rows_w * 2 * I, 16, 128, false) ||
      !map(&txsf, g13.x_sf, H / 32, g13.rows_pad, 16, 128, false) ||
      !map(&tw2, g2.w, I, (uint64_t)rows_w * H, 128, 128, true) ||
      !map(&th, g2.x, I, g2.rows_pad, 128, kChunkMX, true) ||
      !map(&tw2sf, g2.w_sf, I / 32, (uint64_t)rows_w * H, 16, 128, false) ||
      !map(&thsf, g2.x_sf, I / 32, g2.rows_pad, 16, 128, false))
    return cudaErrorInvalidValue;
  FusedMxParams p{};
  p.work = g13.work;
  p.n_work = g13.n_work;
  p.mt13 = I / 128;
  p.mt2 = H / 128;
  p.kb13 = H / 128;
  p.kb2 = I / 128;
  p.I = I;
  p.H = H;
  p.E = g13.E;
  p.expert_lo = g13.expert_lo;
  p.n_local = g13.n_local;
  p.hq = g13.hq;
  p.hsf = g13.hsf;
  p.y = g2.y;
  p.sched = sched;
  const size_t smem = moe_ffn_mx_fused_smem();
  if (const cudaError_t e = ensure_smem(moe_ffn_mx_fused_kernel, smem); e != cudaSuccess) return e;
  return launch_k(ctx.pdl, moe_ffn_mx_fused_kernel, dim3(ctx.num_sms), dim3(fused::kThreads), smem, stream, tw13, tx,
                  tw13sf, txsf, tw2, th, tw2sf, thsf, p);
}

}  // namespace afdk
