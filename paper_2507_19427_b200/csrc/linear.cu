// linear.cu — decode-shaped weight-streaming GEMM on sm_100a (K1/K4 projections).
//
// Y[m_tok, n_out] = X[m_tok, K] . W[n_out, K]^T with m_tok <= 512 decode tokens
// and large bf16 weights (q_down|k|v 2560x7168, q_up 16384x2048, o 7168x16384;
// builtin_catalog.cpp:243-247).  At decode batch sizes the op is bound by
// streaming W from HBM once, so the kernel is "swap-AB": the weight tile is
// the MMA's M=128 side and the tokens are N (<=256), accumulating in TMEM:
//
//   D[128 feats x N tok] += W[128 x 64k] . X[N x 64k]^T   tcgen05.mma kind::f16
//
// (N > 256 — the AFD attention micro-batch above 256 requests — runs as two
// MMAs of N/2 sharing the weight panel: the token panel is loaded as two
// N/2-row boxes, the accumulator spans N TMEM columns, single-buffered.)
//
// Work is split stream-K style: the (tile, k-block) unit space is cut into one
// contiguous range per SM so every SM streams the same weight bytes whatever
// the layer shape.  Each (tile, k-range) segment writes an fp32 partial to
// slot (tile + cta); the row epilogues (mfa_layer.cu, linear_store_kernel) sum
// a tile's partials in CTA order — deterministic, no float atomics — fused
// with the row op that follows (RMSNorm, RoPE, KV append, residual).
//
// Roles (192 threads): w0 TMA producer, w1 MMA issuer + TMEM owner, w2-5 epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "afdk_internal.h"
#include "linear.cuh"
#include "sm100.cuh"

namespace afdk {
namespace lin {

using namespace sm100;

constexpr int kThreads = 192;
constexpr int kABytes = kBM * 128;  // 16 KB weight panel per k-block

struct KParams {
  LinearPlan plan;
  float* part;  // [(tiles + G)][m_tok][128] fp32 segment partials
  int stage_bytes, stages;
  // kRope mode (q_up with NeoX RoPE fused, one whole tile per CTA): tile t
  // holds the 64 pairs [j*64, j*64+64) of head h (h = t / tph, j = t % tph,
  // tph = head_dim/128): weight rows x1 = h*head_dim + j*64 + [0,64) in TMEM
  // lanes 0-63, x2 = x1 + head_dim/2 in lanes 64-127
  __nv_bfloat16* q_out;   // [m_tok, n_out] bf16, rotated
  const float2* rope_cs;  // [m_tok, head_dim/2] (cos, sin) of each row's position
  int head_dim;
  int w_dep;  // the weight operand is a predecessor's output (the router's token rows): no PDL prefill
};

__device__ __forceinline__ void unit_range(int c, int G, int U, int& lo, int& hi) {
  lo = (int)(((long long)c * U) / G);
  hi = (int)(((long long)(c + 1) * U) / G);
}

template <bool kRope, bool kM2, bool kW>  // kW: n_mma > 256, two MMAs of n_mma/2 per k-step
__global__ void __launch_bounds__(kThreads, 1)
linear_bf16_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                   const KParams kp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const LinearPlan& P = kp.plan;
  const int S = kp.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * kp.stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = warp_id(), lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int U = P.tiles * P.kblocks;
  int u_lo, u_hi;
  unit_range(cta, G, U, u_lo, u_hi);

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
  griddep_launch();
  const uint32_t tmem = *tmem_slot;
  const int n_mma = P.n_mma;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const uint32_t bytes = (kM2 ? 2 : 1) * kABytes + n_mma * 128;
      // token panel: one box of n_mma rows, or two of n_mma/2 (kW)
      auto load_x = [&](uint8_t* dst, uint64_t* bar, int kb) {
        tma_load_2d(dst, &tm_x, bar, kb * 64, 0, pol_x);
        if (kW) tma_load_2d(dst + (n_mma / 2) * 128, &tm_x, bar, kb * 64, n_mma / 2, pol_x);
      };
      // kRope: the panel's rows 0-63 are the pairs' x1 rows, 64-127 their x2 rows
      const int tph = kRope ? kp.head_dim / 128 : 1;
      auto load_w = [&](uint8_t* dst, uint64_t* bar, int kb, int tile) {
        if (kRope) {
          const int r1 = (tile / tph) * kp.head_dim + (tile % tph) * 64;
          tma_load_2d(dst, &tm_w, bar, kb * 64, r1, pol_w);
          tma_load_2d(dst + kABytes / 2, &tm_w, bar, kb * 64, r1 + kp.head_dim / 2, pol_w);
        } else if (kM2) {  // two 128-row panels of a 256-row tile
          tma_load_2d(dst, &tm_w, bar, kb * 64, tile * 256, pol_w);
          tma_load_2d(dst + kABytes, &tm_w, bar, kb * 64, tile * 256 + kBM, pol_w);
        } else {
          tma_load_2d(dst, &tm_w, bar, kb * 64, tile * kBM, pol_w);
        }
      };
      // weights never depend on the previous kernel: fill the first S stages'
      // weight panels before waiting for the predecessor (PDL), then the X panels
      const int pro = min(S, u_hi - u_lo);
      if (kp.w_dep) griddep_wait();
      for (int i = 0; i < pro; ++i) {
        const int u = u_lo + i, tile = u / P.kblocks, kb = u % P.kblocks;
        mbar_expect_tx(&full[i], bytes);
        load_w(smem + i * kp.stage_bytes, &full[i], kb, tile);
      }
      if (!kp.w_dep) griddep_wait();
      for (int i = 0; i < pro; ++i) {
        const int u = u_lo + i, kb = u % P.kblocks;
        load_x(smem + i * kp.stage_bytes + (kM2 ? 2 : 1) * kABytes, &full[i], kb);
      }
      for (int u = u_lo + pro, i = pro; u < u_hi; ++u, ++i) {
        const int s = i % S, n = i / S;
        if (n > 0) mbar_wait(&empty[s], (n & 1) ^ 1);
        const int tile = u / P.kblocks, kb = u % P.kblocks;
        uint8_t* st = smem + s * kp.stage_bytes;
        mbar_expect_tx(&full[s], bytes);
        load_w(st, &full[s], kb, tile);
        load_x(st + (kM2 ? 2 : 1) * kABytes, &full[s], kb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, (uint32_t)(kW ? n_mma / 2 : n_mma), false, false);
      // kM2: two accumulators (panel 0 / 1) of n_mma columns per segment; they
      // double-buffer across segments only while 4 x n_mma fits TMEM
      const bool dbuf = kM2 ? n_mma <= 128 : !kW;
      int seg = 0;
      for (int u = u_lo, i = 0; u < u_hi; ++seg) {
        const int tile = u / P.kblocks;
        const int seg_end = min(u_hi, (tile + 1) * P.kblocks);
        const int ab = dbuf ? (seg & 1) : 0, na = dbuf ? (seg >> 1) : seg;
        if (dbuf ? seg >= 2 : seg >= 1) mbar_wait(&acc_empty[ab], (na & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + (kM2 ? ab * 2 * n_mma : ab * 256);
        for (bool first = true; u < seg_end; ++u, ++i, first = false) {
          const int s = i % S, n = i / S;
          mbar_wait(&full[s], n & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * kp.stage_bytes);
          const uint32_t b_base = a_base + (kM2 ? 2 : 1) * kABytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t b = sdesc_sw128(b_base + kk * 32, 0, 1024);
            mma_bf16(d, sdesc_sw128(a_base + kk * 32, 0, 1024), b, idesc, (first && kk == 0) ? 0u : 1u);
            if (kM2)
              mma_bf16(d + n_mma, sdesc_sw128(a_base + kABytes + kk * 32, 0, 1024), b, idesc,
                       (first && kk == 0) ? 0u : 1u);
            if (kW)  // tokens [n_mma/2, n_mma): second half of the panel, columns n_mma/2..
              mma_bf16(d + n_mma / 2, sdesc_sw128(a_base + kk * 32, 0, 1024),
                       sdesc_sw128(b_base + (n_mma / 2) * 128 + kk * 32, 0, 1024), idesc,
                       (first && kk == 0) ? 0u : 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[ab]);
      }
    }
  } else if (kRope) {
    // epilogue (one whole tile): bf16-round the q_up output (the oracle's
    // storage point), exchange x1 / x2 of each pair through smem between the
    // warp pairs (sub 0 <-> 2, 1 <-> 3: lane l of both is pair i = j*64 +
    // (sub&1)*32 + l), rotate with the row's (cos, sin) — the qkv epilogue's
    // double-precision table — and store bf16 q.
    const int sub = warp & 3, pair = sub & 1, hi = sub >> 1;
    const int tile = u_lo / P.kblocks, tph = kp.head_dim / 128, half = kp.head_dim / 2;
    const int fi = (tile % tph) * 64 + pair * 32 + lane;  // frequency / pair index in the head
    const int col = (tile / tph) * kp.head_dim + fi + (hi ? half : 0);
    float* xch = reinterpret_cast<float*>(tmem_slot + 4) + pair * 2 * 32 * 33;  // [2 halves][32 tok][33]
    griddep_wait();  // the (cos, sin) table comes from the qkv epilogue
    // this lane's (cos, sin) for 32 tokens, loaded as one batch (independent
    // L2 loads in flight); chunk 0's before the accumulator is ready
    float2 cs[32];
    auto load_cs = [&](int c) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        cs[j] = (c + j < P.m_tok) ? __ldg(kp.rope_cs + (size_t)(c + j) * half + fi) : make_float2(0.f, 0.f);
    };
    load_cs(0);
    mbar_wait(&acc_full[0], 0);
    tc_fence_after();
    const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16);
    float* mine = xch + hi * 32 * 33;
    const float* other = xch + (hi ^ 1) * 32 * 33;
    for (int c = 0; c < n_mma; c += 32) {
      uint32_t v[32];
      tmem_ld32(t_row + c, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) mine[j * 33 + lane] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(v[j])));
      asm volatile("bar.sync %0, 64;" ::"r"(1 + pair));
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int t = c + j;
        const float x = mine[j * 33 + lane], y = other[j * 33 + lane];
        // x1' = x1 c - x2 s ; x2' = x2 c + x1 s
        const float o = hi ? (x * cs[j].x + y * cs[j].y) : (x * cs[j].x - y * cs[j].y);
        if (t < P.m_tok) kp.q_out[(size_t)t * P.n_out + col] = __float2bfloat16_rn(o);
      }
      asm volatile("bar.sync %0, 64;" ::"r"(1 + pair));
      if (c + 32 < n_mma) load_cs(c + 32);
    }
  } else {
    // epilogue: TMEM lane = weight row = output feature, column = token;
    // each (tile, k-range) segment writes its fp32 partial to slot tile + cta.
    const int sub = warp & 3;
    const int feat = sub * 32 + lane;
    const bool dbuf = kM2 ? n_mma <= 128 : !kW;
    int seg = 0;
    for (int u = u_lo; u < u_hi; ++seg) {
      const int tile = u / P.kblocks;
      const int seg_end = min(u_hi, (tile + 1) * P.kblocks);
      u = seg_end;
      const int ab = dbuf ? (seg & 1) : 0, na = dbuf ? (seg >> 1) : seg;
      mbar_wait(&acc_full[ab], na & 1);
      tc_fence_after();
      constexpr int kMt = kM2 ? 2 * kBM : kBM;  // == P.mtile (compile-time: immediate store offsets)
#pragma unroll 1
      for (int pnl = 0; pnl < (kM2 ? 2 : 1); ++pnl) {
        float* dst = kp.part + ((size_t)(tile + cta) * P.m_tok) * kMt + pnl * kBM + feat;
        const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16) + (kM2 ? (ab * 2 + pnl) * n_mma : ab * 256);
        for (int c = 0; c < n_mma; c += 32) {
          uint32_t v[32];
          tmem_ld32(t_row + c, v);
          tmem_wait_ld();
          float* d = dst + (size_t)c * kMt;
          const int nv = P.m_tok - c;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) d[j * kMt] = __uint_as_float(v[j]);
        }
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

// Plain output: out[row, f] = sum of partials (fixed order), bf16 or fp32.
__global__ void __launch_bounds__(256) linear_store_kernel(const LinearPlan P, const float* __restrict__ part,
                                                           int G, void* __restrict__ out, int out_fp32) {
  __shared__ SlotTable tab;
  build_slot_table(P, G, tab);
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x;
  for (int f = blockIdx.y * 256 + threadIdx.x; f < P.n_out; f += 256 * gridDim.y) {
    const float v = tab.sum(P, part, row, f);
    if (out_fp32) static_cast<float*>(out)[(size_t)row * P.n_out + f] = v;
    else static_cast<__nv_bfloat16*>(out)[(size_t)row * P.n_out + f] = __float2bfloat16_rn(v);
  }
}

}  // namespace lin

int linear_grid(const Ctx& ctx, const LinearPlan& p) {
  // no CTA without units, and no tile shared by more than kMaxSegs CTAs
  long long g = ctx.num_sms;
  const long long U = (long long)p.tiles * p.kblocks;
  if (g > U) g = U;
  if (g > (long long)(lin::kMaxSegs - 1) * p.tiles) g = (long long)(lin::kMaxSegs - 1) * p.tiles;
  // nearly one tile per SM (q_up: 128 tiles on 148 SMs): one whole tile per
  // CTA, no split partials — measured ~1 us faster per layer than stream-K
  if (p.tiles <= ctx.num_sms && (long long)p.tiles * 20 >= (long long)ctx.num_sms * 17) g = p.tiles;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t linear_store_launch(Ctx& ctx, const LinearPlan& p, const float* part, void* out, bool out_fp32,
                                cudaStream_t stream) {
  const int gy = (p.n_out + 255) / 256 > 8 ? 8 : (p.n_out + 255) / 256;
  return launch_k(ctx.pdl, lin::linear_store_kernel, dim3(p.m_tok, gy), dim3(256), 0, stream, p, part,
                  linear_grid(ctx, p), out, out_fp32 ? 1 : 0);
}

LinearPlan make_linear_plan(int m_tok, int n_out, int k) {
  LinearPlan p{};
  p.m_tok = m_tok;
  p.n_mma = ((m_tok + 15) / 16) * 16;
  if (p.n_mma < 16) p.n_mma = 16;
  if (p.n_mma > 256) p.n_mma = ((m_tok + 31) / 32) * 32;  // two MMAs of n_mma/2 (a multiple of 16)
  p.n_out = n_out;
  p.k = k;
  // 256-row tiles (two MMA panels sharing each token panel; AFDK_LIN_MTILE=256)
  // halve the L2->smem bytes per FLOP at wide token panels but were slower
  // end to end: attention layer B=256 317.5 vs 295.0 us, B=128 185.6 vs
  // 177.2 us (3 pipeline stages instead of 4, single-buffered accumulators,
  // half the stream-K tiles), so 128-row tiles stay the default
  static const int env = [] { const char* e = std::getenv("AFDK_LIN_MTILE"); return e ? std::atoi(e) : 0; }();
  p.mtile = (n_out >= 2048 && env == 256 && p.n_mma <= 256) ? 256 : lin::kBM;
  p.tiles = (n_out + p.mtile - 1) / p.mtile;
  p.kblocks = k / 64;
  return p;
}

size_t linear_workspace_bytes(const LinearPlan& p, int num_sms) {
  return align_up((size_t)(p.tiles + num_sms) * p.m_tok * p.mtile * sizeof(float), 256);
}

static cudaError_t linear_launch_impl(Ctx& ctx, const LinearPlan& p, const void* x, const void* w, float* part,
                                      __nv_bfloat16* q_out, const float2* rope_cs, int head_dim,
                                      cudaStream_t stream, bool w_dep = false) {
  using namespace lin;
  const bool rope = q_out != nullptr;
  CUtensorMap tw, tx;
  {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.n_out};
    const uint64_t strides[1] = {(uint64_t)p.k * 2};
    const uint32_t box[2] = {64, rope ? (uint32_t)(kBM / 2) : (uint32_t)kBM};
    if (!encode_tma(ctx, &tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)p.k, (uint64_t)p.m_tok};
    const uint64_t strides[1] = {(uint64_t)p.k * 2};
    const uint32_t box[2] = {64, (uint32_t)(p.n_mma > 256 ? p.n_mma / 2 : p.n_mma)};
    if (!encode_tma(ctx, &tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  KParams kp{};
  kp.plan = p;
  kp.part = part;
  kp.q_out = q_out;
  kp.rope_cs = rope_cs;
  kp.head_dim = head_dim;
  kp.w_dep = w_dep ? 1 : 0;
  const bool m2 = p.mtile == 256 && !rope;
  kp.stage_bytes = (m2 ? 2 : 1) * kABytes + p.n_mma * 128;
  const int xch_bytes = rope ? 2 * 2 * 32 * 33 * 4 : 0;  // x1/x2 exchange of the two warp pairs
  const int budget = 200 * 1024 - xch_bytes;
  kp.stages = budget / kp.stage_bytes;
  if (kp.stages > 8) kp.stages = 8;
  const size_t smem = (size_t)kp.stages * kp.stage_bytes + 1024 + 256 + xch_bytes;
  const int grid = linear_grid(ctx, p);
  auto go = [&](auto kernel) -> cudaError_t {
    if (const cudaError_t e = ensure_smem(kernel, smem); e != cudaSuccess) return e;
    return launch_k(ctx.pdl, kernel, dim3(grid), dim3(kThreads), smem, stream, tw, tx, kp);
  };
  if (rope) return go(linear_bf16_kernel<true, false, false>);
  if (m2) return go(linear_bf16_kernel<false, true, false>);
  return p.n_mma > 256 ? go(linear_bf16_kernel<false, false, true>) : go(linear_bf16_kernel<false, false, false>);
}

cudaError_t linear_bf16_launch(Ctx& ctx, const LinearPlan& p, const void* x, const void* w, float* part,
                               cudaStream_t stream, bool w_dep) {
  return linear_launch_impl(ctx, p, x, w, part, nullptr, nullptr, 0, stream, w_dep);
}

bool linear_rope_fusable(const Ctx& ctx, const LinearPlan& p, int head_dim) {
  return p.mtile == lin::kBM && head_dim % 128 == 0 && p.n_out % head_dim == 0 && linear_grid(ctx, p) == p.tiles;
}

cudaError_t linear_bf16_rope_launch(Ctx& ctx, const LinearPlan& p, const void* x, const void* w,
                                    __nv_bfloat16* q_out, const float2* rope_cs, int head_dim,
                                    cudaStream_t stream) {
  if (!linear_rope_fusable(ctx, p, head_dim)) return cudaErrorInvalidValue;
  return linear_launch_impl(ctx, p, x, w, nullptr, q_out, rope_cs, head_dim, stream);
}


}  // namespace afdk
