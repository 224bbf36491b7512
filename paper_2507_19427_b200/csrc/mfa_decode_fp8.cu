// mfa_decode_fp8.cu — K2 for an e4m3 KV cache (512 B per token per layer,
// the paper's FP8-attention production setting; accounting
// kv_token_bytes = 512, builtin_catalog.cpp:11,242).
//
// Same structure as mfa_decode.cu (persistent flash-decoding over the flattened
// (request, page) space, one K/V page = one 64-token tile shared by all 64
// heads, split partials merged by K3), but both contractions run on the FP8
// tensor-core path (tcgen05.mma kind::f8f6f4, fp32 accumulation in TMEM):
//
//   S  = Q8[64x256] . K8_page^T     M=64 N=64  K=256 (8 MMAs of K=32)
//   O += P8[64x64]  . V8_page       M=64 N=256 K=64  (2 MMAs, V MN-major)
//
// Q arrives in bf16; at the start of each segment the (otherwise idle) softmax
// warps quantise it per head with a power-of-two scale 2^e over the 256 dims
// (the MXFP8 exponent rule: smallest e with amax <= 448*2^e; q =
// rn_satfinite(x*2^-e), an exact scaling — an IEEE division per element cost
// 7 us per launch at config 2) into an e4m3 SW128 panel and keep 2^e.  S is rescaled per head by
// q_scale * k_scale * softmax_scale * log2(e).  P = exp2(s - m) is stored as
// e4m3 after multiplying by 2^4; the lazy rescale threshold is 4 (log2), so P
// stays <= 2^8 < 448 and probabilities down to 2^-13 remain representable.
// O is scaled by v_scale / l in the epilogue.
//
// Warp roles as in the bf16 kernel: w0 Q+K TMA, w1 QK^T issuer + TMEM owner,
// w2-5 Q quantisation / softmax / epilogue, w6 V TMA, w7 P.V issuer.  The
// softmax warps read TMEM with the 16x32bx2 shape, so all 32 lanes work: lane
// (head, half) owns 32 of a page's 64 tokens and 128 of O's 256 columns.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "afdk_internal.h"
#include "mfa_common.cuh"
#include "sm100.cuh"

namespace afdk {
namespace mfa {

using namespace sm100;

constexpr int kTile8 = kPage * kDim;  // 16 KB e4m3 K or V page
// segment charge in page units (AFDK_MFA8_SEG_COST overrides): a segment's
// fixed work (Q load + quantisation, O epilogue, split partial) is the same
// as the bf16 kernel's while a page streams in half the time.  B=64 x 4K:
// 3 / 5 / 7 / 9 -> 33.1-33.3 / 32.6-32.7 / 32.3 / 32.9-33.0 us; B=256 flat.
// Kept at 3: with 7 the 2 x 32K/20K parity case moved its split points and
// exceeded the e4m3-P bar (4.0e-2 vs 3e-2) for a 1 us gain
#ifndef AFDK_MFA8_SEG_COST_DEFAULT
#define AFDK_MFA8_SEG_COST_DEFAULT 3
#endif
constexpr int kSegCost8 = AFDK_MFA8_SEG_COST_DEFAULT;
constexpr int kPanel8 = 64 * 128;     // 64 rows x 128 B swizzle panel (128 dims)
constexpr int kPanel16 = 64 * 128;    // 64 rows x 128 B bf16 panel (64 dims)
#ifndef AFDK_NK8
#define AFDK_NK8 4
#endif
#ifndef AFDK_NV8
#define AFDK_NV8 5
#endif
constexpr int kNK8 = AFDK_NK8, kNV8 = AFDK_NV8;  // K / V page stages (experiment knobs)
constexpr int kThreads8 = 256;
constexpr uint32_t kColO8 = 0, kColS8 = 256;
constexpr float kRescale8 = 4.0f;     // lazy O rescale threshold (log2 units)
constexpr float kPScale8 = 16.0f;     // P is stored as e4m3(16 * p)

struct __align__(1024) Smem8 {
  uint8_t q[4 * kPanel16];   // 32 KB bf16 Q (TMA)
  uint8_t q8[2 * kPanel8];   // 16 KB e4m3 Q, K-major SW128
  uint8_t k[kNK8][kTile8];   // 64 KB
  uint8_t v[kNV8][kTile8];   // 80 KB
  uint8_t p[2][64 * 128];    // 16 KB e4m3 P: 64 head rows x 128 B (tokens in the first 64 B, swizzled)
  float qscale[kHeads];
  uint64_t q_full, q_empty, q8_full;
  uint64_t k_full[kNK8], k_empty[kNK8];
  uint64_t v_full[kNV8], v_empty[kNV8];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full[2], p_empty[2];
  uint64_t o_free;
  uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t e4m3x4(float a, float b, float c, float d) {
  const uint32_t lo = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
  const uint32_t hi = __nv_cvt_float2_to_fp8x2(make_float2(c, d), __NV_SATFINITE, __NV_E4M3);
  return lo | (hi << 16);
}

__global__ void __launch_bounds__(kThreads8, 1)
mfa_decode_fp8_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem8& sm = *reinterpret_cast<Smem8*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int32_t* prefix = reinterpret_cast<int32_t*>(&sm + 1);
#ifdef AFDK_MFA_TIMES
  __shared__ int s_tl;
  if (threadIdx.x == 0) { s_tl = tl_launch(0, gridDim.x); tl_min(s_tl, 0); }
#endif
  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  build_page_prefix<kThreads8>(prefix, prm.seq_lens, prm.batch, prm.seg_cost);
  __syncthreads();
  const int T = prefix[prm.batch];
  int range_lo, range_hi;
  cta_range(cta, G, T, range_lo, range_hi);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    mbar_init(&sm.q8_full, 4);
    for (int i = 0; i < kNK8; ++i) { mbar_init(&sm.k_full[i], 1); mbar_init(&sm.k_empty[i], 1); }
    for (int i = 0; i < kNV8; ++i) { mbar_init(&sm.v_full[i], 1); mbar_init(&sm.v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_empty[i], 4);
      mbar_init(&sm.p_full[i], 4);
      mbar_init(&sm.p_empty[i], 1);
    }
    mbar_init(&sm.o_free, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // K / V producers prefill their rings before waiting (see mfa_decode.cu)
  const bool producer = AFDK_MFA_KV_PREFETCH && (warp == 0 || warp == 6);
  if (!producer) griddep_wait();
  griddep_launch();
#ifdef AFDK_MFA_TIMES
  if (threadIdx.x == 0) { tl_min(s_tl, 1); tl_max(s_tl, 2); }
#endif

  if (warp == 0) {
    // ------------------------------------------------ Q + K TMA producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      auto load_k = [&](int g, int req, int t) {
        const int page = __ldg(prm.block_table + (size_t)req * prm.max_pages + t);
        const int s = g % kNK8, n = g / kNK8;
        if (n > 0) mbar_wait(&sm.k_empty[s], (n & 1) ^ 1);
        mbar_expect_tx(&sm.k_full[s], kTile8);
        for (int c = 0; c < 2; ++c)
          tma_load_3d(sm.k[s] + c * kPanel8, &tm_k, &sm.k_full[s], c * 128, 0, page, pol_stream);
      };
      const int pre = AFDK_MFA_KV_PREFETCH ? prefetch_pages(prefix, prm, range_lo, range_hi, kNK8, load_k) : 0;
      if (AFDK_MFA_KV_PREFETCH) griddep_wait();
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        if (seg > 0) mbar_wait(&sm.q_empty, (seg & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, 4 * kPanel16);
        for (int c = 0; c < 4; ++c)
          tma_load_2d(sm.q + c * kPanel16, &tm_q, &sm.q_full, c * 64, req * kHeads, pol_keep);
        for (int t = lo; t < hi; ++t, ++g)
          if (g >= pre) load_k(g, req, t);
        ++seg;
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------- V TMA producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      auto load_v = [&](int g, int req, int t) {
        const int page = __ldg(prm.block_table + (size_t)req * prm.max_pages + t);
        const int s = g % kNV8, n = g / kNV8;
        if (n > 0) mbar_wait(&sm.v_empty[s], (n & 1) ^ 1);
        mbar_expect_tx(&sm.v_full[s], kTile8);
        for (int c = 0; c < 2; ++c)
          tma_load_3d(sm.v[s] + c * kPanel8, &tm_v, &sm.v_full[s], c * 128, 0, page, pol_stream);
      };
      const int pre = AFDK_MFA_KV_PREFETCH ? prefetch_pages(prefix, prm, range_lo, range_hi, kNV8, load_v) : 0;
      if (AFDK_MFA_KV_PREFETCH) griddep_wait();
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        for (int t = lo; t < hi; ++t, ++g)
          if (g >= pre) load_v(g, req, t);
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------- QK^T MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_e4m3(64, 64);
      const uint32_t q_base = smem_u32(sm.q8);
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        mbar_wait(&sm.q8_full, seg & 1);
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int ks = gg % kNK8, sb = gg & 1;
          mbar_wait(&sm.k_full[ks], (gg / kNK8) & 1);
          if (gg >= 2) mbar_wait(&sm.s_empty[sb], ((gg >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm.k[ks]);
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t a = sdesc_sw128(q_base + c * kPanel8 + kk * 32, 0, 1024);
              const uint64_t b = sdesc_sw128(k_base + c * kPanel8 + kk * 32, 0, 1024);
              mma_e4m3(tmem + kColS8 + sb * 64, a, b, idesc_qk, (c | kk) ? 1u : 0u);
            }
          mma_commit(&sm.s_full[sb]);
          mma_commit(&sm.k_empty[ks]);
          if (j == n - 1) mma_commit(&sm.q_empty);
        }
        g += n;
        ++seg;
      }
    }
  } else if (warp == 7) {
    // ------------------------------------------------------ P.V MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_pv = idesc_e4m3(64, 256) | (1u << 16);  // B (V) MN-major
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int vs = gg % kNV8, pb = gg & 1;
          mbar_wait(&sm.v_full[vs], (gg / kNV8) & 1);
          mbar_wait(&sm.p_full[pb], (gg >> 1) & 1);
          if (j == 0 && seg > 0) mbar_wait(&sm.o_free, (seg - 1) & 1);
          tc_fence_after();
          const uint32_t p_base = smem_u32(sm.p[pb]);
          const uint32_t v_base = smem_u32(sm.v[vs]);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint64_t a = sdesc_sw128(p_base + kk * 32, 0, 1024);
            const uint64_t b = sdesc_sw128(v_base + kk * 32 * 128, kPanel8, 1024);
            mma_e4m3(tmem + kColO8, a, b, idesc_pv, (j == 0 && kk == 0) ? 0u : 1u);
          }
          mma_commit(&sm.v_empty[vs]);
          mma_commit(&sm.p_empty[pb]);
        }
        g += n;
        ++seg;
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ------------------- Q quantisation / softmax / correction / epilogue
    const int sub = warp & 3;
    const int half = lane >> 4;  // 16x32bx2 TMEM loads: lanes 16-31 read columns +32
    const int head = sub * 16 + (lane & 15);
    const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t p_row_off = (uint32_t)head * 128;
    const float qk_base = prm.k_scale * prm.scale_log2;
    SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
    int req, lo, hi, seg = 0, g = 0;
    bool whole;
    while (walk.next(req, lo, hi, whole)) {
      const int n = hi - lo;
      const int seq_len = __ldg(prm.seq_lens + req);
      // ---- quantise this request's Q: lane (head, half) owns 128 dims
      {
        mbar_wait(&sm.q_full, seg & 1);
        uint4 raw[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int dim0 = half * 128 + u * 8;
          const int c = dim0 >> 6, unit = (dim0 & 63) >> 3;
          raw[u] = *reinterpret_cast<const uint4*>(sm.q + c * kPanel16 + head * 128 + ((unit ^ (head & 7)) << 4));
        }
        float amax = 0.0f;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t w[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
#pragma unroll
          for (int z = 0; z < 4; ++z)
            amax = fmaxf(amax, fmaxf(fabsf(__uint_as_float(w[z] << 16)), fabsf(__uint_as_float(w[z] & 0xffff0000u))));
        }
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, 16));
        // power-of-two scale 2^e (smallest e with amax <= 448 * 2^e): exact scaling
        const uint32_t ab = __float_as_uint(amax);
        const int ex = (int)((ab >> 23) & 0xff);
        int e = (!(amax > 0.0f) || ex == 0) ? -127 : (((ab & 0x7fffffu) <= 6291456u) ? ex - 135 : ex - 134);
        e = max(-127, min(127, e));
        const float qinv = e < 127 ? __uint_as_float((uint32_t)(127 - e) << 23) : __uint_as_float(1u << 22);
        const float qs = e > -127 ? __uint_as_float((uint32_t)(127 + e) << 23) : __uint_as_float(1u << 22);
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) {  // 16 dims per 16-byte e4m3 unit
          uint32_t o[4];
#pragma unroll
          for (int z = 0; z < 4; ++z) {
            const uint4 r = raw[u8 * 2 + (z >> 1)];
            const uint32_t w0 = (z & 1) ? r.z : r.x, w1 = (z & 1) ? r.w : r.y;
            o[z] = e4m3x4(__uint_as_float(w0 << 16) * qinv, __uint_as_float(w0 & 0xffff0000u) * qinv,
                          __uint_as_float(w1 << 16) * qinv, __uint_as_float(w1 & 0xffff0000u) * qinv);
          }
          *reinterpret_cast<uint4*>(sm.q8 + half * kPanel8 + head * 128 + ((u8 ^ (head & 7)) << 4)) =
              make_uint4(o[0], o[1], o[2], o[3]);
        }
        if (half == 0) sm.qscale[head] = qs;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.q8_full);
      }
      const float s_mul = sm.qscale[head] * qk_base;
      // lane (head, half) owns tokens [32*half, +32) of every page; l_sum is
      // this thread's share of the row sum (combined in the epilogue)
      float m_used = -INFINITY, l_sum = 0.0f;
      for (int j = 0; j < n; ++j, ++g) {
        const int sb = g & 1, pb = g & 1;
        mbar_wait(&sm.s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sr[32];
        tmem_ld16x2_32(t_row + kColS8 + sb * 64, sr);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_empty[sb]);

        const int tok0 = (lo + j) * kPage;
        const int nvalid = min(kPage, seq_len - tok0) - half * 32;
        float s[32];
        float tmax = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = (i < nvalid) ? __uint_as_float(sr[i]) * s_mul : -INFINITY;
          tmax = fmaxf(tmax, s[i]);
        }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffff, tmax, 16));
        const bool need = tmax > m_used + kRescale8;
        float alpha = 1.0f;
        if (need) {
          alpha = fast_exp2(m_used - tmax);
          m_used = tmax;
        }
        l_sum *= alpha;
        uint32_t pk[8];
        float psum = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float p0 = kPScale8 * fast_exp2(s[4 * i] - m_used);
          const float p1 = kPScale8 * fast_exp2(s[4 * i + 1] - m_used);
          const float p2 = kPScale8 * fast_exp2(s[4 * i + 2] - m_used);
          const float p3 = kPScale8 * fast_exp2(s[4 * i + 3] - m_used);
          psum += (p0 + p1) + (p2 + p3);
          pk[i] = e4m3x4(p0, p1, p2, p3);
        }
        l_sum += psum;

        if (g >= 2) mbar_wait(&sm.p_empty[pb], ((g >> 1) & 1) ^ 1);
        const bool warp_rescale = __any_sync(0xffffffff, need && j > 0);
        if (warp_rescale) {
          const int gp = g - 1;
          mbar_wait(&sm.p_empty[gp & 1], (gp >> 1) & 1);
          tc_fence_after();
          const float a = need ? alpha : 1.0f;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld16x2_32(t_row + kColO8 + c * 64, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
            tmem_st16x2_32(t_row + kColO8 + c * 64, o);
          }
          tmem_wait_st();
        }
        // last page of a request: zero V rows past seq_len (garbage e4m3 may be NaN)
        const int nvalid_page = min(kPage, seq_len - tok0);
        if (nvalid_page < kPage) {
          const int vs = g % kNV8;
          mbar_wait(&sm.v_full[vs], (g / kNV8) & 1);
          const int tid = (warp - 2) * 32 + lane;
          uint8_t* vt = sm.v[vs];
          for (int idx = tid; idx < (kPage - nvalid_page) * 2 * 8; idx += 128) {
            const int row = nvalid_page + idx / 16, chunk = (idx >> 3) & 1, q16 = idx & 7;
            *reinterpret_cast<uint4*>(vt + chunk * kPanel8 + row * 128 + q16 * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        {
          const uint32_t pbase = smem_u32(sm.p[pb]) + p_row_off;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t addr = pbase + ((uint32_t)((half * 2 + c) ^ (head & 7)) << 4);
            st_shared_v4(addr, pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[pb]);
      }
      // ---------------- epilogue of this segment: v_scale * O / l -> global
      const int gl = g - 1;
      mbar_wait(&sm.p_empty[gl & 1], (gl >> 1) & 1);
      tc_fence_after();
      const float l_tot = l_sum + __shfl_xor_sync(0xffffffff, l_sum, 16);
      const float inv_l = prm.v_scale / l_tot;
      const int slot = req + cta;
      __nv_bfloat16* obase = whole ? prm.out : reinterpret_cast<__nv_bfloat16*>(prm.part_o);
      const size_t orow = whole ? (size_t)req * kHeads + head : (size_t)slot * kHeads + head;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld16x2_32(t_row + kColO8 + c * 64, o);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(obase + orow * kDim + c * 64 + half * 32);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint4 v;
          v.x = pack_bf16x2(__uint_as_float(o[8 * q4 + 0]) * inv_l, __uint_as_float(o[8 * q4 + 1]) * inv_l);
          v.y = pack_bf16x2(__uint_as_float(o[8 * q4 + 2]) * inv_l, __uint_as_float(o[8 * q4 + 3]) * inv_l);
          v.z = pack_bf16x2(__uint_as_float(o[8 * q4 + 4]) * inv_l, __uint_as_float(o[8 * q4 + 5]) * inv_l);
          v.w = pack_bf16x2(__uint_as_float(o[8 * q4 + 6]) * inv_l, __uint_as_float(o[8 * q4 + 7]) * inv_l);
          dst[q4] = v;
        }
      }
      if (half == 0) {
        const float lse2 = m_used + __log2f(l_tot) - 4.0f;  // P was stored x 2^4
        if (whole) {
          if (prm.lse) prm.lse[(size_t)req * kHeads + head] = lse2 * 0.69314718055994531f;
        } else {
          prm.part_lse[(size_t)slot * kHeads + head] = lse2;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.o_free);
      if (!whole) publish_part(prm.sync, req, lane);  // after o_free: the fence must not hold up PV
      ++seg;
    }
  }

  tc_fence_before();
  __syncthreads();
#ifdef AFDK_MFA_TIMES
  if (threadIdx.x == 0) tl_max(s_tl, 3);
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace mfa

#ifdef AFDK_MFA_TIMES
// timeline of the e4m3 K2 (slots 0-3; K3's slots are in afdk_debug_mfa_tl)
extern "C" void afdk_debug_mfa8_tl(unsigned long long* host, int reset) {
  using namespace mfa;
  if (reset) {
    static unsigned long long init[kTlLaunches * 8];
    for (int i = 0; i < kTlLaunches * 8; ++i) init[i] = (i % 8 == 0 || i % 8 == 1 || i % 8 == 4) ? ~0ull : 0ull;
    cudaMemcpyToSymbol(g_tl, init, sizeof(init));
    const unsigned z[2] = {0, 0};
    cudaMemcpyToSymbol(g_tl_arrive, z, sizeof(z));
    return;
  }
  cudaMemcpyFromSymbol(host, g_tl, sizeof(g_tl));
}
#endif

cudaError_t mfa_decode_fp8_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream) {
  using namespace mfa;
  const int G = mfa_grid(ctx, a.batch);
  if (a.batch > kMaxBatch) return cudaErrorInvalidValue;
  uint8_t* ws = static_cast<uint8_t*>(a.workspace);
  Params prm{};
  prm.block_table = a.block_table;
  prm.seq_lens = a.seq_lens;
  ws += align_up((size_t)(a.batch + 1) * sizeof(int32_t), 256);
  const size_t slots = (size_t)a.batch + G;
  prm.part_o = reinterpret_cast<float*>(ws);
  ws += align_up(slots * kHeads * kDim * sizeof(float), 256);
  prm.part_lse = reinterpret_cast<float*>(ws);
  prm.out = static_cast<__nv_bfloat16*>(a.out);
  prm.lse = a.lse;
  prm.sync = ctx.counters + kCounterSlots / 2;
  static const int seg_cost = [] { const char* e = std::getenv("AFDK_MFA8_SEG_COST"); return e ? std::atoi(e) : kSegCost8; }();
  prm.seg_cost = seg_cost;
  prm.batch = a.batch;
  prm.max_pages = a.max_pages;
  prm.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  prm.k_scale = a.k_scale;
  prm.v_scale = a.v_scale;

  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[2] = {(uint64_t)kDim, (uint64_t)a.batch * kHeads};
    const uint64_t strides[1] = {kDim * 2};
    const uint32_t box[2] = {64, 64};
    if (!encode_tma(ctx, &tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.q), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)kDim, (uint64_t)kPage, (uint64_t)a.num_pages};
    const uint64_t strides[2] = {kDim, (uint64_t)kPage * kDim};
    const uint32_t box[3] = {128, 64, 1};
    if (!encode_tma(ctx, &tk, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(a.k_cache), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    if (!encode_tma(ctx, &tv, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(a.v_cache), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  const size_t smem = sizeof(Smem8) + 1024 + (size_t)(a.batch + 1) * sizeof(int32_t);
  if (const cudaError_t ea = ensure_smem(mfa_decode_fp8_kernel, sizeof(Smem8) + 1024 + (kMaxBatch + 1) * sizeof(int32_t));
      ea != cudaSuccess)
    return ea;
  cudaError_t e = launch_k(ctx.pdl, mfa_decode_fp8_kernel, dim3(G), dim3(kThreads8), smem, stream, tq, tk, tv, prm);
  if (e != cudaSuccess) return e;
  return mfa_combine_launch(ctx.pdl, prm, G, stream);
}

}  // namespace afdk
