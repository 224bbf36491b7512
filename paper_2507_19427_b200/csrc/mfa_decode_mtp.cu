// mfa_decode_mtp.cu — K2 for multi-token decode (MTP, mtp = 2): the two newest
// tokens of every request query the paged bf16 KV cache together.
//
// The reference prices MTP as a multiplier on the attention FLOPs with the KV
// bytes unchanged (costmodel.cpp:46-58): one KV page now
// feeds 2 x 64 query rows.  On sm_100a that is simply an M=128 contraction
// (every TMEM lane holds a row) instead of M=64:
//
//   S  = Q[128x256] . K_page^T   tcgen05.mma kind::f16 M=128 N=64  K=256
//   O += P[128x64]  . V_page     tcgen05.mma kind::f16 M=128 N=256 K=64
//
// Row r = j*64 + h (query token j of the request, head h).  Token j sits at
// position L-2+j and attends causally to positions <= L-2+j, so the last page
// of a request masks one more key for j = 0 than for j = 1.  A row that sees
// no key (L = 1, j = 0) produces zeros and LSE = -inf, also through K3.
//
// Same persistent flash-decoding split, warp roles and barriers as
// mfa_decode.cu; rings are 2 K + 2 V pages so that the 64 KB query tile fits.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "afdk_internal.h"
#include "mfa_common.cuh"
#include "sm100.cuh"

namespace afdk {
namespace mfa {

using namespace sm100;

constexpr int kMtp = 2;
constexpr int kRowsM = kHeads * kMtp;          // 128 query rows per request
constexpr int kTileM = kPage * kDim * 2;       // 32 KB bf16 K or V page
constexpr int kChunkKV = 64 * 128;             // 64 token rows x 128 B (64 dims)
constexpr int kChunkQ = kRowsM * 128;          // 128 query rows x 128 B (64 dims)
constexpr int kNKm = 2, kNVm = 2;
constexpr int kThreadsM = 256;
constexpr uint32_t kColOm = 0, kColSm = 256;
constexpr float kRescaleM = 8.0f;
constexpr int kMaxBatchMtp = 128;  // the 224 KB of tiles leave ~1.5 KB for the page prefix

struct __align__(1024) SmemM {
  uint8_t q[4 * kChunkQ];          // 64 KB
  uint8_t k[kNKm][kTileM];         // 64 KB
  uint8_t v[kNVm][kTileM];         // 64 KB
  uint8_t p[2][kRowsM * kPage * 2];  // 32 KB bf16 P (K-major SW128, 128 B per row)
  uint64_t q_full, q_empty;
  uint64_t k_full[kNKm], k_empty[kNKm];
  uint64_t v_full[kNVm], v_empty[kNVm];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full[2], p_empty[2];
  uint64_t o_free;
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreadsM, 1)
mfa_decode_mtp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, const Params prm) {
  extern __shared__ uint8_t smem_raw[];
  SmemM& sm = *reinterpret_cast<SmemM*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int32_t* prefix = reinterpret_cast<int32_t*>(&sm + 1);
  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  build_page_prefix<kThreadsM>(prefix, prm.seq_lens, prm.batch, prm.seg_cost);
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
    for (int i = 0; i < kNKm; ++i) { mbar_init(&sm.k_full[i], 1); mbar_init(&sm.k_empty[i], 1); }
    for (int i = 0; i < kNVm; ++i) { mbar_init(&sm.v_full[i], 1); mbar_init(&sm.v_empty[i], 1); }
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
  griddep_wait();
  griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------ Q + K TMA producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      const uint64_t pol_keep = policy_evict_last();
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        if (seg > 0) mbar_wait(&sm.q_empty, (seg & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, 4 * kChunkQ);
        for (int c = 0; c < 4; ++c)
          tma_load_2d(sm.q + c * kChunkQ, &tm_q, &sm.q_full, c * 64, req * kRowsM, pol_keep);
        for (int t = lo; t < hi; ++t, ++g) {
          const int page = __ldg(prm.block_table + (size_t)req * prm.max_pages + t);
          const int s = g % kNKm, n = g / kNKm;
          if (n > 0) mbar_wait(&sm.k_empty[s], (n & 1) ^ 1);
          mbar_expect_tx(&sm.k_full[s], kTileM);
          for (int c = 0; c < 4; ++c)
            tma_load_3d(sm.k[s] + c * kChunkKV, &tm_k, &sm.k_full[s], c * 64, 0, page, pol_stream);
        }
        ++seg;
      }
    }
  } else if (warp == 6) {
    // ---------------------------------------------------- V TMA producer
    if (lane == 0) {
      const uint64_t pol_stream = policy_evict_first();
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        for (int t = lo; t < hi; ++t, ++g) {
          const int page = __ldg(prm.block_table + (size_t)req * prm.max_pages + t);
          const int s = g % kNVm, n = g / kNVm;
          if (n > 0) mbar_wait(&sm.v_empty[s], (n & 1) ^ 1);
          mbar_expect_tx(&sm.v_full[s], kTileM);
          for (int c = 0; c < 4; ++c)
            tma_load_3d(sm.v[s] + c * kChunkKV, &tm_v, &sm.v_full[s], c * 64, 0, page, pol_stream);
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------- QK^T MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(128, 64, false, false);
      const uint32_t q_base = smem_u32(sm.q);
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        mbar_wait(&sm.q_full, seg & 1);
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int ks = gg % kNKm, sb = gg & 1;
          mbar_wait(&sm.k_full[ks], (gg / kNKm) & 1);
          if (gg >= 2) mbar_wait(&sm.s_empty[sb], ((gg >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm.k[ks]);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t a = sdesc_sw128(q_base + c * kChunkQ + kk * 32, 0, 1024);
              const uint64_t b = sdesc_sw128(k_base + c * kChunkKV + kk * 32, 0, 1024);
              mma_bf16(tmem + kColSm + sb * 64, a, b, idesc_qk, (c | kk) ? 1u : 0u);
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
      constexpr uint32_t idesc_pv = idesc_bf16(128, 256, false, true);
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int vs = gg % kNVm, pb = gg & 1;
          mbar_wait(&sm.v_full[vs], (gg / kNVm) & 1);
          mbar_wait(&sm.p_full[pb], (gg >> 1) & 1);
          if (j == 0 && seg > 0) mbar_wait(&sm.o_free, (seg - 1) & 1);
          tc_fence_after();
          const uint32_t p_base = smem_u32(sm.p[pb]);
          const uint32_t v_base = smem_u32(sm.v[vs]);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t a = sdesc_sw128(p_base + kk * 32, 0, 1024);
            const uint64_t b = sdesc_sw128(v_base + kk * 2048, kChunkKV, 1024);
            mma_bf16(tmem + kColOm, a, b, idesc_pv, (j == 0 && kk == 0) ? 0u : 1u);
          }
          mma_commit(&sm.v_empty[vs]);
          mma_commit(&sm.p_empty[pb]);
        }
        g += n;
        ++seg;
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ------------------------------- softmax / correction / epilogue (w2-5)
    const int sub = warp & 3;
    const int r = sub * 32 + lane;               // query row = TMEM lane (M=128)
    const int jt = r / kHeads;  // query token of this row (head = r % 64)
    const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t p_row_off = (uint32_t)r * 128;
    SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
    int req, lo, hi, seg = 0, g = 0;
    bool whole;
    while (walk.next(req, lo, hi, whole)) {
      const int n = hi - lo;
      const int seq_len = __ldg(prm.seq_lens + req);
      const int limit = seq_len - (kMtp - 1 - jt);  // keys visible to this row: [0, limit)
      float m_used = -INFINITY, l_sum = 0.0f;
      for (int j = 0; j < n; ++j, ++g) {
        const int sb = g & 1, pb = g & 1;
        mbar_wait(&sm.s_full[sb], (g >> 1) & 1);
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld32(t_row + kColSm + sb * 64, sr);
        tmem_ld32(t_row + kColSm + sb * 64 + 32, sr + 32);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_empty[sb]);

        const int tok0 = (lo + j) * kPage;
        const int nvalid = min(kPage, limit - tok0);
        float s[64];
        float tmax = -INFINITY;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          s[i] = (i < nvalid) ? __uint_as_float(sr[i]) * prm.scale_log2 : -INFINITY;
          tmax = fmaxf(tmax, s[i]);
        }
        const bool need = tmax > m_used + kRescaleM;
        float alpha = 1.0f;
        if (need) {
          alpha = fast_exp2(m_used - tmax);
          m_used = tmax;
        }
        l_sum *= alpha;
        const float mref = m_used == -INFINITY ? 0.0f : m_used;  // row with no visible key yet
        uint32_t pk[32];
        float psum = 0.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float p0 = fast_exp2(s[2 * i] - mref);
          const float p1 = fast_exp2(s[2 * i + 1] - mref);
          psum += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
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
          for (int c = 0; c < 8; ++c) {
            uint32_t o[32];
            tmem_ld32(t_row + kColOm + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
            tmem_st32(t_row + kColOm + c * 32, o);
          }
          tmem_wait_st();
        }
        const int nvalid_page = min(kPage, seq_len - tok0);
        if (nvalid_page < kPage) {
          const int vs = g % kNVm;
          mbar_wait(&sm.v_full[vs], (g / kNVm) & 1);
          const int tid = (warp - 2) * 32 + lane;
          uint8_t* vt = sm.v[vs];
          for (int idx = tid; idx < (kPage - nvalid_page) * 4 * 8; idx += 128) {
            const int row = nvalid_page + idx / 32, chunk = (idx / 8) & 3, q16 = idx & 7;
            *reinterpret_cast<uint4*>(vt + chunk * kChunkKV + row * 128 + q16 * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        {
          const uint32_t pbase = smem_u32(sm.p[pb]) + p_row_off;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t addr = pbase + ((uint32_t)(c ^ (r & 7)) << 4);
            st_shared_v4(addr, pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[pb]);
      }
      // ---------------- epilogue of this segment: O / l -> global
      const int gl = g - 1;
      mbar_wait(&sm.p_empty[gl & 1], (gl >> 1) & 1);
      tc_fence_after();
      const bool empty_row = !(l_sum > 0.0f);
      const float inv_l = empty_row ? 0.0f : 1.0f / l_sum;
      const int slot = req + cta;
      __nv_bfloat16* base = whole ? prm.out : reinterpret_cast<__nv_bfloat16*>(prm.part_o);
      const size_t orow = whole ? (size_t)req * kRowsM + r : (size_t)slot * kRowsM + r;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t o[32];
        tmem_ld32(t_row + kColOm + c * 32, o);
        tmem_wait_ld();
        uint4* dst = reinterpret_cast<uint4*>(base + orow * kDim + c * 32);
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
      const float lse2 = empty_row ? -INFINITY : m_used + __log2f(l_sum);
      if (whole) {
        if (prm.lse) prm.lse[(size_t)req * kRowsM + r] = lse2 * 0.69314718055994531f;
      } else {
        prm.part_lse[(size_t)slot * kRowsM + r] = lse2;
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
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace mfa

size_t mfa_decode_mtp_workspace_bytes(int batch, int num_sms) {
  const size_t slots = (size_t)batch + num_sms;
  size_t b = align_up((size_t)(batch + 1) * sizeof(int32_t), 256);
  b += align_up(slots * mfa::kRowsM * mfa::kDim * sizeof(float), 256);
  b += align_up(slots * mfa::kRowsM * sizeof(float), 256);
  return b;
}

cudaError_t mfa_decode_mtp_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream) {
  using namespace mfa;
  const int G = ctx.num_sms;
  if (a.batch > kMaxBatchMtp) return cudaErrorInvalidValue;
  uint8_t* ws = static_cast<uint8_t*>(a.workspace);
  Params prm{};
  prm.block_table = a.block_table;
  prm.seq_lens = a.seq_lens;
  ws += align_up((size_t)(a.batch + 1) * sizeof(int32_t), 256);
  const size_t slots = (size_t)a.batch + G;
  prm.part_o = reinterpret_cast<float*>(ws);
  ws += align_up(slots * kRowsM * kDim * sizeof(float), 256);
  prm.part_lse = reinterpret_cast<float*>(ws);
  prm.out = static_cast<__nv_bfloat16*>(a.out);
  prm.lse = a.lse;
  prm.sync = ctx.counters + kCounterSlots / 2;
  prm.seg_cost = kSegCost;
  prm.batch = a.batch;
  prm.max_pages = a.max_pages;
  prm.scale_log2 = a.softmax_scale * 1.4426950408889634f;
  prm.rows = kRowsM;

  CUtensorMap tq, tk, tv;
  {
    const uint64_t dims[2] = {(uint64_t)kDim, (uint64_t)a.batch * kRowsM};
    const uint64_t strides[1] = {kDim * 2};
    const uint32_t box[2] = {64, (uint32_t)kRowsM};
    if (!encode_tma(ctx, &tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.q), dims, strides, box,
                    CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {(uint64_t)kDim, (uint64_t)kPage, (uint64_t)a.num_pages};
    const uint64_t strides[2] = {kDim * 2, (uint64_t)kPage * kDim * 2};
    const uint32_t box[3] = {64, 64, 1};
    if (!encode_tma(ctx, &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.k_cache), dims, strides,
                    box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    if (!encode_tma(ctx, &tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.v_cache), dims, strides,
                    box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  const size_t smem = sizeof(SmemM) + 1024 + (size_t)(a.batch + 1) * sizeof(int32_t);
  if (const cudaError_t ea = ensure_smem(mfa_decode_mtp_kernel, sizeof(SmemM) + 1024 + (kMaxBatchMtp + 1) * sizeof(int32_t));
      ea != cudaSuccess)
    return ea;
  cudaError_t e = launch_k(ctx.pdl, mfa_decode_mtp_kernel, dim3(G), dim3(kThreadsM), smem, stream, tq, tk, tv, prm);
  if (e != cudaSuccess) return e;
  return mfa_combine_launch(ctx.pdl, prm, G, stream);
}

}  // namespace afdk
