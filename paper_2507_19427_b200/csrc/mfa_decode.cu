// mfa_decode.cu — K2/K3: Step-3 MFA decode attention core on sm_100a.
//
// Computes, for every decode request b and every one of the 64 query heads,
//   O[b,h,:] = softmax(scale * q[b,h,:] . K[b,:,:]^T) V[b,:,:]
// against ONE shared 256-dim K head and ONE shared V head held in a paged
// cache (accounting costmodel.cpp:26-44: 2*64*(256+256)*ctx FLOPs
// and 2*256*elt bytes per cached token).  Because the 64 heads share K/V, each
// 64-token page is read from HBM exactly once and consumed as a dense
// [64 heads x 64 tokens x 256] tensor-core contraction:
//
//   S  = Q[64x256] . K_page^T        tcgen05.mma M=64 N=64  K=256 -> TMEM
//   P  = exp2(S*scale*log2e - m)     4 softmax warps, one head per lane
//   O += P[64x64] . V_page[64x256]   tcgen05.mma M=64 N=256 K=64  -> TMEM
//
// Work distribution (flash-decoding, load balanced): the flattened
// (request, page) space is cut into one contiguous range per CTA
// (grid = #SMs, 1 CTA/SM).  A range that covers a whole request writes bf16
// O directly; otherwise it writes a normalised fp32 partial + log2-LSE into
// slot (request + cta), and mfa_combine (K3) merges the partials.  Each CTA
// derives the page prefix of the batch itself (no planning launch).
//
// Warp roles (256 threads):  w0 = Q/K TMA producer, w1 = QK^T MMA issuer +
// TMEM owner, w2..w5 = softmax / O-correction / epilogue (TMEM lanes 0-15 of
// each 32-lane sub-partition hold the M=64 accumulator rows; the 16x32bx2
// load shape hands columns [c,c+32) to lanes 0-15 and [c+32,c+64) to lanes
// 16-31, so every lane owns one head x 32 tokens), w6 = V TMA producer,
// w7 = P.V MMA issuer.  QK^T and P.V are issued by different
// threads so K slots recycle at QK^T completion whatever the softmax does.
#include <cuda.h>
#include <cuda_bf16.h>
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

constexpr int kTileBytes = kPage * kDim * 2;  // 32 KB (K or V of one page, bf16)
constexpr int kChunkBytes = 64 * 128;         // one 64-row x 128B swizzle panel
#ifndef AFDK_MFA_NK
#define AFDK_MFA_NK 2
#endif
#ifndef AFDK_MFA_NV
#define AFDK_MFA_NV 3
#endif
constexpr int kNK = AFDK_MFA_NK;              // K ring depth
constexpr int kNV = AFDK_MFA_NV;              // V ring depth
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColO = 0, kColS = 256;    // O: 256 cols, S: 2 x 64 cols
constexpr float kRescaleThresh = 8.0f;        // lazy O rescale (log2 units)

struct __align__(1024) Smem {
  uint8_t q[4 * kChunkBytes];       // 32 KB  Q of the current request
  uint8_t k[kNK][kTileBytes];       // 64 KB
  uint8_t v[kNV][kTileBytes];       // 96 KB
  uint8_t p[2][kHeads * kPage * 2];  // 16 KB  bf16 probabilities (K-major SW128)
  uint64_t q_full, q_empty;
  uint64_t k_full[kNK], k_empty[kNK];
  uint64_t v_full[kNV], v_empty[kNV];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full[2], p_empty[2];
  uint64_t o_free;
  uint32_t tmem_base;
};

#ifdef AFDK_MFA_TIMES
// diagnostic build: per-CTA %globaltimer stamps {after the PDL wait, first
// S consumed, last page of the last segment done, CTA end}
__device__ unsigned long long g_mfa_times[4 * 256];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define MFA_STAMP(i) g_mfa_times[4 * blockIdx.x + (i)] = gtimer()
#else
#define MFA_STAMP(i)
#endif

__global__ void __launch_bounds__(kThreads, 1)
mfa_decode_kernel(const __grid_constant__ CUtensorMap tm_q,
                  const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const Params prm) {
  extern __shared__ uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int32_t* prefix = reinterpret_cast<int32_t*>(&sm + 1);  // [B+1] after the Smem block
  // (seq_lens is a caller input: no kernel of this library writes it, so it may be read before griddep_wait)
#ifdef AFDK_MFA_TIMES
  __shared__ int s_tl;
  if (threadIdx.x == 0) { s_tl = tl_launch(0, gridDim.x); tl_min(s_tl, 0); }
#endif
  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  build_page_prefix<kThreads>(prefix, prm.seq_lens, prm.batch, prm.seg_cost);
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
    for (int i = 0; i < kNK; ++i) { mbar_init(&sm.k_full[i], 1); mbar_init(&sm.k_empty[i], 1); }
    for (int i = 0; i < kNV; ++i) { mbar_init(&sm.v_full[i], 1); mbar_init(&sm.v_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.s_empty[i], 4);
      mbar_init(&sm.p_full[i], 4);
      mbar_init(&sm.p_empty[i], 1);
    }
    mbar_init(&sm.o_free, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(&sm.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // q, the appended K/V row and the reused workspace belong to the
  // predecessors.  With AFDK_MFA_KV_PREFETCH the K / V producers first fill
  // their rings with pages the predecessors cannot touch (every page of a
  // request but its last, which holds the appended token) and only then wait,
  // so the ring fill overlaps the predecessor's tail; every other role waits here.
  const bool producer = AFDK_MFA_KV_PREFETCH && (warp == 0 || warp == 6);
  if (!producer) griddep_wait();
  griddep_launch();
  if (threadIdx.x == 0) MFA_STAMP(0);
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
        const int s = g % kNK, n = g / kNK;
        if (n > 0) mbar_wait(&sm.k_empty[s], (n & 1) ^ 1);
        mbar_expect_tx(&sm.k_full[s], kTileBytes);
        for (int c = 0; c < 4; ++c)
          tma_load_3d(sm.k[s] + c * kChunkBytes, &tm_k, &sm.k_full[s], c * 64, 0, page, pol_stream);
      };
      const int pre = AFDK_MFA_KV_PREFETCH ? prefetch_pages(prefix, prm, range_lo, range_hi, kNK, load_k) : 0;
      if (AFDK_MFA_KV_PREFETCH) griddep_wait();
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        if (seg > 0) mbar_wait(&sm.q_empty, (seg & 1) ^ 1);
        mbar_expect_tx(&sm.q_full, 4 * kChunkBytes);
        for (int c = 0; c < 4; ++c)
          tma_load_2d(sm.q + c * kChunkBytes, &tm_q, &sm.q_full, c * 64, req * kHeads, pol_keep);
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
        const int s = g % kNV, n = g / kNV;
        if (n > 0) mbar_wait(&sm.v_empty[s], (n & 1) ^ 1);
        mbar_expect_tx(&sm.v_full[s], kTileBytes);
        for (int c = 0; c < 4; ++c)
          tma_load_3d(sm.v[s] + c * kChunkBytes, &tm_v, &sm.v_full[s], c * 64, 0, page, pol_stream);
      };
      const int pre = AFDK_MFA_KV_PREFETCH ? prefetch_pages(prefix, prm, range_lo, range_hi, kNV, load_v) : 0;
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
    // Runs ahead of the softmax by the S double buffer only: K slots are
    // released as soon as their QK completes, independent of PV progress.
    if (lane == 0) {
      constexpr uint32_t idesc_qk = idesc_bf16(64, 64, false, false);
      const uint32_t q_base = smem_u32(sm.q);
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        mbar_wait(&sm.q_full, seg & 1);
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int ks = gg % kNK, sb = gg & 1;
          mbar_wait(&sm.k_full[ks], (gg / kNK) & 1);
          if (gg >= 2) mbar_wait(&sm.s_empty[sb], ((gg >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm.k[ks]);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t a = sdesc_sw128(q_base + c * kChunkBytes + kk * 32, 0, 1024);
              const uint64_t b = sdesc_sw128(k_base + c * kChunkBytes + kk * 32, 0, 1024);
              mma_bf16(tmem + kColS + sb * 64, a, b, idesc_qk, (c | kk) ? 1u : 0u);
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
      constexpr uint32_t idesc_pv = idesc_bf16(64, 256, false, true);
      SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
      int req, lo, hi, seg = 0, g = 0;
      bool whole;
      while (walk.next(req, lo, hi, whole)) {
        const int n = hi - lo;
        for (int j = 0; j < n; ++j) {
          const int gg = g + j;
          const int vs = gg % kNV, pb = gg & 1;
          mbar_wait(&sm.v_full[vs], (gg / kNV) & 1);
          mbar_wait(&sm.p_full[pb], (gg >> 1) & 1);
          if (j == 0 && seg > 0) mbar_wait(&sm.o_free, (seg - 1) & 1);
          tc_fence_after();
          const uint32_t p_base = smem_u32(sm.p[pb]);
          const uint32_t v_base = smem_u32(sm.v[vs]);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t a = sdesc_sw128(p_base + kk * 32, 0, 1024);
            const uint64_t b = sdesc_sw128(v_base + kk * 2048, kChunkBytes, 1024);
            mma_bf16(tmem + kColO, a, b, idesc_pv, (j == 0 && kk == 0) ? 0u : 1u);
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
    const int sub = warp & 3;                 // TMEM sub-partition of this warp
    const int half = lane >> 4;               // 16x32bx2 TMEM loads: lanes 16-31 read columns +32
    const int head = sub * 16 + (lane & 15);
    const uint32_t t_row = tmem + ((uint32_t)(sub * 32) << 16);
    const uint32_t p_row_off = (uint32_t)head * 128;  // K-major SW128: 128B per head row
    SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
    int req, lo, hi, seg = 0, g = 0;
    bool whole;
    while (walk.next(req, lo, hi, whole)) {
      const int n = hi - lo;
      const int seq_len = __ldg(prm.seq_lens + req);
      // lane (head, half) owns tokens [32*half, +32) of each page; l_sum is
      // this thread's share of the row sum (combined in the epilogue)
      float m_used = -INFINITY, l_sum = 0.0f;
      for (int j = 0; j < n; ++j, ++g) {
        const int sb = g & 1, pb = g & 1;
        mbar_wait(&sm.s_full[sb], (g >> 1) & 1);
        if (g == 0 && warp == 2 && lane == 0) MFA_STAMP(1);
        tc_fence_after();
        uint32_t sr[32];
        tmem_ld16x2_32(t_row + kColS + sb * 64, sr);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.s_empty[sb]);

        const int tok0 = (lo + j) * kPage;
        const int nvalid_page = min(kPage, seq_len - tok0);
        const int nvalid = nvalid_page - half * 32;
        float s[32];
        float tmax = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = (i < nvalid) ? __uint_as_float(sr[i]) * prm.scale_log2 : -INFINITY;
          tmax = fmaxf(tmax, s[i]);
        }
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffff, tmax, 16));
        const bool need = tmax > m_used + kRescaleThresh;
        float alpha = 1.0f;
        if (need) {
          alpha = fast_exp2(m_used - tmax);  // m_used=-inf -> 0
          m_used = tmax;
        }
        l_sum *= alpha;
        uint32_t pk[16];
        float psum = 0.0f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = fast_exp2(s[2 * i] - m_used);
          const float p1 = fast_exp2(s[2 * i + 1] - m_used);
          psum += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        l_sum += psum;

        // P slot (and, for a rescale, the O accumulator) must be quiescent
        if (g >= 2) mbar_wait(&sm.p_empty[pb], ((g >> 1) & 1) ^ 1);
        const bool warp_rescale = __any_sync(0xffffffff, need && j > 0);
        if (warp_rescale) {
          const int gp = g - 1;  // PV(g-1) must have landed in O
          mbar_wait(&sm.p_empty[gp & 1], (gp >> 1) & 1);
          tc_fence_after();
          const float a = need ? alpha : 1.0f;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld16x2_32(t_row + kColO + c * 64, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
            tmem_st16x2_32(t_row + kColO + c * 64, o);
          }
          tmem_wait_st();
        }
        // Last page of a request: zero V rows past seq_len so P=0 x garbage stays 0.
        if (nvalid_page < kPage) {
          const int vs = g % kNV;
          mbar_wait(&sm.v_full[vs], (g / kNV) & 1);
          const int tid = (warp - 2) * 32 + lane;  // 0..127
          uint8_t* vt = sm.v[vs];
          for (int idx = tid; idx < (kPage - nvalid_page) * 4 * 8; idx += 128) {
            const int row = nvalid_page + idx / 32, chunk = (idx / 8) & 3, q16 = idx & 7;
            *reinterpret_cast<uint4*>(vt + chunk * kChunkBytes + row * 128 + q16 * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        {
          const uint32_t pbase = smem_u32(sm.p[pb]) + p_row_off;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint32_t addr = pbase + ((uint32_t)((half * 4 + c) ^ (head & 7)) << 4);
            st_shared_v4(addr, pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.p_full[pb]);
      }
      // ---------------- epilogue of this segment: O / l -> global
      if (warp == 2 && lane == 0) MFA_STAMP(2);
      const int gl = g - 1;
      mbar_wait(&sm.p_empty[gl & 1], (gl >> 1) & 1);
      tc_fence_after();
      const float l_tot = l_sum + __shfl_xor_sync(0xffffffff, l_sum, 16);
      const float inv_l = 1.0f / l_tot;
      const int slot = req + cta;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tmem_ld16x2_32(t_row + kColO + c * 64, o);
        tmem_wait_ld();
        const int d0 = c * 64 + half * 32;
        if (whole || AFDK_MFA_BF16_PART) {
          __nv_bfloat16* base = whole ? prm.out : reinterpret_cast<__nv_bfloat16*>(prm.part_o);
          const size_t row = whole ? (size_t)req * kHeads + head : (size_t)slot * kHeads + head;
          uint4* dst = reinterpret_cast<uint4*>(base + row * kDim + d0);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(o[8 * q4 + 0]) * inv_l, __uint_as_float(o[8 * q4 + 1]) * inv_l);
            v.y = pack_bf16x2(__uint_as_float(o[8 * q4 + 2]) * inv_l, __uint_as_float(o[8 * q4 + 3]) * inv_l);
            v.z = pack_bf16x2(__uint_as_float(o[8 * q4 + 4]) * inv_l, __uint_as_float(o[8 * q4 + 5]) * inv_l);
            v.w = pack_bf16x2(__uint_as_float(o[8 * q4 + 6]) * inv_l, __uint_as_float(o[8 * q4 + 7]) * inv_l);
            dst[q4] = v;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(prm.part_o + ((size_t)slot * kHeads + head) * kDim + d0);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            dst[q4] = make_float4(__uint_as_float(o[4 * q4]) * inv_l, __uint_as_float(o[4 * q4 + 1]) * inv_l,
                                  __uint_as_float(o[4 * q4 + 2]) * inv_l, __uint_as_float(o[4 * q4 + 3]) * inv_l);
        }
      }
      if (half == 0) {
        const float lse2 = m_used + __log2f(l_tot);
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
  if (threadIdx.x == 0) MFA_STAMP(3);
#ifdef AFDK_MFA_TIMES
  if (threadIdx.x == 0) tl_max(s_tl, 3);
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

constexpr int kMaxSplit = 160;  // CTAs one request may span (>= #SMs + 1)
static_assert(kMaxSplit == kMfaMaxSplit, "afdk_create checks the SM count against kMfaMaxSplit");
static_assert(kMaxBatch == kMfaMaxBatch, "the C-ABI checks batch against kMfaMaxBatch");
// K3: merge the split partials of requests that spanned several CTAs (fixed
// CTA order => deterministic), zero-fill empty requests.  grid (B, R/16): 16
// rows per CTA, 32 threads per row, 8 dims per thread.
//
// K3 does not wait for the whole of K2: its CTAs become resident under PDL
// while K2 runs (every K2 CTA is resident by then, so spinning cannot starve
// it) and each waits only for its own request's parts (K2's publish_part
// counters), so merges overlap K2's tail.  The page prefix is recomputed from
// seq_lens (a caller input) because K2's copy is not final yet.  Every CTA
// ends with griddepcontrol.wait, so K3 completes only after K2 has, and the
// next kernel sees the whole-request outputs K2 wrote directly.
#ifndef AFDK_K3_BATCH
#define AFDK_K3_BATCH 1  // batched loads for 2-4 part merges (0: the generic loop, for A/B)
#endif
#ifndef AFDK_K3_SLEEP_MAX
#define AFDK_K3_SLEEP_MAX 1024  // K3's poll back-off cap (ns)
#endif
constexpr int kK3Rows = 16;     // query rows per K3 CTA
constexpr int kK3Threads = 512;  // 32 threads per row, 8 dims (16 B of bf16) per thread
__global__ void __launch_bounds__(kK3Threads) mfa_combine_kernel(const Params prm, int G) {
  __shared__ int s_slot[kMaxSplit];
  __shared__ float s_w[kK3Rows][kMaxSplit];
  __shared__ int s_n;
  __shared__ int s_red[2][kK3Threads / 32];
  griddep_launch();
#ifdef AFDK_MFA_TIMES
  __shared__ int s_tl;
  if (threadIdx.x == 0) { s_tl = tl_launch(1, gridDim.x * gridDim.y); tl_min(s_tl, 4); }
#endif
  const int R = prm.rows > 0 ? prm.rows : kHeads;  // query rows per request
  const int req = blockIdx.x;
  const int hl = threadIdx.x >> 5, head = blockIdx.y * kK3Rows + hl;
  const int d = (threadIdx.x & 31) * 8;
  {  // p0 = units before this request, T = all units
    int before = 0, all = 0;
    for (int i = threadIdx.x; i < prm.batch; i += blockDim.x) {
      const int pg = request_units(__ldg(prm.seq_lens + i), prm.seg_cost);
      all += pg;
      if (i < req) before += pg;
    }
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffff, before, o);
      all += __shfl_xor_sync(0xffffffff, all, o);
    }
    if ((threadIdx.x & 31) == 0) { s_red[0][threadIdx.x >> 5] = before; s_red[1][threadIdx.x >> 5] = all; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int p0 = 0, T = 0;
    for (int w = 0; w < kK3Threads / 32; ++w) { p0 += s_red[0][w]; T += s_red[1][w]; }
    const int p1 = p0 + request_units(__ldg(prm.seq_lens + req), prm.seg_cost);
    p0 += prm.seg_cost;  // the request's page units: [p0, p1)
    int n = 0;
    if (p1 > p0) {
      int c = (int)(((long long)p0 * G) / T);
      while (c > 0 && (((long long)c * T) / G) > p0) --c;
      while ((((long long)(c + 1) * T) / G) <= p0) ++c;
      for (; c < G && n < kMaxSplit; ++c) {
        const int lo = (int)(((long long)c * T) / G), hi = (int)(((long long)(c + 1) * T) / G);
        if (lo >= p1) break;
        if (hi > lo) s_slot[n++] = req + c;
      }
    }
    s_n = n;
    if (n > 1) {  // wait until K2 has published all n parts (bounded: trap rather than hang)
      const int target = 4 * n;
      const int* cnt = prm.sync + req;
      unsigned ns = 128;
      long long spins = 0;
      while (ld_acquire_gpu(cnt) < target) {
        __nanosleep(ns);
        if (ns < AFDK_K3_SLEEP_MAX) ns <<= 1;
        if (++spins > (1ll << 24)) __trap();
      }
    }
#ifdef AFDK_MFA_TIMES
    tl_max(s_tl, 5);
#endif
  }
  __syncthreads();
  const int n = s_n;
  __nv_bfloat16* out = prm.out + ((size_t)req * R + head) * kDim + d;
  const bool lse_lane = prm.lse && (threadIdx.x & 31) == 0;
  if (n == 0) {  // empty request
    *reinterpret_cast<uint4*>(out) = make_uint4(0, 0, 0, 0);
    if (lse_lane) prm.lse[(size_t)req * R + head] = -INFINITY;
#if AFDK_MFA_BF16_PART && AFDK_K3_BATCH
  } else if (n > 1 && n <= 4) {
    // the common split (2-4 parts): every part's LSE and 8-dim slice loaded in
    // one batch, so the merge after the last publish is one L2 round trip
    float l[4];
    uint4 raw[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < n) {
        const size_t row = (size_t)s_slot[k] * R + head;
        l[k] = __ldcg(prm.part_lse + row);
        raw[k] = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(prm.part_o) +
                                                      row * kDim + d));
      }
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (k < n) m = fmaxf(m, l[k]);
    if (m == -INFINITY) {  // a causal MTP row that sees no token in any part
      *reinterpret_cast<uint4*>(out) = make_uint4(0, 0, 0, 0);
      if (lse_lane) prm.lse[(size_t)req * R + head] = -INFINITY;
    } else {
      float wsum = 0.0f;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k >= n) break;
        const float w = exp2f(l[k] - m);
        wsum += w;
        const uint32_t wv[4] = {raw[k].x, raw[k].y, raw[k].z, raw[k].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[j]));
          acc[2 * j] += w * f.x;
          acc[2 * j + 1] += w * f.y;
        }
      }
      const float inv = 1.0f / wsum;
      uint4 o;
      o.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
      o.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
      o.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
      o.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
      *reinterpret_cast<uint4*>(out) = o;
      if (lse_lane) prm.lse[(size_t)req * R + head] = (m + __log2f(wsum)) * 0.69314718055994531f;
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(prm.sync + kMaxBatch + req, 1) == (int)gridDim.y - 1) {
      prm.sync[req] = 0;
      prm.sync[kMaxBatch + req] = 0;
    }
#endif
  } else if (n > 1) {
    for (int i = threadIdx.x; i < kK3Rows * n; i += blockDim.x)
      s_w[i / n][i % n] = __ldcg(prm.part_lse + (size_t)s_slot[i % n] * R + blockIdx.y * kK3Rows + i / n);
    __syncthreads();
    float m = -INFINITY;
    for (int k = 0; k < n; ++k) m = fmaxf(m, s_w[hl][k]);
    if (m == -INFINITY) {  // a causal MTP row that sees no token in any part
      *reinterpret_cast<uint4*>(out) = make_uint4(0, 0, 0, 0);
      if (lse_lane) prm.lse[(size_t)req * R + head] = -INFINITY;
    } else {
      float wsum = 0.0f;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int k = 0; k < n; ++k) {
        const float w = exp2f(s_w[hl][k] - m);
        wsum += w;
#if AFDK_MFA_BF16_PART
        const uint4 raw = __ldcg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(prm.part_o) +
                                                                ((size_t)s_slot[k] * R + head) * kDim + d));
        const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv[j]));
          acc[2 * j] += w * f.x;
          acc[2 * j + 1] += w * f.y;
        }
#else
        const float4* src = reinterpret_cast<const float4*>(prm.part_o + ((size_t)s_slot[k] * R + head) * kDim + d);
        const float4 a = __ldcg(src), b = __ldcg(src + 1);
        acc[0] += w * a.x; acc[1] += w * a.y; acc[2] += w * a.z; acc[3] += w * a.w;
        acc[4] += w * b.x; acc[5] += w * b.y; acc[6] += w * b.z; acc[7] += w * b.w;
#endif
      }
      const float inv = 1.0f / wsum;
      uint4 o;
      o.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
      o.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
      o.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
      o.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
      *reinterpret_cast<uint4*>(out) = o;
      if (lse_lane) prm.lse[(size_t)req * R + head] = (m + __log2f(wsum)) * 0.69314718055994531f;
    }
    // the last of this request's gridDim.y CTAs re-arms both counters
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(prm.sync + kMaxBatch + req, 1) == (int)gridDim.y - 1) {
      prm.sync[req] = 0;
      prm.sync[kMaxBatch + req] = 0;
    }
  }
#ifdef AFDK_MFA_TIMES
  if (threadIdx.x == 0) tl_max(s_tl, 6);
#endif
  griddep_wait();
}

}  // namespace mfa

#ifdef AFDK_MFA_TIMES
extern "C" void afdk_debug_mfa_times(unsigned long long* host) {
  cudaMemcpyFromSymbol(host, mfa::g_mfa_times, sizeof(mfa::g_mfa_times));
}
// timeline of the bf16 K2 + K3 (host: kTlLaunches x 8); reset = re-arm before a run
extern "C" void afdk_debug_mfa_tl(unsigned long long* host, int reset) {
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

// ------------------------------------------------------------------ host side
size_t mfa_decode_workspace_bytes(int batch, int num_sms) {
  const size_t slots = (size_t)batch + num_sms;
  size_t b = align_up((size_t)(batch + 1) * sizeof(int32_t), 256);     // prefix
  b += align_up(slots * mfa::kHeads * mfa::kDim * sizeof(float), 256);  // part_o
  b += align_up(slots * mfa::kHeads * sizeof(float), 256);              // part_lse
  return b;
}

cudaError_t mfa_decode_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream) {
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
  static const int seg_cost = [] { const char* e = std::getenv("AFDK_MFA_SEG_COST_RT"); return e ? std::atoi(e) : kSegCost; }();
  prm.seg_cost = seg_cost;
  prm.batch = a.batch;
  prm.max_pages = a.max_pages;
  prm.scale_log2 = a.softmax_scale * 1.4426950408889634f;

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
    const uint64_t strides[2] = {kDim * 2, (uint64_t)kPage * kDim * 2};
    const uint32_t box[3] = {64, 64, 1};
    if (!encode_tma(ctx, &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.k_cache), dims, strides,
                    box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    if (!encode_tma(ctx, &tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.v_cache), dims, strides,
                    box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  const size_t smem = sizeof(Smem) + 1024 + (size_t)(a.batch + 1) * sizeof(int32_t);
  if (const cudaError_t ea = ensure_smem(mfa_decode_kernel, sizeof(Smem) + 1024 + (kMaxBatch + 1) * sizeof(int32_t));
      ea != cudaSuccess)
    return ea;
  cudaError_t e = launch_k(ctx.pdl, mfa_decode_kernel, dim3(G), dim3(kThreads), smem, stream, tq, tk, tv, prm);
  if (e != cudaSuccess) return e;
  return mfa_combine_launch(ctx.pdl, prm, G, stream);
}

cudaError_t mfa_combine_launch(bool pdl, const mfa::Params& prm, int G, cudaStream_t stream) {
  const int R = prm.rows > 0 ? prm.rows : mfa::kHeads;
  const cudaError_t e = launch_k(pdl, mfa::mfa_combine_kernel, dim3(prm.batch, R / mfa::kK3Rows),
                                 dim3(mfa::kK3Threads), 0, stream, prm, G);
  // K2 has already published its parts: re-arm the counters K3 would have reset
  if (e != cudaSuccess) cudaMemsetAsync(prm.sync, 0, 2 * mfa::kMaxBatch * sizeof(int), stream);
  return e;
}

}  // namespace afdk
