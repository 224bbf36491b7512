// mfa_common.cuh — pieces shared by the bf16 (mfa_decode.cu) and e4m3
// (mfa_decode_fp8.cu) MFA decode kernels: work split, segment walker, the
// split-KV partial layout consumed by K3 (mfa_combine_kernel).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace afdk {
namespace mfa {

constexpr int kHeads = 64;
constexpr int kDim = 256;
constexpr int kPage = 64;  // tokens per KV page == one tile
#ifndef AFDK_MFA_BF16_PART
#define AFDK_MFA_BF16_PART 1
#endif

constexpr int kMaxBatch = 2048;  // prefix of work units per request lives in smem

// Work split: request r is kSegCost + pages_r units (0 when empty), and CTA c
// of G takes the contiguous unit range [cU/G, (c+1)U/G).  The kSegCost units
// at the head of each request carry no page: they charge a CTA that starts a
// new request segment for its extra Q load, O epilogue and split partial
// (~2-3 pages of streaming time measured per extra segment), so CTAs that
// straddle a request boundary get fewer pages and all CTAs end together.
#ifndef AFDK_MFA_SEG_COST
#define AFDK_MFA_SEG_COST 3
#endif
constexpr int kSegCost = AFDK_MFA_SEG_COST;

__device__ __forceinline__ int request_pages(int seq_len) { return (max(seq_len, 0) + kPage - 1) / kPage; }
__device__ __forceinline__ int request_units(int seq_len, int seg_cost) {
  const int pg = request_pages(seq_len);
  return pg > 0 ? pg + seg_cost : 0;
}


#ifdef AFDK_MFA_TIMES
// diagnostic build: launch timeline over back-to-back launches, one record of
// 8 stamps per launch (%globaltimer, ns): K2 {first entry, first / last PDL
// release, last end}, K3 {first entry, last wait done, last exit}.  Launch
// index = arrival count / grid size.  One copy per translation unit (static).
constexpr int kTlLaunches = 64;
static __device__ unsigned long long g_tl[kTlLaunches * 8];
static __device__ unsigned int g_tl_arrive[2];
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int tl_launch(int which, unsigned grid) {
  return (int)(atomicAdd(&g_tl_arrive[which], 1u) / grid) % kTlLaunches;
}
__device__ __forceinline__ void tl_min(int launch, int i) { atomicMin(&g_tl[launch * 8 + i], tl_now()); }
__device__ __forceinline__ void tl_max(int launch, int i) { atomicMax(&g_tl[launch * 8 + i], tl_now()); }
#endif

struct Params {
  const int32_t* block_table;  // [B, max_pages]
  const int32_t* seq_lens;     // [B]
  __nv_bfloat16* out;          // [B, 64, 256]
  float* lse;                  // [B, 64] natural log, optional
  float* part_o;               // [(B+G), 64, 256] split partials (bf16 when AFDK_MFA_BF16_PART)
  float* part_lse;             // [(B+G), 64] log2 domain
  int batch, max_pages;
  float scale_log2;            // softmax scale * log2(e)
  float k_scale, v_scale;      // e4m3 KV cache dequantisation scales (fp8 kernel)
  int rows;                    // query rows per request: 64 heads x mtp (0 = 64)
  int* sync;                   // [2][kMaxBatch] zeroed counters: split parts published / K3 CTAs done
  int seg_cost;                // page-less units charged per request segment (kSegCost; the e4m3
                               // kernel's pages cost half the time, so its charge is larger)
};

// A split part of request `req` is in memory: each of the 4 epilogue warps of
// the K2 CTA publishes its share (K3 waits for 4 x parts arrivals).
__device__ __forceinline__ void publish_part(int* sync, int req, int lane) {
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicAdd(sync + req, 1);
}

// Contiguous unit range of CTA c out of G over T total units.
__device__ __forceinline__ void cta_range(int c, int G, int T, int& lo, int& hi) {
  lo = (int)(((long long)c * T) / G);
  hi = (int)(((long long)(c + 1) * T) / G);
}

// First request whose unit range contains unit `t` (prefix is non-decreasing;
// empty requests are skipped because prefix[r+1] > t fails).
__device__ __forceinline__ int find_request(const int32_t* prefix, int B, int t) {
  int lo = 0, hi = B - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (prefix[mid + 1] > t) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Walks the segments (request, [lo,hi) local pages) of one CTA's unit range in order.
struct SegmentWalker {
  const int32_t* prefix;
  int B, end, r, pos, seg_cost;
  __device__ SegmentWalker(const int32_t* pf, int b, int start, int stop, int sc = kSegCost)
      : prefix(pf), B(b), end(stop), r(0), pos(start), seg_cost(sc) {
    if (start < stop) r = find_request(pf, b, start);
  }
  // returns false when the range is exhausted
  __device__ bool next(int& req, int& lo, int& hi, bool& whole) {
    while (pos < end) {
      while (prefix[r + 1] <= pos) ++r;
      const int p0 = prefix[r] + seg_cost, p1 = prefix[r + 1];  // the request's page units
      const int a = pos > p0 ? pos : p0;
      const int b = p1 < end ? p1 : end;
      pos = b;
      if (a < b) {
        req = r;
        lo = a - p0;
        hi = b - p0;
        whole = (a == p0) && (b == p1);
        return true;
      }
    }
    return false;
  }
};

// K / V ring prefill before griddepcontrol.wait: the first `cap` pages of
// this CTA's walk, in walk order, stopping at the first page a predecessor
// may write (a request's last page receives the appended token).  Returns how
// many pages were issued (the main loop skips them).
#ifndef AFDK_MFA_KV_PREFETCH
#define AFDK_MFA_KV_PREFETCH 1
#endif
template <class Load>
__device__ __forceinline__ int prefetch_pages(const int32_t* prefix, const Params& prm, int range_lo, int range_hi,
                                              int cap, Load&& load) {
  SegmentWalker walk(prefix, prm.batch, range_lo, range_hi, prm.seg_cost);
  int req, lo, hi, g = 0;
  bool whole;
  while (g < cap && walk.next(req, lo, hi, whole)) {
    const int last = request_pages(__ldg(prm.seq_lens + req)) - 1;
    for (int t = lo; t < hi && g < cap; ++t, ++g) {
      if (t >= last) return g;
      load(g, req, t);
    }
  }
  return g;
}

// work units per request -> exclusive prefix in smem (every CTA; B <= kMaxBatch).
// seq_lens is a caller input (no kernel of this library writes it), so this
// may run before griddepcontrol.wait.
template <int kThreads>
__device__ __forceinline__ void build_page_prefix(int32_t* prefix, const int32_t* seq_lens, int batch,
                                                  int seg_cost = kSegCost) {
  __shared__ int s_wsum[kThreads / 32];
  __shared__ int s_carry;
  constexpr int nw = kThreads / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { s_carry = 0; prefix[0] = 0; }
  for (int base = 0; base < batch; base += kThreads) {
    const int i = base + threadIdx.x;
    const int v = (i < batch) ? request_units(__ldg(seq_lens + i), seg_cost) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffff, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    int off = s_carry;
    for (int w = 0; w < warp; ++w) off += s_wsum[w];
    if (i < batch) prefix[i + 1] = off + x;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += s_wsum[w];
      s_carry += t;
    }
    __syncthreads();
  }
}

}  // namespace mfa

// K3 launch (defined in mfa_decode.cu)
cudaError_t mfa_combine_launch(bool pdl, const mfa::Params& prm, int G, cudaStream_t stream);

}  // namespace afdk
