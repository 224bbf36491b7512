// moe_route.cu — K5 router + FP8 dispatch quantization, K6 permutation,
// dispatch gather and K9 combine for the Step-3 MoE FFN.
//
// Semantics (restated in oracle/afd_oracle.c, pinned by tests/golden/router.npz):
//   router   logits = h . Wg^T (fp32, fixed summation order), softmax over E,
//            top-k by logit with ties to the lower expert id, weights =
//            softmax probabilities of the selected experts (vllm FusedMoE,
//            renormalize = norm_expert_weight = False); runs on the ATTENTION
//            side.
//   quant    per token, per 128 contiguous features: scale = max(amax,1e-10)/448,
//            q = e4m3_rn_satfinite(x / scale) — the FP8 dispatch payload and its
//            scale factors.
//   permute  expert-major, then token, then k (stable): the "expert
//            distribution" metadata that organises the FFN input.
//   combine  out[t] = sum_j w[t,j] * y[slot(t,j)] + y_shared[t]  -> bf16
//            (BF16 return).
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "afdk_internal.h"
#include "linear.cuh"
#include "moe.cuh"
#include "sm100.cuh"

namespace afdk {
namespace moe {


__device__ __forceinline__ uint8_t to_e4m3(float v) {
  return (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3);
}

// ---------------------------------------------------------------- K5 router
// logits = h . gate^T runs on the tcgen05 stream-K linear kernel (linear.cu:
// gate rows on MMA M, up to 256 tokens on N, fp32 partials); this epilogue
// sums the partials in fixed segment order (deterministic; identical gate rows
// give identical logits), then per token (one warp, lanes own experts l and
// l+32): max-subtracted softmax, top-k by repeated warp argmax with ties to
// the lower expert id, weights = softmax[id] (optionally renormalised).
__global__ void __launch_bounds__(256) router_topk_kernel(const LinearPlan P, const float* __restrict__ part, int G,
                                                          RouterArgs a, int t_base) {
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;  // token within this chunk
  if (row >= P.n_out) return;  // tokens of this chunk (the GEMM's weight rows)
  const int tok = t_base + row;
  const int e0 = lane, e1 = lane + 32;
  // the GEMM ran with the tokens on the weight side (P.m_tok = E experts,
  // P.n_out = tokens): logit (token, e) is "row" e, "feature" token
  const float l0 = e0 < a.E ? tab.sum(P, part, e0, row) : -INFINITY;
  const float l1 = e1 < a.E ? tab.sum(P, part, e1, row) : -INFINITY;
  if (a.logits) {
    if (e0 < a.E) a.logits[(size_t)tok * a.E + e0] = l0;
    if (e1 < a.E) a.logits[(size_t)tok * a.E + e1] = l1;
  }
  float mx = fmaxf(l0, l1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffff, mx, o));
  float sum = (e0 < a.E ? expf(l0 - mx) : 0.0f) + (e1 < a.E ? expf(l1 - mx) : 0.0f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffff, sum, o);
  bool t0 = e0 >= a.E, t1 = e1 >= a.E;  // taken (or absent)
  float wk[kMaxTopK];
  int idk[kMaxTopK];
  float wsum = 0.0f;
  for (int j = 0; j < a.k; ++j) {
    // lane candidate: its larger untaken logit (lower id on ties)
    float bv = -INFINITY;
    int bi = 1 << 30;
    if (!t0) { bv = l0; bi = e0; }
    if (!t1 && (l1 > bv || bi == (1 << 30))) { bv = l1; bi = e1; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffff, bv, o);
      const int oi = __shfl_xor_sync(0xffffffff, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (bi == e0) t0 = true;
    if (bi == e1) t1 = true;
    idk[j] = bi;
    wk[j] = expf(bv - mx) / sum;
    wsum += wk[j];
  }
  if (lane == 0)
    for (int j = 0; j < a.k; ++j) {
      a.ids[(size_t)tok * a.k + j] = idk[j];
      a.weights[(size_t)tok * a.k + j] = a.renormalize ? wk[j] / wsum : wk[j];
    }
}

// FP8 dispatch payload (1x128 blocks): one warp per (token, block), 4 features per lane
__global__ void __launch_bounds__(256) router_quant_kernel(RouterArgs a) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int nb = a.H / 128;
  const int blk = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (blk >= a.T * nb) return;
  const int t = blk / nb, b = blk % nb;
  const __nv_bfloat16* src = a.h + (size_t)t * a.H + b * 128 + lane * 4;
  const uint2 raw = *reinterpret_cast<const uint2*>(src);
  const float2 f01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
  const float2 f23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
  float amax = fmaxf(fmaxf(fabsf(f01.x), fabsf(f01.y)), fmaxf(fabsf(f23.x), fabsf(f23.y)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffff, amax, o));
  const float sc = __fdiv_rn(fmaxf(amax, 1e-10f), 448.0f);
  const uint32_t q = (uint32_t)to_e4m3(__fdiv_rn(f01.x, sc)) | ((uint32_t)to_e4m3(__fdiv_rn(f01.y, sc)) << 8) |
                     ((uint32_t)to_e4m3(__fdiv_rn(f23.x, sc)) << 16) | ((uint32_t)to_e4m3(__fdiv_rn(f23.y, sc)) << 24);
  *reinterpret_cast<uint32_t*>(a.xq + (size_t)t * a.H + b * 128 + lane * 4) = q;
  if (lane == 0) a.xs[(size_t)t * nb + b] = sc;
}

// ------------------------------------------------------------- K6 permute
// One CTA of 32 warps; warp w owns the contiguous entry segment w of the
// [T*k] routing.  Pass 1 counts each expert per segment (__match_any_sync
// groups equal experts within a 32-entry batch); the per-(segment, expert)
// counts are scanned into slot bases in expert-major, segment-minor order;
// pass 2 repeats the batches and places every entry at base + running count
// + rank within its batch.  Segments are in entry order, so the result is the
// stable (expert, token, j) permutation exactly.  Also emits the grouped-GEMM
// work list: chunks of <= a.chunk rows per group, groups 0..E-1 routed (rows
// at offsets[e]) and group E = shared expert over its token range.
__global__ void __launch_bounds__(1024) permute_kernel(PermuteArgs a) {
  extern __shared__ uint8_t s_ids[];
  __shared__ int s_cnt[32][kMaxExperts];
  __shared__ int s_tot[kMaxExperts], s_off[kMaxExperts + 1];
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int n = a.T * a.k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s_ids[i] = (uint8_t)a.ids[i];
  for (int i = threadIdx.x; i < 32 * kMaxExperts; i += blockDim.x) (&s_cnt[0][0])[i] = 0;
  if (a.sched)
    for (int i = threadIdx.x; i < a.sched_len; i += blockDim.x) a.sched[i] = 0;
  __syncthreads();
  const int seg = (n + 31) / 32;
  const int lo = warp * seg, hi = min(n, lo + seg);
  const unsigned lt = (1u << lane) - 1u;
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const bool valid = i < hi;
    const int e = valid ? s_ids[i] : 255;
    const unsigned m = __match_any_sync(0xffffffff, e);
    if (valid && (m & lt) == 0) s_cnt[warp][e] += __popc(m);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < a.E) {
    const int e = threadIdx.x;
    int run = 0;
    for (int w = 0; w < 32; ++w) { const int c = s_cnt[w][e]; s_cnt[w][e] = run; run += c; }
    s_tot[e] = run;
  }
  __syncthreads();
  if (warp == 0) {
    // expert offsets and the work list, one lane per expert (E <= 64): warp
    // scans instead of a serial loop (the CTA waits on this section)
    const int e0 = lane, e1 = lane + 32;
    const int c0 = e0 < a.E ? s_tot[e0] : 0, c1 = e1 < a.E ? s_tot[e1] : 0;
    int x0 = c0, x1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffff, x0, o), y1 = __shfl_up_sync(0xffffffff, x1, o);
      if (lane >= o) { x0 += y0; x1 += y1; }
    }
    const int tot0 = __shfl_sync(0xffffffff, x0, 31), tot1 = __shfl_sync(0xffffffff, x1, 31);
    if (e0 < a.E) { s_off[e0] = x0 - c0; a.offsets[e0] = x0 - c0; }
    if (e1 < a.E) { s_off[e1] = tot0 + x1 - c1; a.offsets[e1] = tot0 + x1 - c1; }
    if (lane == 0) { s_off[a.E] = tot0 + tot1; a.offsets[a.E] = tot0 + tot1; }
    // items per group: ceil(rows/chunk) near-equal pieces (multiples of 32 rows)
    auto items = [&](int rows) { return (rows + a.chunk - 1) / a.chunk; };
    const bool l0 = e0 < a.E && e0 >= a.expert_lo && e0 < a.expert_hi;
    const bool l1 = e1 < a.E && e1 >= a.expert_lo && e1 < a.expert_hi;
    const int n0 = l0 ? items(c0) : 0, n1 = l1 ? items(c1) : 0;
    int y0 = n0, y1 = n1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int z0 = __shfl_up_sync(0xffffffff, y0, o), z1 = __shfl_up_sync(0xffffffff, y1, o);
      if (lane >= o) { y0 += z0; y1 += z1; }
    }
    const int w0 = __shfl_sync(0xffffffff, y0, 31), w1 = __shfl_sync(0xffffffff, y1, 31);
    auto emit = [&](int g, int group, int row0, int rows) {
      const int n_it = items(rows);
      const int per = n_it > 0 ? ((rows + n_it - 1) / n_it + 31) & ~31 : 0;
      const int first = g;
      for (int r = 0; r < rows; r += per, ++g) {
        a.work[g].group = group;
        a.work[g].row0 = row0 + r;
        a.work[g].rows = min(per, rows - r);
        a.work[g].xrow0 = row0 + r;
        a.work[g].gfirst = first;
        a.work[g].gcnt = n_it;
      }
    };
    if (l0) emit(y0 - n0, e0, x0 - c0, c0);
    if (l1) emit(w0 + y1 - n1, e1, tot0 + x1 - c1, c1);
    if (lane == 0) {
      int g = w0 + w1;
      if (a.shared_local) {
        const int rows = a.shared_hi - a.shared_lo;
        emit(g, a.E, n + a.shared_lo, rows);
        g += items(rows);
      }
      *a.n_work = g;
    }
  }
  __syncthreads();
  if (threadIdx.x < a.E)
    for (int w = 0; w < 32; ++w) s_cnt[w][threadIdx.x] += s_off[threadIdx.x];
  __syncthreads();
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const bool valid = i < hi;
    const int e = valid ? s_ids[i] : 255;
    const unsigned m = __match_any_sync(0xffffffff, e);
    if (valid) {
      const int pos = s_cnt[warp][e] + __popc(m & lt);
      a.perm[pos] = i;
      a.inv[i] = pos;
    }
    __syncwarp();
    if (valid && (m & lt) == 0) s_cnt[warp][e] += __popc(m);
    __syncwarp();
  }
}

// ---------------------------------------------------------- dispatch gather
// rows [0, T*k): routed copies in permuted order; rows [T*k, T*k + T): the
// shared expert's tokens in order.  Scales are written transposed
// [H/128][rows] so the GEMM fetches one k-block's row scales with a TMA box.
__global__ void __launch_bounds__(256) gather_kernel(GatherArgs a) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int s = blockIdx.x;
  const int n_routed = a.T * a.k;
  const int src = (s < n_routed) ? __ldg(a.perm + s) / a.k : s - n_routed;
  const uint4* in = reinterpret_cast<const uint4*>(a.xq + (size_t)src * a.H);
  uint4* out = reinterpret_cast<uint4*>(a.xp + (size_t)s * a.H);
  for (int i = threadIdx.x; i < a.H / 16; i += blockDim.x) out[i] = __ldg(in + i);
  if (a.xs) {
    const int nb = a.H / 128;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a.xs_t[(size_t)b * a.rows_pad + s] = __ldg(a.xs + (size_t)src * nb + b);
  } else if (a.xsf) {
    const int nb = a.H / 32;  // MXFP8: copy the row's UE8M0 scales
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a.xsf_p[(size_t)s * nb + b] = __ldg(a.xsf + (size_t)src * nb + b);
  }
}

// ------------------------------------------------------- MXFP8 quantisation
// One thread per 32-element block: e = smallest exponent with amax <= 448*2^e
// (exact, from amax's exponent/mantissa bits), q = e4m3(x * 2^-e).
__device__ __forceinline__ int mx_exponent(float amax) {
  const uint32_t u = __float_as_uint(amax);
  const int E = (int)((u >> 23) & 0xff);
  if (!(amax > 0.0f) || E == 0) return -127;
  const int e = ((u & 0x7fffffu) <= 6291456u) ? E - 135 : E - 134;
  return max(-127, min(127, e));
}
__device__ __forceinline__ float mx_inv_scale(int e) {
  return e < 127 ? __uint_as_float((uint32_t)(127 - e) << 23) : __uint_as_float(1u << 22);
}

__global__ void __launch_bounds__(256) quant_mx_kernel(QuantMxArgs a) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int nb = a.H / 32;
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk >= a.T * nb) return;
  const uint4* src = reinterpret_cast<const uint4*>(a.x + (size_t)blk * 32);
  float v[32];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 w = __ldg(src + c);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[c * 8 + 2 * j] = __uint_as_float(ws[j] << 16);
      v[c * 8 + 2 * j + 1] = __uint_as_float(ws[j] & 0xffff0000u);
    }
  }
  float amax = 0.0f;
#pragma unroll
  for (int j = 0; j < 32; ++j) amax = fmaxf(amax, fabsf(v[j]));
  const int e = mx_exponent(amax);
  const float inv = mx_inv_scale(e);
  uint32_t out[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      w |= (uint32_t)__nv_cvt_float_to_fp8(v[4 * j + b] * inv, __NV_SATFINITE, __NV_E4M3) << (8 * b);
    out[j] = w;
  }
  uint4* dst = reinterpret_cast<uint4*>(a.q + (size_t)blk * 32);
  dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
  dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
  a.sf[blk] = (uint8_t)(e + 127);
}

// --------------------------------------------------------------- K9 combine
// out[t] = sum_j w[t,j] y[inv[t,j]] (local experts only) + y[shared row of t]
__global__ void __launch_bounds__(256) combine_kernel(CombineArgs a) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int t = blockIdx.x;
  const int n_routed = a.T * a.k;
  float w[kMaxTopK];
  int slot[kMaxTopK];
  for (int j = 0; j < a.k; ++j) {
    const int e = __ldg(a.ids + (size_t)t * a.k + j);
    const bool local = e >= a.expert_lo && e < a.expert_hi;
    w[j] = local ? __ldg(a.weights + (size_t)t * a.k + j) : 0.0f;
    slot[j] = local ? __ldg(a.inv + (size_t)t * a.k + j) : -1;
  }
  const bool sh = a.shared_local && t >= a.shared_lo && t < a.shared_hi;
  const size_t sh_row = (size_t)n_routed + t;
  __nv_bfloat16* orow = a.dst ? reinterpret_cast<__nv_bfloat16*>(__ldg(a.dst + t / a.rows_per_dst)) +
                                    (size_t)(t % a.rows_per_dst) * a.H
                              : a.out + (size_t)t * a.H;
  for (int f = threadIdx.x * 4; f < a.H; f += blockDim.x * 4) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (sh) acc = __ldcg(reinterpret_cast<const float4*>(a.y + sh_row * a.H + f));
    for (int j = 0; j < a.k; ++j) {
      if (slot[j] < 0) continue;
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.y + (size_t)slot[j] * a.H + f));
      acc.x = fmaf(w[j], v.x, acc.x);
      acc.y = fmaf(w[j], v.y, acc.y);
      acc.z = fmaf(w[j], v.z, acc.z);
      acc.w = fmaf(w[j], v.w, acc.w);
    }
    __nv_bfloat162 o0 = __floats2bfloat162_rn(acc.x, acc.y), o1 = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&o0);
    o.y = *reinterpret_cast<uint32_t*>(&o1);
    *reinterpret_cast<uint2*>(orow + f) = o;
  }
}

}  // namespace moe

// Router GEMM with the roles of linear.cu swapped: the token rows stream as
// the 128-row M panels and the E <= 64 gate rows are the MMA's N, so the
// tiles are token blocks (ceil(T/128) of them, spread over up to 15 CTAs
// each) and the split partials are E columns wide.  With the gate rows as M
// (one 128-row tile for all experts) the k-loop of all tokens ran on at most
// 15 CTAs (kMaxSegs) in 256-token chunks: ~20-40 us at the AFD micro-batch.
constexpr int kRouterChunk = 8192;  // tokens per GEMM (tiles <= kMaxTiles)

size_t router_workspace_bytes(int H, int E, int num_sms) {
  return linear_workspace_bytes(make_linear_plan(E, kRouterChunk, H), num_sms);
}

cudaError_t router_launch(Ctx& ctx, const moe::RouterArgs& a, void* ws, cudaStream_t stream) {
  float* part = static_cast<float*>(ws);
  for (int c0 = 0; c0 < a.T; c0 += kRouterChunk) {
    const int m = min(kRouterChunk, a.T - c0);
    const LinearPlan p = make_linear_plan(a.E, m, a.H);
    // the token rows (the GEMM's weight side) are the predecessor's output: w_dep
    cudaError_t e = linear_bf16_launch(ctx, p, a.gate_w, a.h + (size_t)c0 * a.H, part, stream, true);
    if (e == cudaSuccess)
      e = launch_k(ctx.pdl, moe::router_topk_kernel, dim3((m + 7) / 8), dim3(256), 0, stream, p, (const float*)part,
                   linear_grid(ctx, p), a, c0);
    if (e != cudaSuccess) return e;
  }
  if (!a.xq) return cudaSuccess;
  const int blocks = a.T * (a.H / 128);
  return launch_k(ctx.pdl, moe::router_quant_kernel, dim3((blocks + 7) / 8), dim3(256), 0, stream, a);
}

cudaError_t permute_launch(const moe::PermuteArgs& a, cudaStream_t stream, bool pdl) {
  return launch_k(pdl, moe::permute_kernel, dim3(1), dim3(1024), (size_t)a.T * a.k, stream, a);
}

cudaError_t gather_launch(const moe::GatherArgs& a, cudaStream_t stream, bool pdl) {
  return launch_k(pdl, moe::gather_kernel, dim3(a.T * a.k + a.T), dim3(256), 0, stream, a);
}

cudaError_t quant_mx_launch(const moe::QuantMxArgs& a, cudaStream_t stream, bool pdl) {
  const int n = a.T * (a.H / 32);
  return launch_k(pdl, moe::quant_mx_kernel, dim3((n + 255) / 256), dim3(256), 0, stream, a);
}

cudaError_t combine_launch(const moe::CombineArgs& a, cudaStream_t stream, bool pdl) {
  return launch_k(pdl, moe::combine_kernel, dim3(a.T), dim3(256), 0, stream, a);
}

}  // namespace afdk
