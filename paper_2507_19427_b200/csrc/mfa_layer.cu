// mfa_layer.cu — the attention-side Step-3 decode layer (K1 + K2/K3 + K4).
//
// x -> input RMSNorm -> [q_down|k|v] GEMM -> q RMSNorm -> q_up GEMM -> RoPE(q,k)
//   -> paged KV append -> MFA decode core -> o_proj GEMM + residual
//   -> post-attention RMSNorm (the FFN input that AFD dispatches)
// (vllm step3_text.py Step3TextAttention/DecoderLayer;
// projection shapes builtin_catalog.cpp:243-247).
//
// The GEMMs run on the stream-K tcgen05 kernel (linear.cu); everything that
// needs a whole row (RMSNorm, RoPE pairs, KV append, residual) is fused into
// the row epilogue that sums that GEMM's partials (lin::SlotTable).  Intermediates are
// stored in bf16 exactly where the oracle (orc_mfa_layer) rounds.
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "afdk_internal.h"
#include "linear.cuh"
#include "sm100.cuh"

namespace afdk {
namespace layer {

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

__device__ __forceinline__ float block_sum(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = (l < (int)(blockDim.x >> 5)) ? red[l] : 0.0f;
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffff, t, o);
  return t;
}

// xn = RMSNorm(x) * w, bf16 out (input_layernorm); dim % 4 == 0
__global__ void __launch_bounds__(1024) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ w,
                                                       __nv_bfloat16* __restrict__ out, int dim, float eps) {
  __shared__ float red[32];
  sm100::griddep_wait();
  sm100::griddep_launch();
  const size_t row = blockIdx.x;
  const __nv_bfloat16* xr = x + row * dim;
  float ss = 0.0f;
  for (int i = threadIdx.x * 4; i < dim; i += blockDim.x * 4) {
    const uint2 xb = *reinterpret_cast<const uint2*>(xr + i);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.y));
    ss += a.x * a.x + a.y * a.y + b.x * b.x + b.y * b.y;
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / dim + eps);
  for (int i = threadIdx.x * 4; i < dim; i += blockDim.x * 4) {
    const uint2 xb = *reinterpret_cast<const uint2*>(xr + i);
    const uint2 wb = *reinterpret_cast<const uint2*>(w + i);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.y));
    const float2 wa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.x));
    const float2 wc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.y));
    uint2 o;
    o.x = sm100::pack_bf16x2((a.x * inv) * wa.x, (a.y * inv) * wa.y);
    o.y = sm100::pack_bf16x2((b.x * inv) * wc.x, (b.y * inv) * wc.y);
    *reinterpret_cast<uint2*>(out + row * dim + i) = o;
  }
}

struct QkvEpi {
  int q_lora, head_dim, page, max_pages, n_out;
  float eps;
  const __nv_bfloat16* q_norm_w;
  __nv_bfloat16* qa;            // [B, q_lora]
  __nv_bfloat16* k_cache;       // [num_pages, page, head_dim]
  __nv_bfloat16* v_cache;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const double* inv_freq;       // [head_dim/2]
  float k_scale, v_scale;       // > 0: caches are e4m3, store e4m3(bf16(x) / scale)
};

__device__ __forceinline__ uint8_t kv_e4m3(float x, float scale) {
  return (uint8_t)__nv_cvt_float_to_fp8(__fdiv_rn(x, scale), __NV_SATFINITE, __NV_E4M3);
}

// y = [q_down|k|v] projection of one token row (fp32): q -> RMSNorm -> qa;
// k -> RoPE -> K cache slot of position seq_len-1; v -> V cache slot.
__global__ void __launch_bounds__(512) qkv_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                           int G, const QkvEpi e) {
  extern __shared__ float row_s[];  // n_out floats
  __shared__ float red[32];
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int row = blockIdx.x;
  float ss = 0.0f;
  for (int f = threadIdx.x; f < e.n_out; f += blockDim.x) {
    const float v = bf16r(tab.sum(P, part, row, f));
    row_s[f] = v;
    if (f < e.q_lora) ss += v * v;
  }
  ss = block_sum(ss, red);  // includes __syncthreads: row_s complete
  const float inv = rsqrtf(ss / e.q_lora + e.eps);
  for (int f = threadIdx.x; f < e.q_lora; f += blockDim.x)
    e.qa[(size_t)row * e.q_lora + f] = __float2bfloat16_rn((row_s[f] * inv) * __bfloat162float(e.q_norm_w[f]));
  const int pos = __ldg(e.seq_lens + row) - 1;
  if (pos < 0) return;
  const int pg = __ldg(e.block_table + (size_t)row * e.max_pages + pos / e.page);
  const size_t slot = ((size_t)pg * e.page + pos % e.page) * e.head_dim;
  const int half = e.head_dim / 2;
  const float* k = row_s + e.q_lora;
  const float* v = k + e.head_dim;
  const bool fp8 = e.k_scale > 0.0f;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    double sn, cs;
    sincos((double)pos * e.inv_freq[i], &sn, &cs);
    const float c = (float)cs, s = (float)sn;
    const float x1 = k[i], x2 = k[i + half];
    const __nv_bfloat16 k1 = __float2bfloat16_rn(x1 * c - x2 * s), k2 = __float2bfloat16_rn(x2 * c + x1 * s);
    if (fp8) {
      uint8_t* k8 = reinterpret_cast<uint8_t*>(e.k_cache);
      k8[slot + i] = kv_e4m3(__bfloat162float(k1), e.k_scale);
      k8[slot + i + half] = kv_e4m3(__bfloat162float(k2), e.k_scale);
    } else {
      e.k_cache[slot + i] = k1;
      e.k_cache[slot + i + half] = k2;
    }
  }
  for (int i = threadIdx.x; i < e.head_dim; i += blockDim.x) {
    if (fp8)
      reinterpret_cast<uint8_t*>(e.v_cache)[slot + i] = kv_e4m3(v[i], e.v_scale);
    else
      e.v_cache[slot + i] = __float2bfloat16_rn(v[i]);
  }
}

// y = q_up projection (fp32 [B, n_heads*head_dim]); per-head NeoX RoPE -> q bf16.
// grid (B, n_heads/8), 8 heads x head_dim/2 pairs per CTA.
__global__ void __launch_bounds__(1024) qup_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                            int G, int n_out, int head_dim,
                                                            const int32_t* __restrict__ seq_lens,
                                                            const double* __restrict__ inv_freq,
                                                            __nv_bfloat16* __restrict__ q) {
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int row = blockIdx.x;
  const int half = head_dim / 2;
  const int pos = max(__ldg(seq_lens + row) - 1, 0);
  const int idx = blockIdx.y * blockDim.x + threadIdx.x;  // pair index in the row
  if (idx >= n_out / 2) return;
  const int h = idx / half, i = idx % half;
  const int c1 = h * head_dim + i;
  const size_t f1 = (size_t)row * n_out + c1, f2 = f1 + half;
  const float x1 = bf16r(tab.sum(P, part, row, c1)), x2 = bf16r(tab.sum(P, part, row, c1 + half));
  double sn, cs;
  sincos((double)pos * inv_freq[i], &sn, &cs);
  const float c = (float)cs, s = (float)sn;
  q[f1] = __float2bfloat16_rn(x1 * c - x2 * s);
  q[f2] = __float2bfloat16_rn(x2 * c + x1 * s);
}

// y = o_proj (fp32); h_res = bf16(x + y); h_norm = RMSNorm(h_res) (post_attention_layernorm)
__global__ void __launch_bounds__(1024) o_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                          int G, int n, const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ w_post, float eps,
                                                          __nv_bfloat16* __restrict__ h_res,
                                                          __nv_bfloat16* __restrict__ h_norm) {
  extern __shared__ float row_s[];
  __shared__ float red[32];
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  sm100::griddep_wait();
  sm100::griddep_launch();
  const size_t row = blockIdx.x;
  float ss = 0.0f;
  for (int f = threadIdx.x * 4; f < n; f += blockDim.x * 4) {
    const float4 o = make_float4(tab.sum(P, part, (int)row, f), tab.sum(P, part, (int)row, f + 1),
                                 tab.sum(P, part, (int)row, f + 2), tab.sum(P, part, (int)row, f + 3));
    const uint2 xb = *reinterpret_cast<const uint2*>(x + row * n + f);
    const __nv_bfloat162 x01 = *reinterpret_cast<const __nv_bfloat162*>(&xb.x);
    const __nv_bfloat162 x23 = *reinterpret_cast<const __nv_bfloat162*>(&xb.y);
    const float r[4] = {bf16r(__low2float(x01) + o.x), bf16r(__high2float(x01) + o.y),
                        bf16r(__low2float(x23) + o.z), bf16r(__high2float(x23) + o.w)};
    uint2 ob;
    ob.x = sm100::pack_bf16x2(r[0], r[1]);
    ob.y = sm100::pack_bf16x2(r[2], r[3]);
    *reinterpret_cast<uint2*>(h_res + row * n + f) = ob;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      row_s[f + q] = r[q];
      ss += r[q] * r[q];
    }
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / n + eps);
  for (int f = threadIdx.x * 4; f < n; f += blockDim.x * 4) {
    const uint2 wb = *reinterpret_cast<const uint2*>(w_post + f);
    const __nv_bfloat162 w01 = *reinterpret_cast<const __nv_bfloat162*>(&wb.x);
    const __nv_bfloat162 w23 = *reinterpret_cast<const __nv_bfloat162*>(&wb.y);
    uint2 ob;
    ob.x = sm100::pack_bf16x2((row_s[f] * inv) * __low2float(w01), (row_s[f + 1] * inv) * __high2float(w01));
    ob.y = sm100::pack_bf16x2((row_s[f + 2] * inv) * __low2float(w23), (row_s[f + 3] * inv) * __high2float(w23));
    *reinterpret_cast<uint2*>(h_norm + row * n + f) = ob;
  }
}

}  // namespace layer

const double* rope_inv_freq(Ctx& ctx, int head_dim, float theta) {
  if (ctx.rope_freq && ctx.rope_dim == head_dim && ctx.rope_theta == theta) return ctx.rope_freq;
  std::vector<double> h(head_dim / 2);
  for (int i = 0; i < head_dim / 2; ++i) h[i] = std::pow((double)theta, -(2.0 * i) / head_dim);
  if (ctx.rope_freq) cudaFree(ctx.rope_freq);
  ctx.rope_freq = nullptr;
  if (cudaMalloc(&ctx.rope_freq, h.size() * sizeof(double)) != cudaSuccess) return nullptr;
  cudaMemcpy(ctx.rope_freq, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
  ctx.rope_dim = head_dim;
  ctx.rope_theta = theta;
  return ctx.rope_freq;
}

size_t mfa_layer_workspace_bytes(const MfaLayerArgs& a, int num_sms) {
  const int B = a.batch, Hd = a.hidden, QL = a.q_lora, NQ = a.n_heads * a.head_dim;
  size_t b = 0;
  b += align_up((size_t)B * Hd * 2, 256);                       // xn
  b += align_up((size_t)B * QL * 2, 256);                       // qa
  b += align_up((size_t)B * NQ * 2, 256);                       // q
  b += align_up((size_t)B * NQ * 2, 256);                       // attn
  size_t part = linear_workspace_bytes(make_linear_plan(B, QL + 2 * a.head_dim, Hd), num_sms);
  const size_t p2 = linear_workspace_bytes(make_linear_plan(B, NQ, QL), num_sms);
  const size_t p3 = linear_workspace_bytes(make_linear_plan(B, Hd, NQ), num_sms);
  const size_t p4 = mfa_decode_workspace_bytes(B, num_sms);
  part = part > p2 ? part : p2;
  part = part > p3 ? part : p3;
  part = part > p4 ? part : p4;
  return b + part;
}

cudaError_t mfa_layer_launch(Ctx& ctx, const MfaLayerArgs& a, void* ws_base, cudaStream_t stream) {
  using namespace layer;
  const int B = a.batch, Hd = a.hidden, QL = a.q_lora, D = a.head_dim, NQ = a.n_heads * a.head_dim;
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* xn = static_cast<__nv_bfloat16*>(take((size_t)B * Hd * 2));
  auto* qa = static_cast<__nv_bfloat16*>(take((size_t)B * QL * 2));
  auto* q = static_cast<__nv_bfloat16*>(take((size_t)B * NQ * 2));
  auto* attn = static_cast<__nv_bfloat16*>(take((size_t)B * NQ * 2));
  float* part = reinterpret_cast<float*>(ws);
  const double* inv_freq = rope_inv_freq(ctx, D, a.rope_theta);
  if (!inv_freq) return cudaErrorMemoryAllocation;
  cudaError_t e;

  // K1a: input RMSNorm
  if ((e = launch_k(ctx.pdl, rmsnorm_kernel, dim3(B), dim3(1024), 0, stream, static_cast<const __nv_bfloat16*>(a.x),
                    static_cast<const __nv_bfloat16*>(a.w_in_norm), xn, Hd, a.rms_eps)) != cudaSuccess)
    return e;
  // K1b: [q_down | k | v] projection, then q RMSNorm + RoPE(k) + paged KV append
  const LinearPlan p1 = make_linear_plan(B, QL + 2 * D, Hd);
  if ((e = linear_bf16_launch(ctx, p1, xn, a.w_qkv, part, stream)) != cudaSuccess) return e;
  QkvEpi qe{QL, D, a.page_size, a.max_pages, p1.n_out, a.rms_eps,
            static_cast<const __nv_bfloat16*>(a.w_q_norm), qa, static_cast<__nv_bfloat16*>(a.k_cache),
            static_cast<__nv_bfloat16*>(a.v_cache), a.block_table, a.seq_lens, inv_freq, a.k_scale, a.v_scale};
  if ((e = launch_k(ctx.pdl, qkv_epilogue_kernel, dim3(B), dim3(512), p1.n_out * sizeof(float), stream, p1,
                    (const float*)part, linear_grid(ctx, p1), qe)) != cudaSuccess)
    return e;
  // K1c: q_up projection + RoPE(q)
  const LinearPlan p2 = make_linear_plan(B, NQ, QL);
  if ((e = linear_bf16_launch(ctx, p2, qa, a.w_q_up, part, stream)) != cudaSuccess) return e;
  if ((e = launch_k(ctx.pdl, qup_epilogue_kernel, dim3(B, (NQ / 2 + 1023) / 1024), dim3(1024), 0, stream, p2,
                    (const float*)part, linear_grid(ctx, p2), NQ, D, a.seq_lens, inv_freq, q)) != cudaSuccess)
    return e;
  // K2/K3: MFA decode core over the paged cache (now including this token)
  MfaDecodeArgs md{B, q, a.k_cache, a.v_cache, a.num_pages, a.block_table, a.max_pages, a.seq_lens,
                   a.softmax_scale, attn, nullptr, part, a.k_scale, a.v_scale};
  if ((e = (a.k_scale > 0.0f ? mfa_decode_fp8_launch(ctx, md, stream) : mfa_decode_launch(ctx, md, stream))) !=
      cudaSuccess)
    return e;
  // K4: o_proj, then residual + post-attention RMSNorm
  const LinearPlan p3 = make_linear_plan(B, Hd, NQ);
  if ((e = linear_bf16_launch(ctx, p3, attn, a.w_o, part, stream)) != cudaSuccess) return e;
  if ((e = launch_k(ctx.pdl, o_epilogue_kernel, dim3(B), dim3(1024), Hd * sizeof(float), stream, p3,
                    (const float*)part, linear_grid(ctx, p3), Hd, static_cast<const __nv_bfloat16*>(a.x),
                    static_cast<const __nv_bfloat16*>(a.w_post_norm), a.rms_eps,
                    static_cast<__nv_bfloat16*>(a.h_res), static_cast<__nv_bfloat16*>(a.h_norm))) != cudaSuccess)
    return e;
  return cudaGetLastError();
}

}  // namespace afdk
