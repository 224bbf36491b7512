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
// the row epilogue that reduces that GEMM's partials.  Intermediates are
// stored in bf16 exactly where the oracle (orc_mfa_layer) rounds.
#include <cuda_bf16.h>
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

// xn = RMSNorm(x) * w, bf16 out (input_layernorm)
__global__ void rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                               __nv_bfloat16* __restrict__ out, int dim, float eps) {
  __shared__ float red[32];
  const size_t row = blockIdx.x;
  const __nv_bfloat16* xr = x + row * dim;
  float ss = 0.0f;
  for (int i = threadIdx.x; i < dim; i += blockDim.x) {
    const float v = __bfloat162float(xr[i]);
    ss += v * v;
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / dim + eps);
  for (int i = threadIdx.x; i < dim; i += blockDim.x)
    out[row * dim + i] = __float2bfloat16_rn((__bfloat162float(xr[i]) * inv) * __bfloat162float(w[i]));
}

struct QkvEpi {
  int q_lora, head_dim, page, max_pages;
  float eps;
  const __nv_bfloat16* q_norm_w;
  __nv_bfloat16* qa;            // [B, q_lora]
  __nv_bfloat16* k_cache;       // [num_pages, page, head_dim]
  __nv_bfloat16* v_cache;
  const int32_t* block_table;
  const int32_t* seq_lens;
  const double* inv_freq;       // [head_dim/2]
};

// reduce [q_down|k|v] partials of one token row; q: RMSNorm -> qa; k: RoPE ->
// K cache slot of position seq_len-1; v -> V cache slot.
__global__ void qkv_epilogue_kernel(const LinearPlan P, const float* __restrict__ part, int G, const QkvEpi e) {
  extern __shared__ float row_s[];  // n_out floats
  __shared__ float red[32];
  const int row = blockIdx.x;
  float ss = 0.0f;
  for (int f = threadIdx.x; f < P.n_out; f += blockDim.x) {
    const float v = bf16r(lin::linear_partial_sum(P, part, G, row, f));
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
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    double sn, cs;
    sincos((double)pos * e.inv_freq[i], &sn, &cs);
    const float c = (float)cs, s = (float)sn;
    const float x1 = k[i], x2 = k[i + half];
    e.k_cache[slot + i] = __float2bfloat16_rn(x1 * c - x2 * s);
    e.k_cache[slot + i + half] = __float2bfloat16_rn(x2 * c + x1 * s);
  }
  for (int i = threadIdx.x; i < e.head_dim; i += blockDim.x) e.v_cache[slot + i] = __float2bfloat16_rn(v[i]);
}

// reduce q_up partials; per-head NeoX RoPE; q [B, n_heads, head_dim] bf16
__global__ void qup_epilogue_kernel(const LinearPlan P, const float* __restrict__ part, int G, int head_dim,
                                    const int32_t* __restrict__ seq_lens, const double* __restrict__ inv_freq,
                                    __nv_bfloat16* __restrict__ q) {
  const int row = blockIdx.x;
  const int half = head_dim / 2;
  const int pos = max(__ldg(seq_lens + row) - 1, 0);
  for (int idx = threadIdx.x; idx < P.n_out / 2; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    const int f1 = h * head_dim + i, f2 = f1 + half;
    const float x1 = bf16r(lin::linear_partial_sum(P, part, G, row, f1));
    const float x2 = bf16r(lin::linear_partial_sum(P, part, G, row, f2));
    double sn, cs;
    sincos((double)pos * inv_freq[i], &sn, &cs);
    const float c = (float)cs, s = (float)sn;
    q[(size_t)row * P.n_out + f1] = __float2bfloat16_rn(x1 * c - x2 * s);
    q[(size_t)row * P.n_out + f2] = __float2bfloat16_rn(x2 * c + x1 * s);
  }
}

// reduce o_proj partials; h_res = bf16(x + o); h_norm = RMSNorm(h_res) (post_attention_layernorm)
__global__ void o_epilogue_kernel(const LinearPlan P, const float* __restrict__ part, int G,
                                  const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w_post,
                                  float eps, __nv_bfloat16* __restrict__ h_res, __nv_bfloat16* __restrict__ h_norm) {
  extern __shared__ float row_s[];
  __shared__ float red[32];
  const int row = blockIdx.x;
  const int n = P.n_out;
  float ss = 0.0f;
  for (int f = threadIdx.x; f < n; f += blockDim.x) {
    const float r = bf16r(__bfloat162float(x[(size_t)row * n + f]) + lin::linear_partial_sum(P, part, G, row, f));
    row_s[f] = r;
    h_res[(size_t)row * n + f] = __float2bfloat16_rn(r);
    ss += r * r;
  }
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / n + eps);
  for (int f = threadIdx.x; f < n; f += blockDim.x)
    h_norm[(size_t)row * n + f] = __float2bfloat16_rn((row_s[f] * inv) * __bfloat162float(w_post[f]));
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
  b += align_up((size_t)B * Hd * 2, 256);  // xn
  b += align_up((size_t)B * QL * 2, 256);  // qa
  b += align_up((size_t)B * NQ * 2, 256);  // q
  b += align_up((size_t)B * NQ * 2, 256);  // attn
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
  const int G = ctx.num_sms;
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
  rmsnorm_kernel<<<B, 512, 0, stream>>>(static_cast<const __nv_bfloat16*>(a.x),
                                         static_cast<const __nv_bfloat16*>(a.w_in_norm), xn, Hd, a.rms_eps);
  // K1b: [q_down | k | v] projection + q RMSNorm + RoPE(k) + paged KV append
  const LinearPlan p1 = make_linear_plan(B, QL + 2 * D, Hd);
  if ((e = linear_bf16_launch(ctx, p1, xn, a.w_qkv, part, stream)) != cudaSuccess) return e;
  QkvEpi qe{QL, D, a.page_size, a.max_pages, a.rms_eps, static_cast<const __nv_bfloat16*>(a.w_q_norm), qa,
            static_cast<__nv_bfloat16*>(a.k_cache), static_cast<__nv_bfloat16*>(a.v_cache), a.block_table,
            a.seq_lens, inv_freq};
  qkv_epilogue_kernel<<<B, 256, p1.n_out * sizeof(float), stream>>>(p1, part, G, qe);
  // K1c: q_up projection + RoPE(q)
  const LinearPlan p2 = make_linear_plan(B, NQ, QL);
  if ((e = linear_bf16_launch(ctx, p2, qa, a.w_q_up, part, stream)) != cudaSuccess) return e;
  qup_epilogue_kernel<<<B, 512, 0, stream>>>(p2, part, G, D, a.seq_lens, inv_freq, q);
  // K2/K3: MFA decode core over the paged cache (now including this token)
  MfaDecodeArgs md{B, q, a.k_cache, a.v_cache, a.num_pages, a.block_table, a.max_pages, a.seq_lens,
                   a.softmax_scale, attn, nullptr, part};
  if ((e = mfa_decode_launch(ctx, md, stream)) != cudaSuccess) return e;
  // K4: o_proj + residual + post-attention RMSNorm
  const LinearPlan p3 = make_linear_plan(B, Hd, NQ);
  if ((e = linear_bf16_launch(ctx, p3, attn, a.w_o, part, stream)) != cudaSuccess) return e;
  o_epilogue_kernel<<<B, 512, Hd * sizeof(float), stream>>>(p3, part, G, static_cast<const __nv_bfloat16*>(a.x),
                                                            static_cast<const __nv_bfloat16*>(a.w_post_norm),
                                                            a.rms_eps, static_cast<__nv_bfloat16*>(a.h_res),
                                                            static_cast<__nv_bfloat16*>(a.h_norm));
  return cudaGetLastError();
}

}  // namespace afdk
