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
#include <cstdlib>
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

// Row statistics over a 4-CTA cluster (one row per cluster, a quarter of the
// features per CTA): every CTA pushes its block sum into slot [its rank] of
// all four CTAs with st.async (completing 4 bytes on each receiver's
// mbarrier), then adds the four slots in rank order, so all four hold the
// identical total.  No cluster barrier (and no fence) on the critical path:
// row_red_init arms the barrier and publishes it before the PDL wait.
// kC = CTAs per row (4 at decode batches; 2 from 128 token rows, where 4
// would launch 4 x B CTAs, several waves of the latency-bound kernel).
template <int kC>
struct RowRed {
  uint64_t bar;
  float slot[kC];
};
template <int kC>
__device__ __forceinline__ void row_red_init(RowRed<kC>& rr) {
  if (threadIdx.x == 0) {
    sm100::mbar_init(&rr.bar, 1);
    sm100::fence_barrier_init();
    sm100::mbar_expect_tx(&rr.bar, 4 * kC);
  }
  sm100::cluster_sync();  // every CTA's barrier is initialised before any peer stores into it
}
template <int kC>
__device__ __forceinline__ float cluster_row_sum(float v, float* red, RowRed<kC>& rr) {
  v = block_sum(v, red);
  if (threadIdx.x == 0) {
    const uint32_t me = sm100::cluster_ctarank();
#pragma unroll
    for (int r = 0; r < kC; ++r)
      sm100::st_async_f32(sm100::mapa_shared(&rr.slot[me], r), v, sm100::mapa_shared(&rr.bar, r));
  }
  sm100::mbar_wait(&rr.bar, 0);
  float t = 0.0f;
#pragma unroll
  for (int r = 0; r < kC; ++r) t += rr.slot[r];
  return t;
}

// xn = RMSNorm(x) * w, bf16 out (input_layernorm); grid B*4 in 4-CTA clusters,
// CTA r of a row's cluster owns features [r*dim/4, (r+1)*dim/4); dim % 16 == 0
template <int kC>
__global__ void __launch_bounds__(512) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ w,
                                                      __nv_bfloat16* __restrict__ out, int dim, float eps) {
  __shared__ float red[32];
  __shared__ RowRed<kC> rr;
  row_red_init(rr);
  sm100::griddep_wait();
  sm100::griddep_launch();
  const size_t row = blockIdx.x / kC;
  const int q = dim / kC, f0 = (int)sm100::cluster_ctarank() * q;
  const __nv_bfloat16* xr = x + row * dim;
  constexpr int kMax = 4;  // float4 groups per thread (dim/4 <= 4*4*512)
  float2 a[kMax], b[kMax];
  float ss = 0.0f;
#pragma unroll
  for (int j = 0; j < kMax; ++j) {
    const int i = f0 + (threadIdx.x + j * blockDim.x) * 4;
    a[j] = b[j] = make_float2(0.f, 0.f);
    if (i < f0 + q) {
      const uint2 xb = *reinterpret_cast<const uint2*>(xr + i);
      a[j] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.x));
      b[j] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xb.y));
      ss += a[j].x * a[j].x + a[j].y * a[j].y + b[j].x * b[j].x + b[j].y * b[j].y;
    }
  }
  ss = cluster_row_sum(ss, red, rr);
  const float inv = rsqrtf(ss / dim + eps);
#pragma unroll
  for (int j = 0; j < kMax; ++j) {
    const int i = f0 + (threadIdx.x + j * blockDim.x) * 4;
    if (i < f0 + q) {
      const uint2 wb = *reinterpret_cast<const uint2*>(w + i);
      const float2 wa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.x));
      const float2 wc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.y));
      uint2 o;
      o.x = sm100::pack_bf16x2((a[j].x * inv) * wa.x, (a[j].y * inv) * wa.y);
      o.y = sm100::pack_bf16x2((b[j].x * inv) * wc.x, (b[j].y * inv) * wc.y);
      *reinterpret_cast<uint2*>(out + row * dim + i) = o;
    }
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
  int mtp;                      // row r = token r % mtp of request r / mtp, position seq_len - mtp + j
  float2* rope_cs;              // out (optional): [B, head_dim/2] (cos, sin) of each row's position,
                                // for the RoPE(q) fused into the q_up GEMM
};

__device__ __forceinline__ uint8_t kv_e4m3(float x, float scale) {
  return (uint8_t)__nv_cvt_float_to_fp8(__fdiv_rn(x, scale), __NV_SATFINITE, __NV_E4M3);
}

// y = [q_down|k|v] projection of one token row (fp32): q -> RMSNorm -> qa;
// k -> RoPE -> K cache slot of position seq_len-1; v -> V cache slot.
// grid B*4 in 4-CTA clusters: CTA r < 3 owns q features [r*QL/4, (r+1)*QL/4),
// CTA 3 the last quarter of q plus all of k and v (q RMSNorm statistics over
// the cluster; CTA 3 does the RoPE + KV append).  QL/4 + 2*head_dim <= 2048.
template <int kC>
__global__ void __launch_bounds__(512) qkv_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                           int G, const QkvEpi e) {
  __shared__ float red[32];
  __shared__ RowRed<kC> rr;
  __shared__ float kv_s[2 * 256];  // k then v of this row (head_dim <= 256)
  __shared__ float2 cs_s[128];     // RoPE (cos, sin) of this row's position (head_dim <= 256)
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  row_red_init(rr);
  const int row = blockIdx.x / kC;
  const int rank = (int)sm100::cluster_ctarank();
  const int qs = e.q_lora / kC, f0 = rank * qs;
  const int f1 = rank == kC - 1 ? e.n_out : f0 + qs;
  const int req = row / e.mtp;
  const int pos = __ldg(e.seq_lens + req) - e.mtp + row % e.mtp;
  if (f1 > e.q_lora) {
    // the rotation depends only on inputs (seq_lens, inv_freq): one
    // double-precision sincos per frequency, before the PDL wait (rows with
    // no position yet, L < mtp, rotate q by position 0 like the oracle)
    const int p0 = max(pos, 0);
    for (int i = threadIdx.x; i < e.head_dim / 2; i += blockDim.x) {
      double sn, cs;
      sincos((double)p0 * e.inv_freq[i], &sn, &cs);
      cs_s[i] = make_float2((float)cs, (float)sn);
    }
  }
  sm100::griddep_wait();
  sm100::griddep_launch();
  if (f1 > e.q_lora && e.rope_cs) {
    __syncthreads();
    for (int i = threadIdx.x; i < e.head_dim / 2; i += blockDim.x) e.rope_cs[(size_t)row * (e.head_dim / 2) + i] = cs_s[i];
  }
  const int f = f0 + threadIdx.x * 4;  // 4 features per thread ((f1 - f0)/4 <= blockDim)
  const bool act = f < f1;
  float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float ss = 0.0f;
  if (act) {
    v4 = tab.sum4(P, part, row, f);
    v4 = make_float4(bf16r(v4.x), bf16r(v4.y), bf16r(v4.z), bf16r(v4.w));
    if (f < e.q_lora) ss = v4.x * v4.x + v4.y * v4.y + v4.z * v4.z + v4.w * v4.w;
    else {
      const int o = f - e.q_lora;  // k (and v) features of this row
      kv_s[o] = v4.x; kv_s[o + 1] = v4.y; kv_s[o + 2] = v4.z; kv_s[o + 3] = v4.w;
    }
  }
  ss = cluster_row_sum(ss, red, rr);  // includes __syncthreads: kv_s complete
  const float inv = rsqrtf(ss / e.q_lora + e.eps);
  if (act && f < e.q_lora) {
    const uint2 wb = *reinterpret_cast<const uint2*>(e.q_norm_w + f);
    const float2 wa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.x));
    const float2 wc = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wb.y));
    uint2 o;
    o.x = sm100::pack_bf16x2((v4.x * inv) * wa.x, (v4.y * inv) * wa.y);
    o.y = sm100::pack_bf16x2((v4.z * inv) * wc.x, (v4.w * inv) * wc.y);
    *reinterpret_cast<uint2*>(e.qa + (size_t)row * e.q_lora + f) = o;
  }
  if (f1 <= e.q_lora) return;  // this CTA holds no k/v features
  if (pos < 0) return;
  const int pg = __ldg(e.block_table + (size_t)req * e.max_pages + pos / e.page);
  const size_t kslot = ((size_t)pg * e.page + pos % e.page) * e.head_dim;
  const int half = e.head_dim / 2;
  const float* k = kv_s;
  const float* v = kv_s + e.head_dim;
  const bool fp8 = e.k_scale > 0.0f;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float c = cs_s[i].x, s = cs_s[i].y;
    const float x1 = k[i], x2 = k[i + half];
    const __nv_bfloat16 k1 = __float2bfloat16_rn(x1 * c - x2 * s), k2 = __float2bfloat16_rn(x2 * c + x1 * s);
    if (fp8) {
      uint8_t* k8 = reinterpret_cast<uint8_t*>(e.k_cache);
      k8[kslot + i] = kv_e4m3(__bfloat162float(k1), e.k_scale);
      k8[kslot + i + half] = kv_e4m3(__bfloat162float(k2), e.k_scale);
    } else {
      e.k_cache[kslot + i] = k1;
      e.k_cache[kslot + i + half] = k2;
    }
  }
  for (int i = threadIdx.x; i < e.head_dim; i += blockDim.x) {
    if (fp8)
      reinterpret_cast<uint8_t*>(e.v_cache)[kslot + i] = kv_e4m3(v[i], e.v_scale);
    else
      e.v_cache[kslot + i] = __float2bfloat16_rn(v[i]);
  }
}

// y = q_up projection (fp32 [B, n_heads*head_dim]); per-head NeoX RoPE -> q bf16.
// grid (B, ceil(n_out/8/blockDim)): each thread rotates 4 consecutive pairs.
__global__ void __launch_bounds__(256) qup_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                            int G, int n_out, int head_dim,
                                                            const int32_t* __restrict__ seq_lens, int mtp,
                                                            const double* __restrict__ inv_freq,
                                                            __nv_bfloat16* __restrict__ q) {
  __shared__ lin::SlotTable tab;
  __shared__ float2 cs_s[256];  // (cos, sin) of the row's position per frequency (head_dim <= 512)
  lin::build_slot_table(P, G, tab);
  const int row = blockIdx.x;
  const int half = head_dim / 2;
  const int pos = max(__ldg(seq_lens + row / mtp) - mtp + row % mtp, 0);
  // every head shares the row's rotation: one double-precision sincos per
  // frequency per CTA (seq_lens / inv_freq are inputs: before griddep_wait)
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    double sn, cs;
    sincos((double)pos * inv_freq[i], &sn, &cs);
    cs_s[i] = make_float2((float)cs, (float)sn);
  }
  __syncthreads();
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int idx = (blockIdx.y * blockDim.x + threadIdx.x) * 4;  // first of 4 consecutive pairs in the row
  if (idx >= n_out / 2) return;
  const int h = idx / half, i = idx % half;  // half % 4 == 0: the 4 pairs share the head
  const int c1 = h * head_dim + i;
  const float4 a = tab.sum4(P, part, row, c1), b = tab.sum4(P, part, row, c1 + half);
  const float x1[4] = {bf16r(a.x), bf16r(a.y), bf16r(a.z), bf16r(a.w)};
  const float x2[4] = {bf16r(b.x), bf16r(b.y), bf16r(b.z), bf16r(b.w)};
  float o1[4], o2[4];
#pragma unroll
  for (int z = 0; z < 4; ++z) {
    const float c = cs_s[i + z].x, s = cs_s[i + z].y;
    o1[z] = x1[z] * c - x2[z] * s;
    o2[z] = x2[z] * c + x1[z] * s;
  }
  const size_t f1 = (size_t)row * n_out + c1;
  *reinterpret_cast<uint2*>(q + f1) = make_uint2(sm100::pack_bf16x2(o1[0], o1[1]), sm100::pack_bf16x2(o1[2], o1[3]));
  *reinterpret_cast<uint2*>(q + f1 + half) =
      make_uint2(sm100::pack_bf16x2(o2[0], o2[1]), sm100::pack_bf16x2(o2[2], o2[3]));
}

// y = o_proj (fp32); h_res = bf16(x + y); h_norm = RMSNorm(h_res) (post_attention_layernorm)
// grid B*4 in 4-CTA clusters, CTA r owns features [r*n/4, (r+1)*n/4); n % 16 == 0
template <int kC>
__global__ void __launch_bounds__(512) o_epilogue_kernel(const LinearPlan P, const float* __restrict__ part,
                                                         int G, int n, const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ w_post, float eps,
                                                         __nv_bfloat16* __restrict__ h_res,
                                                         __nv_bfloat16* __restrict__ h_norm) {
  __shared__ float red[32];
  __shared__ RowRed<kC> rr;
  __shared__ lin::SlotTable tab;
  lin::build_slot_table(P, G, tab);
  row_red_init(rr);
  const size_t row = blockIdx.x / kC;
  const int q = n / kC, f0 = (int)sm100::cluster_ctarank() * q;
  constexpr int kMax = 2;  // float4 groups per thread (n/4 <= 2*4*512)
  // the residual input x and the norm weight are inputs of the layer (x was
  // complete before its first kernel ran): load them before the PDL wait
  uint2 xbv[kMax], wbv[kMax];
#pragma unroll
  for (int j = 0; j < kMax; ++j) {
    const int f = f0 + (threadIdx.x + j * blockDim.x) * 4;
    if (f < f0 + q) {
      xbv[j] = *reinterpret_cast<const uint2*>(x + row * n + f);
      wbv[j] = *reinterpret_cast<const uint2*>(w_post + f);
    }
  }
  sm100::griddep_wait();
  sm100::griddep_launch();
  float r[kMax][4];
  float ss = 0.0f;
#pragma unroll
  for (int j = 0; j < kMax; ++j) {
    const int f = f0 + (threadIdx.x + j * blockDim.x) * 4;
    if (f < f0 + q) {
      const float4 o = tab.sum4(P, part, (int)row, f);
      const uint2 xb = xbv[j];
      const __nv_bfloat162 x01 = *reinterpret_cast<const __nv_bfloat162*>(&xb.x);
      const __nv_bfloat162 x23 = *reinterpret_cast<const __nv_bfloat162*>(&xb.y);
      r[j][0] = bf16r(__low2float(x01) + o.x);
      r[j][1] = bf16r(__high2float(x01) + o.y);
      r[j][2] = bf16r(__low2float(x23) + o.z);
      r[j][3] = bf16r(__high2float(x23) + o.w);
      uint2 ob;
      ob.x = sm100::pack_bf16x2(r[j][0], r[j][1]);
      ob.y = sm100::pack_bf16x2(r[j][2], r[j][3]);
      *reinterpret_cast<uint2*>(h_res + row * n + f) = ob;
#pragma unroll
      for (int z = 0; z < 4; ++z) ss += r[j][z] * r[j][z];
    }
  }
  ss = cluster_row_sum(ss, red, rr);
  const float inv = rsqrtf(ss / n + eps);
#pragma unroll
  for (int j = 0; j < kMax; ++j) {
    const int f = f0 + (threadIdx.x + j * blockDim.x) * 4;
    if (f < f0 + q) {
      const uint2 wb = wbv[j];
      const __nv_bfloat162 w01 = *reinterpret_cast<const __nv_bfloat162*>(&wb.x);
      const __nv_bfloat162 w23 = *reinterpret_cast<const __nv_bfloat162*>(&wb.y);
      uint2 ob;
      ob.x = sm100::pack_bf16x2((r[j][0] * inv) * __low2float(w01), (r[j][1] * inv) * __high2float(w01));
      ob.y = sm100::pack_bf16x2((r[j][2] * inv) * __low2float(w23), (r[j][3] * inv) * __high2float(w23));
      *reinterpret_cast<uint2*>(h_norm + row * n + f) = ob;
    }
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
  const int B = a.batch * a.mtp, Hd = a.hidden, QL = a.q_lora, NQ = a.n_heads * a.head_dim;
  size_t b = 0;
  b += align_up((size_t)B * Hd * 2, 256);                       // xn
  b += align_up((size_t)B * QL * 2, 256);                       // qa
  b += align_up((size_t)B * NQ * 2, 256);                       // q
  b += align_up((size_t)B * NQ * 2, 256);                       // attn
  b += align_up((size_t)B * (a.head_dim / 2) * 8, 256);         // rope (cos, sin)
  size_t part = linear_workspace_bytes(make_linear_plan(B, QL + 2 * a.head_dim, Hd), num_sms);
  const size_t p2 = linear_workspace_bytes(make_linear_plan(B, NQ, QL), num_sms);
  const size_t p3 = linear_workspace_bytes(make_linear_plan(B, Hd, NQ), num_sms);
  const size_t p4 = a.mtp > 1 ? mfa_decode_mtp_workspace_bytes(a.batch, num_sms) : mfa_decode_workspace_bytes(B, num_sms);
  part = part > p2 ? part : p2;
  part = part > p3 ? part : p3;
  part = part > p4 ? part : p4;
  return b + part;
}

cudaError_t mfa_layer_launch(Ctx& ctx, const MfaLayerArgs& a, void* ws_base, cudaStream_t stream) {
  using namespace layer;
  // B = token rows (requests x mtp) for norms, projections and epilogues
  const int B = a.batch * a.mtp, Hd = a.hidden, QL = a.q_lora, D = a.head_dim, NQ = a.n_heads * a.head_dim;
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* xn = static_cast<__nv_bfloat16*>(take((size_t)B * Hd * 2));
  auto* qa = static_cast<__nv_bfloat16*>(take((size_t)B * QL * 2));
  auto* q = static_cast<__nv_bfloat16*>(take((size_t)B * NQ * 2));
  auto* attn = static_cast<__nv_bfloat16*>(take((size_t)B * NQ * 2));
  auto* rope_cs = static_cast<float2*>(take((size_t)B * (D / 2) * 8));
  float* part = reinterpret_cast<float*>(ws);
  const double* inv_freq = rope_inv_freq(ctx, D, a.rope_theta);
  if (!inv_freq) return cudaErrorMemoryAllocation;
  cudaError_t e;

  // row epilogues: 4-CTA clusters per token row at decode batches, 2-CTA
  // clusters from 128 rows (AFDK_ROW_CLUSTER=2/4 forces)
  static const int env_c = [] { const char* v = std::getenv("AFDK_ROW_CLUSTER"); return v ? std::atoi(v) : 0; }();
  const bool wide = env_c ? env_c == 2 : B >= 128;
  auto row_launch = [&](auto k2, auto k4, auto&&... args) {
    return wide ? launch_cluster_k(ctx.pdl, 2, k2, dim3(B * 2), dim3(512), 0, stream, args...)
                : launch_cluster_k(ctx.pdl, 4, k4, dim3(B * 4), dim3(512), 0, stream, args...);
  };
  // K1a: input RMSNorm
  if ((e = row_launch(rmsnorm_kernel<2>, rmsnorm_kernel<4>, static_cast<const __nv_bfloat16*>(a.x),
                      static_cast<const __nv_bfloat16*>(a.w_in_norm), xn, Hd, a.rms_eps)) != cudaSuccess)
    return e;
  // K1b: [q_down | k | v] projection, then q RMSNorm + RoPE(k) + paged KV append
  const LinearPlan p1 = make_linear_plan(B, QL + 2 * D, Hd);
  if ((e = linear_bf16_launch(ctx, p1, xn, a.w_qkv, part, stream)) != cudaSuccess) return e;
  QkvEpi qe{QL, D, a.page_size, a.max_pages, p1.n_out, a.rms_eps,
            static_cast<const __nv_bfloat16*>(a.w_q_norm), qa, static_cast<__nv_bfloat16*>(a.k_cache),
            static_cast<__nv_bfloat16*>(a.v_cache), a.block_table, a.seq_lens, inv_freq, a.k_scale, a.v_scale,
            a.mtp, nullptr};
  const LinearPlan p2 = a.w_qup_mx ? make_linear_mx_plan(B, NQ, QL) : make_linear_plan(B, NQ, QL);
  // fused RoPE(q) epilogue: one launch less and equal time at decode batches
  // (B=64: 124.9 vs 124.2 us/layer); its 4 epilogue warps serialise the
  // rotation of every token, so from 128 token rows the separate row
  // epilogue is faster (B=256: 308 vs 302 us, e4m3 KV 240 vs 230 us)
  const bool qup_mx = a.w_qup_mx != nullptr;
  const bool fused_rope =
      !qup_mx && linear_rope_fusable(ctx, p2, D) && B <= 64 && !std::getenv("AFDK_NO_ROPE_FUSION");
  if (fused_rope) qe.rope_cs = rope_cs;
  if ((e = row_launch(qkv_epilogue_kernel<2>, qkv_epilogue_kernel<4>, p1, (const float*)part, linear_grid(ctx, p1),
                      qe)) != cudaSuccess)
    return e;
  // K1c: q_up projection + RoPE(q): fused into the GEMM's epilogue when every
  // CTA owns a whole tile (the layer's shape on 148 SMs), else a row epilogue
  if (fused_rope) {
    if ((e = linear_bf16_rope_launch(ctx, p2, qa, a.w_q_up, q, rope_cs, D, stream)) != cudaSuccess) return e;
  } else {
    if (qup_mx) {  // MXFP8 q_up: the q latent MX-quantised into the (not yet written) attention buffer
      uint8_t* q8 = reinterpret_cast<uint8_t*>(attn);
      uint8_t* qsf = q8 + (size_t)B * QL;
      moe::QuantMxArgs qm{qa, B, QL, q8, qsf};
      if ((e = quant_mx_launch(qm, stream, ctx.pdl)) != cudaSuccess) return e;
      if ((e = linear_mx_launch(ctx, p2, q8, qsf, a.w_qup_mx, a.w_qup_sf, part, stream)) != cudaSuccess) return e;
    } else if ((e = linear_bf16_launch(ctx, p2, qa, a.w_q_up, part, stream)) != cudaSuccess) {
      return e;
    }
    if ((e = launch_k(ctx.pdl, qup_epilogue_kernel, dim3(B, (NQ / 8 + 255) / 256), dim3(256), 0, stream, p2,
                      (const float*)part, linear_grid(ctx, p2), NQ, D, a.seq_lens, a.mtp, inv_freq, q)) !=
        cudaSuccess)
      return e;
  }
  // K2/K3: MFA decode core over the paged cache (now including this token)
  MfaDecodeArgs md{a.batch, q, a.k_cache, a.v_cache, a.num_pages, a.block_table, a.max_pages, a.seq_lens,
                   a.softmax_scale, attn, nullptr, part, a.k_scale, a.v_scale};
  if ((e = (a.mtp > 1 ? mfa_decode_mtp_launch(ctx, md, stream)
            : a.k_scale > 0.0f ? mfa_decode_fp8_launch(ctx, md, stream) : mfa_decode_launch(ctx, md, stream))) !=
      cudaSuccess)
    return e;
  // K4: o_proj, then residual + post-attention RMSNorm.  With MXFP8 o_proj
  // weights the attention output is MX-quantised into the (consumed) q buffer
  // and the projection runs on the block-scaled MMA (linear_mx.cu).
  const bool o_mx = a.w_o_mx != nullptr;
  const LinearPlan p3 = o_mx ? make_linear_mx_plan(B, Hd, NQ) : make_linear_plan(B, Hd, NQ);
  if (o_mx) {
    uint8_t* oq = reinterpret_cast<uint8_t*>(q);
    uint8_t* osf = oq + (size_t)B * NQ;
    moe::QuantMxArgs qa{attn, B, NQ, oq, osf};
    if ((e = quant_mx_launch(qa, stream, ctx.pdl)) != cudaSuccess) return e;
    if ((e = linear_mx_launch(ctx, p3, oq, osf, a.w_o_mx, a.w_o_sf, part, stream)) != cudaSuccess) return e;
  } else if ((e = linear_bf16_launch(ctx, p3, attn, a.w_o, part, stream)) != cudaSuccess) {
    return e;
  }
  if ((e = row_launch(o_epilogue_kernel<2>, o_epilogue_kernel<4>, p3, (const float*)part, linear_grid(ctx, p3), Hd,
                      static_cast<const __nv_bfloat16*>(a.x), static_cast<const __nv_bfloat16*>(a.w_post_norm),
                      a.rms_eps, static_cast<__nv_bfloat16*>(a.h_res), static_cast<__nv_bfloat16*>(a.h_norm))) !=
      cudaSuccess)
    return e;
  return cudaGetLastError();
}

}  // namespace afdk
