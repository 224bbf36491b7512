// afdk_api.cu — the extern "C" entry points of include/afdk.h.
//
// Validation mirrors the reference's error convention (types.hpp:12-25: the
// message names the offending field); the C++ wrapper in afd_ops.cpp maps
// AFDK_ERR_INVALID back to afd::SpecError.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/afdk.h"
#include "afdk_internal.h"

namespace afdk {

cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{func, dev}];
  if (bytes <= have) return cudaSuccess;
  if ((e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)) != cudaSuccess)
    return e;
  have = bytes;
  return cudaSuccess;
}

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

void* workspace(Ctx& ctx, size_t bytes) {
  if (bytes <= ctx.ws_bytes) return ctx.ws;
  if (ctx.ws) cudaFree(ctx.ws);
  ctx.ws = nullptr;
  ctx.ws_bytes = 0;
  const size_t want = align_up(bytes, size_t(1) << 21);
  if (cudaMalloc(&ctx.ws, want) != cudaSuccess) return nullptr;
  ctx.ws_bytes = want;
  return ctx.ws;
}

bool encode_tma(Ctx& ctx, CUtensorMap* map, CUtensorMapDataType dt, int rank, void* base,
                const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                CUtensorMapSwizzle swizzle) {
  cuuint64_t d[5];
  cuuint64_t s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i + 1 < rank) s[i] = strides[i];
  }
  const CUresult r = ctx.encode(map, dt, (cuuint32_t)rank, base, d, s, b, e,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return false;
  }
  return true;
}

}  // namespace afdk

struct afdk_ctx {
  afdk::Ctx c;
};

using afdk::set_error;

static afdk_status cuda_fail(const char* what, cudaError_t e) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return AFDK_ERR_CUDA;
}

extern "C" {

int afdk_abi_version(void) { return AFDK_ABI_VERSION; }

const char* afdk_last_error(void) { return afdk::g_last_error.c_str(); }

afdk_status afdk_create(afdk_ctx** out, const afdk_cfg* cfg) {
  if (!out) { set_error("afdk_create: out is NULL"); return AFDK_ERR_INVALID; }
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    set_error("afdk_create: no CUDA device visible");
    return AFDK_ERR_NO_DEVICE;
  }
  const int dev = cfg ? cfg->device : 0;
  if (dev < 0 || dev >= n) { set_error("afdk_create: cfg.device out of range"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard device_guard(dev);
  cudaDeviceProp prop{};
  cudaError_t e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) return cuda_fail("cudaGetDeviceProperties", e);
  if (prop.major != 10 || prop.minor != 0) {
    set_error("afdk_create: device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
              ", this library is built for sm_100a only");
    return AFDK_ERR_UNSUPPORTED;
  }
  if (prop.multiProcessorCount >= afdk::kMfaMaxSplit) {
    set_error("afdk_create: " + std::to_string(prop.multiProcessorCount) +
              " SMs exceed the split-KV merge limit (" + std::to_string(afdk::kMfaMaxSplit - 1) + ")");
    return AFDK_ERR_UNSUPPORTED;
  }
  auto* ctx = new afdk_ctx();
  ctx->c.device = dev;
  ctx->c.sm_major = prop.major;
  ctx->c.sm_minor = prop.minor;
  ctx->c.num_sms = (cfg && cfg->num_sms > 0 && cfg->num_sms < prop.multiProcessorCount)
                       ? cfg->num_sms
                       : prop.multiProcessorCount;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) {
    delete ctx;
    set_error("afdk_create: cuTensorMapEncodeTiled unavailable");
    return AFDK_ERR_CUDA;
  }
  ctx->c.encode = reinterpret_cast<afdk::EncodeTiledFn>(fn);
  ctx->c.pdl = std::getenv("AFDK_NO_PDL") == nullptr;
  if ((e = cudaMalloc(&ctx->c.counters, afdk::kCounterSlots * sizeof(int))) != cudaSuccess ||
      (e = cudaMemset(ctx->c.counters, 0, afdk::kCounterSlots * sizeof(int))) != cudaSuccess) {
    delete ctx;
    return cuda_fail("afdk_create: counters", e);
  }
  *out = ctx;
  return AFDK_OK;
}

void afdk_destroy(afdk_ctx* ctx) {
  if (!ctx) return;
  if (ctx->c.ws) cudaFree(ctx->c.ws);
  if (ctx->c.rope_freq) cudaFree(ctx->c.rope_freq);
  if (ctx->c.counters) cudaFree(ctx->c.counters);
  delete ctx;
}

int afdk_num_sms(const afdk_ctx* ctx) { return ctx ? ctx->c.num_sms : 0; }
int afdk_ctx_device(const afdk_ctx* ctx) { return ctx ? ctx->c.device : -1; }

static afdk_status mfa_decode_entry(afdk_ctx* ctx, const afdk_mfa_decode_args* a, bool fp8, float k_scale,
                                    float v_scale, afdk_stream stream) {
  if (!ctx || !a) { set_error("afdk_mfa_decode_attention: NULL ctx/args"); return AFDK_ERR_INVALID; }
  if (a->n_heads != 64) { set_error("mfa_decode: n_heads must be 64"); return AFDK_ERR_INVALID; }
  if (a->head_dim != 256) { set_error("mfa_decode: head_dim must be 256"); return AFDK_ERR_INVALID; }
  if (a->page_size != 64) { set_error("mfa_decode: page_size must be 64"); return AFDK_ERR_INVALID; }
  if (a->batch <= 0 || a->batch > afdk::kMfaMaxBatch) {
    set_error("mfa_decode: batch must be in [1, " + std::to_string(afdk::kMfaMaxBatch) + "]");
    return AFDK_ERR_INVALID;
  }
  if (a->num_pages <= 0 || a->max_pages <= 0) { set_error("mfa_decode: num_pages/max_pages must be > 0"); return AFDK_ERR_INVALID; }
  if (!a->q || !a->k_cache || !a->v_cache || !a->block_table || !a->seq_lens || !a->out) {
    set_error("mfa_decode: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  if ((reinterpret_cast<uintptr_t>(a->q) | reinterpret_cast<uintptr_t>(a->k_cache) |
       reinterpret_cast<uintptr_t>(a->v_cache) | reinterpret_cast<uintptr_t>(a->out)) & 15) {
    set_error("mfa_decode: q/k_cache/v_cache/out must be 16-byte aligned");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  void* ws = afdk::workspace(c, afdk::mfa_decode_workspace_bytes(a->batch, c.num_sms));
  if (!ws) { set_error("mfa_decode: workspace allocation failed"); return AFDK_ERR_CUDA; }
  afdk::MfaDecodeArgs m{a->batch, a->q, a->k_cache, a->v_cache, a->num_pages, a->block_table,
                        a->max_pages, a->seq_lens, a->softmax_scale, a->out, a->lse, ws, k_scale, v_scale};
  const cudaError_t e = fp8 ? afdk::mfa_decode_fp8_launch(c, m, static_cast<cudaStream_t>(stream))
                            : afdk::mfa_decode_launch(c, m, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("mfa_decode launch", e);
  return AFDK_OK;
}

afdk_status afdk_mfa_decode_attention(afdk_ctx* ctx, const afdk_mfa_decode_args* a, afdk_stream stream) {
  return mfa_decode_entry(ctx, a, false, 1.0f, 1.0f, stream);
}

afdk_status afdk_mfa_decode_attention_fp8(afdk_ctx* ctx, const afdk_mfa_decode_args* a, float k_scale,
                                          float v_scale, afdk_stream stream) {
  if (!(k_scale > 0.0f) || !(v_scale > 0.0f) || !std::isfinite(k_scale) || !std::isfinite(v_scale)) {
    set_error("mfa_decode_fp8: k_scale and v_scale must be positive and finite");
    return AFDK_ERR_INVALID;
  }
  return mfa_decode_entry(ctx, a, true, k_scale, v_scale, stream);
}

afdk_status afdk_mfa_decode_attention_mtp(afdk_ctx* ctx, const afdk_mfa_decode_args* a, int mtp,
                                          afdk_stream stream) {
  if (!ctx || !a) { set_error("afdk_mfa_decode_attention_mtp: NULL ctx/args"); return AFDK_ERR_INVALID; }
  if (mtp == 1) return mfa_decode_entry(ctx, a, false, 1.0f, 1.0f, stream);
  if (mtp != 2) { set_error("mfa_decode_mtp: mtp must be 1 or 2"); return AFDK_ERR_INVALID; }
  if (a->n_heads != 64 || a->head_dim != 256 || a->page_size != 64) {
    set_error("mfa_decode_mtp: n_heads/head_dim/page_size must be 64/256/64");
    return AFDK_ERR_INVALID;
  }
  if (a->batch <= 0 || a->batch > 128) { set_error("mfa_decode_mtp: batch must be in [1, 128]"); return AFDK_ERR_INVALID; }
  if (a->num_pages <= 0 || a->max_pages <= 0) { set_error("mfa_decode_mtp: num_pages/max_pages must be > 0"); return AFDK_ERR_INVALID; }
  if (!a->q || !a->k_cache || !a->v_cache || !a->block_table || !a->seq_lens || !a->out) {
    set_error("mfa_decode_mtp: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  void* ws = afdk::workspace(c, afdk::mfa_decode_mtp_workspace_bytes(a->batch, c.num_sms));
  if (!ws) { set_error("mfa_decode_mtp: workspace allocation failed"); return AFDK_ERR_CUDA; }
  afdk::MfaDecodeArgs m{a->batch, a->q, a->k_cache, a->v_cache, a->num_pages, a->block_table,
                        a->max_pages, a->seq_lens, a->softmax_scale, a->out, a->lse, ws};
  const cudaError_t e = afdk::mfa_decode_mtp_launch(c, m, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("mfa_decode_mtp launch", e);
  return AFDK_OK;
}

afdk_status afdk_linear(afdk_ctx* ctx, const void* x, const void* w, void* out, int m, int n, int k,
                        int out_fp32, afdk_stream stream) {
  if (!ctx || !x || !w || !out) { set_error("afdk_linear: NULL argument"); return AFDK_ERR_INVALID; }
  if (m < 1 || m > 512) { set_error("afdk_linear: m must be in [1, 512]"); return AFDK_ERR_INVALID; }
  if (n < 1 || k < 64 || k % 64) { set_error("afdk_linear: k must be a positive multiple of 64"); return AFDK_ERR_INVALID; }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const afdk::LinearPlan p = afdk::make_linear_plan(m, n, k);
  float* part = static_cast<float*>(afdk::workspace(c, afdk::linear_workspace_bytes(p, c.num_sms)));
  if (!part) { set_error("afdk_linear: workspace allocation failed"); return AFDK_ERR_CUDA; }
  auto st = static_cast<cudaStream_t>(stream);
  // w may be any caller matrix, possibly written by this library's previous kernel: no PDL weight prefill
  cudaError_t e = afdk::linear_bf16_launch(c, p, x, w, part, st, /*w_dep=*/true);
  if (e == cudaSuccess) e = afdk::linear_store_launch(c, p, part, out, out_fp32 != 0, st);
  if (e != cudaSuccess) return cuda_fail("afdk_linear", e);
  return AFDK_OK;
}

afdk_status afdk_linear_mx(afdk_ctx* ctx, const void* xq, const uint8_t* xsf, const void* wq, const uint8_t* wsf,
                           void* out, int m, int n, int k, int out_fp32, afdk_stream stream) {
  if (!ctx || !xq || !xsf || !wq || !wsf || !out) { set_error("afdk_linear_mx: NULL argument"); return AFDK_ERR_INVALID; }
  if (m < 1 || m > 384) { set_error("afdk_linear_mx: m must be in [1, 384]"); return AFDK_ERR_INVALID; }
  if (n < 1 || k < 512 || k % 512) {  // scale rows (k/32 bytes) are TMA-loaded: 16-byte multiples
    set_error("afdk_linear_mx: k must be a positive multiple of 512");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const afdk::LinearPlan p = afdk::make_linear_mx_plan(m, n, k);
  float* part = static_cast<float*>(afdk::workspace(c, afdk::linear_workspace_bytes(p, c.num_sms)));
  if (!part) { set_error("afdk_linear_mx: workspace allocation failed"); return AFDK_ERR_CUDA; }
  auto st = static_cast<cudaStream_t>(stream);
  cudaError_t e = afdk::linear_mx_launch(c, p, xq, xsf, wq, wsf, part, st, /*w_dep=*/true);  // caller weights
  if (e == cudaSuccess) e = afdk::linear_store_launch(c, p, part, out, out_fp32 != 0, st);
  if (e != cudaSuccess) return cuda_fail("afdk_linear_mx", e);
  return AFDK_OK;
}

static afdk_status mfa_layer_entry(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a,
                                   float k_scale, float v_scale, afdk_stream stream, int mtp = 1) {
  if (!ctx || !w || !a) { set_error("afdk_mfa_layer: NULL ctx/weights/args"); return AFDK_ERR_INVALID; }
  if (w->n_heads != 64 || w->head_dim != 256 || a->page_size != 64) {
    set_error("afdk_mfa_layer: n_heads/head_dim/page_size must be 64/256/64");
    return AFDK_ERR_INVALID;
  }
  if (w->hidden % 64 || w->q_lora % 64 || w->q_lora < 64) {
    set_error("afdk_mfa_layer: hidden and q_lora must be multiples of 64");
    return AFDK_ERR_INVALID;
  }
  if (w->hidden > 16384 || w->q_lora > 4096) {
    set_error("afdk_mfa_layer: hidden <= 16384 and q_lora <= 4096 (row epilogues span one 4-CTA cluster)");
    return AFDK_ERR_INVALID;
  }
  if (a->batch < 1 || a->batch * mtp > 512 || (mtp > 1 && a->batch * mtp > 256)) {
    set_error("afdk_mfa_layer: batch must be in [1, 512] (batch x mtp <= 256 for mtp > 1)");
    return AFDK_ERR_INVALID;
  }
  if (!a->x || !a->k_cache || !a->v_cache || !a->block_table || !a->seq_lens || !a->h_res || !a->h_norm ||
      !w->in_norm || !w->w_qkv || !w->q_norm || (!w->w_q_up && !w->w_q_up_mx) || (!w->w_o && !w->w_o_mx) ||
      !w->post_norm) {
    set_error("afdk_mfa_layer: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  afdk::MfaLayerArgs m{a->batch, w->hidden, w->q_lora, w->n_heads, w->head_dim, a->page_size,
                       w->in_norm, w->w_qkv, w->q_norm, w->w_q_up, w->w_o, w->post_norm,
                       w->rms_eps, w->rope_theta, w->softmax_scale, a->x, a->k_cache, a->v_cache,
                       a->num_pages, a->block_table, a->max_pages, a->seq_lens, a->h_res, a->h_norm,
                       k_scale, v_scale, mtp, w->w_o_mx, w->w_o_sf, w->w_q_up_mx, w->w_q_up_sf};
  if ((w->w_o_mx != nullptr) != (w->w_o_sf != nullptr) || (w->w_o_mx && (a->batch * mtp > 384 || mtp > 1))) {
    set_error("afdk_mfa_layer: MXFP8 o_proj needs both w_o_mx and w_o_sf, mtp 1 and batch <= 384");
    return AFDK_ERR_INVALID;
  }
  if ((w->w_q_up_mx != nullptr) != (w->w_q_up_sf != nullptr) ||
      (w->w_q_up_mx && (a->batch * mtp > 384 || mtp > 1 || w->q_lora % 512 != 0))) {
    set_error("afdk_mfa_layer: MXFP8 q_up needs both w_q_up_mx and w_q_up_sf, mtp 1, batch <= 384 and q_lora % 512 == 0 (16-byte scale rows)");
    return AFDK_ERR_INVALID;
  }
  void* ws = afdk::workspace(c, afdk::mfa_layer_workspace_bytes(m, c.num_sms));
  if (!ws) { set_error("afdk_mfa_layer: workspace allocation failed"); return AFDK_ERR_CUDA; }
  const cudaError_t e = afdk::mfa_layer_launch(c, m, ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_mfa_layer", e);
  return AFDK_OK;
}

afdk_status afdk_mfa_layer(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a,
                           afdk_stream stream) {
  return mfa_layer_entry(ctx, w, a, 0.0f, 0.0f, stream);
}

afdk_status afdk_mfa_layer_mtp(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a, int mtp,
                               afdk_stream stream) {
  if (mtp == 1) return mfa_layer_entry(ctx, w, a, 0.0f, 0.0f, stream);
  if (mtp != 2) { set_error("afdk_mfa_layer_mtp: mtp must be 1 or 2"); return AFDK_ERR_INVALID; }
  if (a && a->batch > 128) { set_error("afdk_mfa_layer_mtp: batch must be <= 128"); return AFDK_ERR_INVALID; }
  return mfa_layer_entry(ctx, w, a, 0.0f, 0.0f, stream, mtp);
}

afdk_status afdk_mfa_layer_fp8(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a,
                               float k_scale, float v_scale, afdk_stream stream) {
  if (!(k_scale > 0.0f) || !(v_scale > 0.0f) || !std::isfinite(k_scale) || !std::isfinite(v_scale)) {
    set_error("afdk_mfa_layer_fp8: k_scale and v_scale must be positive and finite");
    return AFDK_ERR_INVALID;
  }
  return mfa_layer_entry(ctx, w, a, k_scale, v_scale, stream);
}

afdk_status afdk_router_topk(afdk_ctx* ctx, const void* h, const void* gate_w, int T, int H, int E, int k,
                             int renormalize, float* logits, int32_t* ids, float* weights, void* xq,
                             float* xs, afdk_stream stream) {
  if (!ctx || !h || !gate_w || !ids || !weights) { set_error("afdk_router_topk: NULL argument"); return AFDK_ERR_INVALID; }
  if (E < 1 || E > afdk::moe::kMaxExperts) { set_error("afdk_router_topk: E must be in [1, 64]"); return AFDK_ERR_INVALID; }
  if (k < 1 || k > afdk::moe::kMaxTopK || k > E) { set_error("afdk_router_topk: k must be in [1, min(8, E)]"); return AFDK_ERR_INVALID; }
  if (T < 1 || H < 256 || H % 256) { set_error("afdk_router_topk: H must be a positive multiple of 256"); return AFDK_ERR_INVALID; }
  if (H > 65536) { set_error("afdk_router_topk: H must be <= 65536"); return AFDK_ERR_INVALID; }
  if (xq && !xs) { set_error("afdk_router_topk: xq requires xs"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard device_guard(ctx->c.device);
  afdk::moe::RouterArgs a{static_cast<const __nv_bfloat16*>(h), static_cast<const __nv_bfloat16*>(gate_w), T, H, E, k,
                          renormalize, logits, ids, weights, static_cast<uint8_t*>(xq), xs};
  void* ws = afdk::workspace(ctx->c, afdk::router_workspace_bytes(H, E, ctx->c.num_sms));
  if (!ws) { set_error("afdk_router_topk: workspace allocation failed"); return AFDK_ERR_CUDA; }
  const cudaError_t e = afdk::router_launch(ctx->c, a, ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_router_topk", e);
  return AFDK_OK;
}

afdk_status afdk_moe_permute(afdk_ctx* ctx, const int32_t* ids, int T, int k, int E, int32_t* offsets,
                             int32_t* perm, int32_t* inv, afdk_stream stream) {
  if (!ctx || !ids || !offsets || !perm || !inv) { set_error("afdk_moe_permute: NULL argument"); return AFDK_ERR_INVALID; }
  if (E < 1 || E > afdk::moe::kMaxExperts || k < 1 || k > afdk::moe::kMaxTopK || T < 1 || T * k > 65536) {
    set_error("afdk_moe_permute: need 1 <= E <= 64, 1 <= k <= 8, T*k <= 65536");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const size_t wbytes = afdk::align_up((size_t)afdk::moe::max_work(T, k, E) * sizeof(afdk::moe::Work), 256) + 256;
  uint8_t* ws = static_cast<uint8_t*>(afdk::workspace(c, wbytes));
  if (!ws) { set_error("afdk_moe_permute: workspace allocation failed"); return AFDK_ERR_CUDA; }
  afdk::moe::PermuteArgs a{ids, T, k, E, 0, E, 0, 0, 0, offsets, perm, inv,
                           reinterpret_cast<afdk::moe::Work*>(ws), reinterpret_cast<int*>(ws + wbytes - 256),
                           afdk::moe::kChunk};
  const cudaError_t e = afdk::permute_launch(a, static_cast<cudaStream_t>(stream), ctx->c.pdl);
  if (e != cudaSuccess) return cuda_fail("afdk_moe_permute", e);
  return AFDK_OK;
}

static bool scatter_ok(const afdk_row_scatter* sc, int T, const char* who) {
  if (!sc) return true;
  if (!sc->dst || sc->n_dst < 1 || sc->rows_per_dst < 1 || (long)sc->n_dst * sc->rows_per_dst < T) {
    set_error(std::string(who) + ": scatter needs dst[n_dst] with n_dst * rows_per_dst >= T");
    return false;
  }
  return true;
}

static afdk_status moe_ffn_entry(afdk_ctx* ctx, const afdk_moe_weights* w, const afdk_moe_args* a,
                                 const afdk_row_scatter* sc, afdk_stream stream) {
  if (!ctx || !w || !a) { set_error("afdk_moe_ffn: NULL ctx/weights/args"); return AFDK_ERR_INVALID; }
  if (w->hidden % 128 || w->inter % 128 || w->hidden < 128 || w->inter < 128) {
    set_error("afdk_moe_ffn: hidden and inter must be positive multiples of 128");
    return AFDK_ERR_INVALID;
  }
  if (w->n_experts < 1 || w->n_experts > afdk::moe::kMaxExperts || w->top_k < 1 || w->top_k > afdk::moe::kMaxTopK) {
    set_error("afdk_moe_ffn: need 1 <= n_experts <= 64 and 1 <= top_k <= 8");
    return AFDK_ERR_INVALID;
  }
  if (w->expert_lo < 0 || w->expert_hi > w->n_experts || w->expert_lo > w->expert_hi) {
    set_error("afdk_moe_ffn: expert range out of bounds");
    return AFDK_ERR_INVALID;
  }
  if (a->T < 1 || a->T * w->top_k > 65536) { set_error("afdk_moe_ffn: T out of range"); return AFDK_ERR_INVALID; }
  if (!a->xq || !a->xs || !a->ids || !a->weights || !a->out || !w->w13 || !w->s13 || !w->w2 || !w->s2) {
    set_error("afdk_moe_ffn: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const int sh_lo = a->shared_lo < 0 ? 0 : a->shared_lo;
  const int sh_hi = a->shared_hi > a->T ? a->T : a->shared_hi;
  afdk::MoeFfnArgs m{a->T, w->top_k, w->n_experts, w->hidden, w->inter, w->expert_lo, w->expert_hi,
                     w->w13, w->s13, w->w2, w->s2, static_cast<const uint8_t*>(a->xq), a->xs, a->ids,
                     a->weights, sh_lo, sh_hi, a->out};
  if (!scatter_ok(sc, a->T, "afdk_moe_ffn")) return AFDK_ERR_INVALID;
  if (sc) { m.dst = sc->dst; m.rows_per_dst = sc->rows_per_dst; }
  void* ws = afdk::workspace(c, afdk::moe_ffn_workspace_bytes(a->T, w->top_k, w->n_experts, w->hidden, w->inter));
  if (!ws) { set_error("afdk_moe_ffn: workspace allocation failed"); return AFDK_ERR_CUDA; }
  const cudaError_t e = afdk::moe_ffn_launch(c, m, ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return AFDK_ERR_CUDA;  // message set by moe_ffn_launch
  return AFDK_OK;
}

static afdk_status moe_ffn_mx_entry(afdk_ctx* ctx, const afdk_moe_mx_weights* w, const afdk_moe_mx_args* a,
                                    const afdk_row_scatter* sc, afdk_stream stream) {
  if (!ctx || !w || !a) { set_error("afdk_moe_ffn_mx: NULL ctx/weights/args"); return AFDK_ERR_INVALID; }
  if (w->hidden % 512 || w->inter % 512 || w->hidden < 512 || w->inter < 512) {
    set_error("afdk_moe_ffn_mx: hidden and inter must be positive multiples of 512");
    return AFDK_ERR_INVALID;
  }
  if (w->n_experts < 1 || w->n_experts > afdk::moe::kMaxExperts || w->top_k < 1 || w->top_k > afdk::moe::kMaxTopK) {
    set_error("afdk_moe_ffn_mx: need 1 <= n_experts <= 64 and 1 <= top_k <= 8");
    return AFDK_ERR_INVALID;
  }
  if (w->expert_lo < 0 || w->expert_hi > w->n_experts || w->expert_lo > w->expert_hi) {
    set_error("afdk_moe_ffn_mx: expert range out of bounds");
    return AFDK_ERR_INVALID;
  }
  if (a->T < 1 || a->T * w->top_k > 65536) { set_error("afdk_moe_ffn_mx: T out of range"); return AFDK_ERR_INVALID; }
  if (!a->xq || !a->xsf || !a->ids || !a->weights || !a->out || !w->w13 || !w->sf13 || !w->w2 || !w->sf2) {
    set_error("afdk_moe_ffn_mx: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const int sh_lo = a->shared_lo < 0 ? 0 : a->shared_lo;
  const int sh_hi = a->shared_hi > a->T ? a->T : a->shared_hi;
  afdk::MoeFfnMxArgs m{a->T, w->top_k, w->n_experts, w->hidden, w->inter, w->expert_lo, w->expert_hi,
                       w->w13, w->sf13, w->w2, w->sf2, static_cast<const uint8_t*>(a->xq), a->xsf, a->ids,
                       a->weights, sh_lo, sh_hi, a->out};
  if (!scatter_ok(sc, a->T, "afdk_moe_ffn_mx")) return AFDK_ERR_INVALID;
  if (sc) { m.dst = sc->dst; m.rows_per_dst = sc->rows_per_dst; }
  void* ws = afdk::workspace(c, afdk::moe_ffn_mx_workspace_bytes(a->T, w->top_k, w->n_experts, w->hidden, w->inter));
  if (!ws) { set_error("afdk_moe_ffn_mx: workspace allocation failed"); return AFDK_ERR_CUDA; }
  const cudaError_t e = afdk::moe_ffn_mx_launch(c, m, ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return AFDK_ERR_CUDA;
  return AFDK_OK;
}

afdk_status afdk_moe_ffn(afdk_ctx* ctx, const afdk_moe_weights* w, const afdk_moe_args* a, afdk_stream stream) {
  return moe_ffn_entry(ctx, w, a, nullptr, stream);
}
afdk_status afdk_moe_ffn_scatter(afdk_ctx* ctx, const afdk_moe_weights* w, const afdk_moe_args* a,
                                 const afdk_row_scatter* sc, afdk_stream stream) {
  if (!sc) { set_error("afdk_moe_ffn_scatter: NULL scatter"); return AFDK_ERR_INVALID; }
  return moe_ffn_entry(ctx, w, a, sc, stream);
}
afdk_status afdk_moe_ffn_mx(afdk_ctx* ctx, const afdk_moe_mx_weights* w, const afdk_moe_mx_args* a,
                            afdk_stream stream) {
  return moe_ffn_mx_entry(ctx, w, a, nullptr, stream);
}
afdk_status afdk_moe_ffn_mx_scatter(afdk_ctx* ctx, const afdk_moe_mx_weights* w, const afdk_moe_mx_args* a,
                                    const afdk_row_scatter* sc, afdk_stream stream) {
  if (!sc) { set_error("afdk_moe_ffn_mx_scatter: NULL scatter"); return AFDK_ERR_INVALID; }
  return moe_ffn_mx_entry(ctx, w, a, sc, stream);
}

static afdk_status moe_ffn_bf16_entry(afdk_ctx* ctx, const afdk_moe_bf16_weights* w, const afdk_moe_bf16_args* a,
                                      const afdk_row_scatter* sc, afdk_stream stream) {
  if (!ctx || !w || !a) { set_error("afdk_moe_ffn_bf16: NULL ctx/weights/args"); return AFDK_ERR_INVALID; }
  if (w->hidden % 128 || w->inter % 128 || w->hidden < 128 || w->inter < 128) {
    set_error("afdk_moe_ffn_bf16: hidden and inter must be positive multiples of 128");
    return AFDK_ERR_INVALID;
  }
  if (w->n_experts < 1 || w->n_experts > afdk::moe::kMaxExperts || w->top_k < 1 || w->top_k > afdk::moe::kMaxTopK) {
    set_error("afdk_moe_ffn_bf16: need 1 <= n_experts <= 64 and 1 <= top_k <= 8");
    return AFDK_ERR_INVALID;
  }
  if (w->expert_lo < 0 || w->expert_hi > w->n_experts || w->expert_lo > w->expert_hi) {
    set_error("afdk_moe_ffn_bf16: expert range out of bounds");
    return AFDK_ERR_INVALID;
  }
  if (a->T < 1 || a->T * w->top_k > 65536) { set_error("afdk_moe_ffn_bf16: T out of range"); return AFDK_ERR_INVALID; }
  if (!a->x || !a->ids || !a->weights || (!a->out && !sc) || !w->w13 || !w->w2) {
    set_error("afdk_moe_ffn_bf16: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  if (!scatter_ok(sc, a->T, "afdk_moe_ffn_bf16")) return AFDK_ERR_INVALID;
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  const int sh_lo = a->shared_lo < 0 ? 0 : a->shared_lo;
  const int sh_hi = a->shared_hi > a->T ? a->T : a->shared_hi;
  afdk::MoeFfnBf16Args m{a->T, w->top_k, w->n_experts, w->hidden, w->inter, w->expert_lo, w->expert_hi,
                         w->w13, w->w2, a->x, a->ids, a->weights, sh_lo, sh_hi, a->out};
  if (sc) { m.dst = sc->dst; m.rows_per_dst = sc->rows_per_dst; }
  void* ws = afdk::workspace(c, afdk::moe_ffn_bf16_workspace_bytes(a->T, w->top_k, w->n_experts, w->hidden, w->inter));
  if (!ws) { set_error("afdk_moe_ffn_bf16: workspace allocation failed"); return AFDK_ERR_CUDA; }
  if (afdk::moe_ffn_bf16_launch(c, m, ws, static_cast<cudaStream_t>(stream)) != cudaSuccess) return AFDK_ERR_CUDA;
  return AFDK_OK;
}

afdk_status afdk_moe_ffn_bf16(afdk_ctx* ctx, const afdk_moe_bf16_weights* w, const afdk_moe_bf16_args* a,
                              afdk_stream stream) {
  return moe_ffn_bf16_entry(ctx, w, a, nullptr, stream);
}
afdk_status afdk_moe_ffn_bf16_scatter(afdk_ctx* ctx, const afdk_moe_bf16_weights* w, const afdk_moe_bf16_args* a,
                                      const afdk_row_scatter* sc, afdk_stream stream) {
  if (!sc) { set_error("afdk_moe_ffn_bf16_scatter: NULL scatter"); return AFDK_ERR_INVALID; }
  return moe_ffn_bf16_entry(ctx, w, a, sc, stream);
}

static afdk_status dense_ffn_mx_entry(afdk_ctx* ctx, const afdk_dense_mx_weights* w, int T, const void* xq,
                                      const uint8_t* xsf, void* out, const afdk_row_scatter* sc, afdk_stream stream) {
  if (!ctx || !w) { set_error("afdk_dense_ffn_mx: NULL ctx/weights"); return AFDK_ERR_INVALID; }
  if (w->hidden % 512 || w->hidden < 512 || w->inter_split % 512 || w->inter_split < 512) {
    set_error("afdk_dense_ffn_mx: hidden and inter_split must be positive multiples of 512");
    return AFDK_ERR_INVALID;
  }
  if (w->n_split < 1 || w->n_split > 64) { set_error("afdk_dense_ffn_mx: n_split must be in [1, 64]"); return AFDK_ERR_INVALID; }
  if (T < 1 || T > 65536) { set_error("afdk_dense_ffn_mx: T out of range"); return AFDK_ERR_INVALID; }
  if (!xq || !xsf || (!out && !sc) || !w->w13 || !w->sf13 || !w->w2 || !w->sf2) {
    set_error("afdk_dense_ffn_mx: NULL tensor pointer");
    return AFDK_ERR_INVALID;
  }
  afdk::Ctx& c = ctx->c;
  afdk::DeviceGuard device_guard(c.device);
  afdk::DenseFfnMxArgs d{T, w->hidden, w->inter_split, w->n_split, w->w13, w->sf13, w->w2, w->sf2,
                         static_cast<const uint8_t*>(xq), xsf, out};
  if (!scatter_ok(sc, T, "afdk_dense_ffn_mx")) return AFDK_ERR_INVALID;
  if (sc) { d.dst = sc->dst; d.rows_per_dst = sc->rows_per_dst; }
  void* ws = afdk::workspace(c, afdk::dense_ffn_mx_workspace_bytes(T, w->n_split, w->hidden, w->inter_split));
  if (!ws) { set_error("afdk_dense_ffn_mx: workspace allocation failed"); return AFDK_ERR_CUDA; }
  if (afdk::dense_ffn_mx_launch(c, d, ws, static_cast<cudaStream_t>(stream)) != cudaSuccess) return AFDK_ERR_CUDA;
  return AFDK_OK;
}

afdk_status afdk_dense_ffn_mx(afdk_ctx* ctx, const afdk_dense_mx_weights* w, int T, const void* xq,
                              const uint8_t* xsf, void* out, afdk_stream stream) {
  return dense_ffn_mx_entry(ctx, w, T, xq, xsf, out, nullptr, stream);
}
afdk_status afdk_dense_ffn_mx_scatter(afdk_ctx* ctx, const afdk_dense_mx_weights* w, int T, const void* xq,
                                      const uint8_t* xsf, const afdk_row_scatter* sc, afdk_stream stream) {
  if (!sc) { set_error("afdk_dense_ffn_mx_scatter: NULL scatter"); return AFDK_ERR_INVALID; }
  return dense_ffn_mx_entry(ctx, w, T, xq, xsf, nullptr, sc, stream);
}

afdk_status afdk_quant_mx(afdk_ctx* ctx, const void* x, int T, int H, void* q, uint8_t* sf, afdk_stream stream) {
  if (!ctx || !x || !q || !sf) { set_error("afdk_quant_mx: NULL argument"); return AFDK_ERR_INVALID; }
  if (T < 0 || H <= 0 || H % 32) { set_error("afdk_quant_mx: need T >= 0 and H % 32 == 0"); return AFDK_ERR_INVALID; }
  if (T == 0) return AFDK_OK;
  afdk::DeviceGuard device_guard(ctx->c.device);
  afdk::moe::QuantMxArgs a{static_cast<const __nv_bfloat16*>(x), T, H, static_cast<uint8_t*>(q), sf};
  const cudaError_t e = afdk::quant_mx_launch(a, static_cast<cudaStream_t>(stream), ctx->c.pdl);
  if (e != cudaSuccess) return cuda_fail("afdk_quant_mx", e);
  return AFDK_OK;
}

// The handle names the whole allocation containing dev_ptr (allocators
// sub-allocate); bytes [64,72) carry dev_ptr's offset from that base.
afdk_status afdk_ipc_handle(afdk_ctx* ctx, const void* dev_ptr, void* handle72) {
  if (!ctx || !dev_ptr || !handle72) { set_error("afdk_ipc_handle: NULL argument"); return AFDK_ERR_INVALID; }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = nullptr;
  if (!range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
      set_error("afdk_ipc_handle: cuMemGetAddressRange unavailable");
      return AFDK_ERR_CUDA;
    }
    range = reinterpret_cast<RangeFn>(fn);
  }
  afdk::DeviceGuard device_guard(ctx->c.device);
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) {
    set_error("afdk_ipc_handle: pointer is not a device allocation");
    return AFDK_ERR_INVALID;
  }
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail("cudaIpcGetMemHandle", e);
  const uint64_t off = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  std::memcpy(handle72, &h, 64);
  std::memcpy(static_cast<uint8_t*>(handle72) + 64, &off, 8);
  return AFDK_OK;
}

afdk_status afdk_ipc_open(afdk_ctx* ctx, const void* handle72, void** dev_ptr) {
  if (!ctx || !handle72 || !dev_ptr) { set_error("afdk_ipc_open: NULL argument"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard device_guard(ctx->c.device);
  cudaIpcMemHandle_t h;
  uint64_t off = 0;
  std::memcpy(&h, handle72, 64);
  std::memcpy(&off, static_cast<const uint8_t*>(handle72) + 64, 8);
  void* base = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail("cudaIpcOpenMemHandle", e);
  *dev_ptr = static_cast<uint8_t*>(base) + off;
  return AFDK_OK;
}

afdk_status afdk_ipc_close(afdk_ctx* ctx, void* dev_ptr) {
  if (!ctx || !dev_ptr) { set_error("afdk_ipc_close: NULL argument"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard device_guard(ctx->c.device);
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUdeviceptr base = reinterpret_cast<CUdeviceptr>(dev_ptr);
  size_t size = 0;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
    reinterpret_cast<RangeFn>(fn)(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr));
  const cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail("cudaIpcCloseMemHandle", e);
  return AFDK_OK;
}

afdk_status afdk_copy(afdk_ctx* ctx, void* dst, const void* src, size_t bytes, afdk_stream stream) {
  if (!ctx || !dst || !src) { set_error("afdk_copy: NULL argument"); return AFDK_ERR_INVALID; }
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_copy", e);
  return AFDK_OK;
}

afdk_status afdk_signal(afdk_ctx* ctx, uint32_t* flag, uint32_t value, afdk_stream stream) {
  if (!ctx || !flag) { set_error("afdk_signal: NULL argument"); return AFDK_ERR_INVALID; }
  const cudaError_t e = afdk::exchange_signal(flag, value, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_signal (cuStreamWriteValue32)", e);
  return AFDK_OK;
}

afdk_status afdk_wait(afdk_ctx* ctx, const uint32_t* flag, uint32_t value, afdk_stream stream) {
  if (!ctx || !flag) { set_error("afdk_wait: NULL argument"); return AFDK_ERR_INVALID; }
  const cudaError_t e = afdk::exchange_wait(flag, value, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_wait (cuStreamWaitValue32)", e);
  return AFDK_OK;
}

afdk_status afdk_add_partials(afdk_ctx* ctx, const void* base, const void* const* parts_dev, int n, size_t count,
                              void* out, afdk_stream stream) {
  if (!ctx || !out || (n > 0 && !parts_dev) || n < 0) { set_error("afdk_add_partials: bad argument"); return AFDK_ERR_INVALID; }
  if (count % 8) { set_error("afdk_add_partials: count must be a multiple of 8"); return AFDK_ERR_INVALID; }
  const cudaError_t e = afdk::add_partials_launch(base, parts_dev, n, count, out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail("afdk_add_partials", e);
  return AFDK_OK;
}

}  // extern "C"
