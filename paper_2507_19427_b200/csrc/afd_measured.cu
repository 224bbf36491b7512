// afd_measured.cu — measure_stage_times: the reference's per-layer stage
// times (pipesim.cpp:59-127) produced by running the B200 kernels instead of
// the roofline formulas.  Synthetic weights/caches of the Step-3 shapes are
// generated on the device; timings are CUDA-event averages after warm-up.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/afd_b200.hpp"
#include "afdk_internal.h"

namespace afd {
namespace b200 {

namespace {

constexpr int kQLora = 2048, kHeads = 64, kHeadDim = 256, kPage = 64;
constexpr int kExperts = 48, kTopK = 3, kInter = 5120, kDenseInter = 18432;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// kind 0: bf16 ~ U(-1,1)*scale + offset; kind 1: finite e4m3 codes
__global__ void fill_kernel(void* p, size_t n, uint64_t seed, int kind, float scale, float offset) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t r = mix(seed * 0x9e3779b97f4a7c15ull + i);
    if (kind == 0) {
      const float u = (float)(r >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;
      static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(u * scale + offset);
    } else {
      static_cast<uint8_t*>(p)[i] = (uint8_t)(0x18 + (r % 0x28)) | (uint8_t)((r >> 8) & 0x80);
    }
  }
}

__global__ void fill_f32_kernel(float* p, size_t n, float v) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void iota_pages_kernel(int32_t* bt, int n, int pages_per_req, int rot) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bt[i] = (int)(((long long)i * rot) % n);  // scattered page ids (rot coprime with n)
}

// routing: token t -> experts (t*7 + j*17) % E, distinct for E=48
__global__ void route_kernel(int32_t* ids, float* w, int T, int k, int E) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T * k; i += gridDim.x * blockDim.x) {
    const int t = i / k, j = i % k;
    ids[i] = (t * 7 + j * 17) % E;
    w[i] = 1.0f / k;
  }
}

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t n) {
    if (cudaMalloc(&p, n ? n : 1) != cudaSuccess) throw Error("measure_stage_times: cudaMalloc failed");
  }
  ~DevBuf() { if (p) cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T> T* as() const { return static_cast<T*>(p); }
};

void fill(DevBuf& b, size_t n, uint64_t seed, int kind, float scale = 1.0f, float offset = 0.0f) {
  fill_kernel<<<592, 256>>>(b.p, n, seed, kind, scale, offset);
}

template <class F>
double time_it(F&& f, int warmup = 2, int iters = 5) {
  for (int i = 0; i < warmup; ++i) f();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, nullptr);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b, nullptr);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(std::string("measure_stage_times: ") + cudaGetErrorString(e));
  return ms * 1e-3 / iters;
}

void ok(afdk_status s) { ops::check(s); }

double attention_layer_s(afdk_ctx* ctx, int hidden, int64_t batch, int64_t ctx_len, int ffn_format, bool kv8) {
  const int64_t chunks = (batch + 511) / 512;  // afdk_mfa_layer takes up to 512 requests per call
  const int B = (int)((batch + chunks - 1) / chunks);
  const int pages_per = (int)((ctx_len + kPage - 1) / kPage);
  const int n_pages = B * pages_per;
  DevBuf in_norm(hidden * 2), qkv((size_t)(kQLora + 2 * kHeadDim) * hidden * 2), q_norm(kQLora * 2),
      q_up((size_t)kHeads * kHeadDim * kQLora * 2), wo((size_t)hidden * kHeads * kHeadDim * 2), post(hidden * 2),
      gate((size_t)kExperts * hidden * 2);
  fill(in_norm, hidden, 1, 0, 0.1f, 1.0f);
  fill(qkv, (size_t)(kQLora + 2 * kHeadDim) * hidden, 2, 0, 1.0f / std::sqrt((float)hidden));
  fill(q_norm, kQLora, 3, 0, 0.1f, 1.0f);
  fill(q_up, (size_t)kHeads * kHeadDim * kQLora, 4, 0, 1.0f / std::sqrt((float)kQLora));
  fill(wo, (size_t)hidden * kHeads * kHeadDim, 5, 0, 1.0f / 128.0f);
  fill(post, hidden, 6, 0, 0.1f, 1.0f);
  fill(gate, (size_t)kExperts * hidden, 7, 0, 1.0f / std::sqrt((float)hidden));
  const size_t kv_elems = (size_t)n_pages * kPage * kHeadDim;
  DevBuf kc(kv_elems * (kv8 ? 1 : 2)), vc(kv_elems * (kv8 ? 1 : 2));
  fill(kc, kv_elems, 8, kv8 ? 1 : 0);
  fill(vc, kv_elems, 9, kv8 ? 1 : 0);
  DevBuf bt((size_t)n_pages * 4), sl((size_t)B * 4);
  iota_pages_kernel<<<64, 256>>>(bt.as<int32_t>(), n_pages, pages_per, 7919);
  std::vector<int32_t> lens(B, (int32_t)ctx_len);
  cudaMemcpy(sl.p, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice);
  DevBuf x((size_t)B * hidden * 2), h_res((size_t)B * hidden * 2), h_norm((size_t)B * hidden * 2);
  fill(x, (size_t)B * hidden, 10, 0);
  DevBuf ids((size_t)B * kTopK * 4), wts((size_t)B * kTopK * 4), xq((size_t)B * hidden * 2),
      xs((size_t)B * hidden / 32 * 4);
  afdk_mfa_weights w{hidden, kQLora, kHeads, kHeadDim, in_norm.p, qkv.p, q_norm.p, q_up.p, wo.p, post.p,
                     1e-5f, 5e5f, 1.0f / 16.0f};
  afdk_mfa_layer_args a{B, x.p, kc.p, vc.p, n_pages, kPage, bt.as<int32_t>(), pages_per, sl.as<int32_t>(),
                        h_res.p, h_norm.p};
  const double t = time_it([&] {
    ok(kv8 ? afdk_mfa_layer_fp8(ctx, &w, &a, 1.0f / 64.0f, 1.0f / 64.0f, nullptr) : afdk_mfa_layer(ctx, &w, &a, nullptr));
    // router + the dispatch payload in the FFN tier's format (the AFD runtime's ATTN op)
    if (ffn_format == AFDK_FFN_FP8) {
      ok(afdk_router_topk(ctx, h_norm.p, gate.p, B, hidden, kExperts, kTopK, 0, nullptr, ids.as<int32_t>(),
                          wts.as<float>(), xq.p, xs.as<float>(), nullptr));
      return;
    }
    ok(afdk_router_topk(ctx, h_norm.p, gate.p, B, hidden, kExperts, kTopK, 0, nullptr, ids.as<int32_t>(),
                        wts.as<float>(), nullptr, nullptr, nullptr));
    if (ffn_format == AFDK_FFN_MX)
      ok(afdk_quant_mx(ctx, h_norm.p, B, hidden, xq.p, xs.as<uint8_t>(), nullptr));
    else
      ok(afdk_copy(ctx, xq.p, h_norm.p, (size_t)B * hidden * 2, nullptr));
  });
  return t * (double)chunks;
}

double ffn_layer_s(afdk_ctx* ctx, int hidden, int inter, int n_experts, int top_k, int expert_lo, int expert_hi,
                   int64_t tokens, int64_t shared_tokens, int ffn_format) {
  const int n_local = expert_hi - expert_lo;
  const int64_t chunks = (tokens * top_k + 65535) / 65536;
  const int T = (int)((tokens + chunks - 1) / chunks);
  const int sh = (int)((shared_tokens + chunks - 1) / chunks);
  const size_t w13n = (size_t)(n_local + 1) * 2 * inter * hidden, w2n = (size_t)(n_local + 1) * hidden * inter;
  DevBuf ids((size_t)T * top_k * 4), wts((size_t)T * top_k * 4), out((size_t)T * hidden * 2);
  route_kernel<<<64, 256>>>(ids.as<int32_t>(), wts.as<float>(), T, top_k, n_experts);
  if (ffn_format == AFDK_FFN_BF16) {
    DevBuf w13(w13n * 2), w2(w2n * 2), x((size_t)T * hidden * 2);
    fill(w13, w13n, 11, 0, 1.0f / std::sqrt((float)hidden));
    fill(w2, w2n, 12, 0, 1.0f / std::sqrt((float)inter));
    fill(x, (size_t)T * hidden, 13, 0);
    afdk_moe_bf16_weights w{hidden, inter, n_experts, top_k, expert_lo, expert_hi, w13.p, w2.p};
    afdk_moe_bf16_args a{T, x.p, ids.as<int32_t>(), wts.as<float>(), 0, sh, out.p};
    return time_it([&] { ok(afdk_moe_ffn_bf16(ctx, &w, &a, nullptr)); }) * (double)chunks;
  }
  DevBuf w13(w13n), w2(w2n), xq((size_t)T * hidden);
  fill(w13, w13n, 11, 1);
  fill(w2, w2n, 12, 1);
  fill(xq, (size_t)T * hidden, 13, 1);
  if (ffn_format == AFDK_FFN_MX) {  // UE8M0 2^-7 weights, 2^-6 activations (|x| ~ O(1))
    DevBuf sf13(w13n / 32), sf2(w2n / 32), xsf((size_t)T * hidden / 32);
    cudaMemset(sf13.p, 120, w13n / 32);
    cudaMemset(sf2.p, 120, w2n / 32);
    cudaMemset(xsf.p, 121, (size_t)T * hidden / 32);
    afdk_moe_mx_weights w{hidden, inter, n_experts, top_k, expert_lo, expert_hi, w13.p, sf13.as<uint8_t>(), w2.p,
                          sf2.as<uint8_t>()};
    afdk_moe_mx_args a{T, xq.p, xsf.as<uint8_t>(), ids.as<int32_t>(), wts.as<float>(), 0, sh, out.p};
    return time_it([&] { ok(afdk_moe_ffn_mx(ctx, &w, &a, nullptr)); }) * (double)chunks;
  }
  const size_t s13n = (size_t)(n_local + 1) * (2 * inter / 128) * (hidden / 128);
  const size_t s2n = (size_t)(n_local + 1) * (hidden / 128) * (inter / 128);
  DevBuf s13(s13n * 4), s2(s2n * 4), xs((size_t)T * (hidden / 128) * 4);
  fill_f32_kernel<<<64, 256>>>(s13.as<float>(), s13n, 0.5f / std::sqrt((float)hidden));
  fill_f32_kernel<<<64, 256>>>(s2.as<float>(), s2n, 0.5f / std::sqrt((float)inter));
  fill_f32_kernel<<<64, 256>>>(xs.as<float>(), (size_t)T * (hidden / 128), 0.01f);
  afdk_moe_weights w{hidden, inter, n_experts, top_k, expert_lo, expert_hi, w13.p, s13.as<float>(), w2.p,
                     s2.as<float>()};
  afdk_moe_args a{T, xq.p, xs.as<float>(), ids.as<int32_t>(), wts.as<float>(), 0, sh, out.p};
  return time_it([&] { ok(afdk_moe_ffn(ctx, &w, &a, nullptr)); }) * (double)chunks;
}

// The dense Step-3 FFN as one FFN GPU's tensor-parallel share: dense_inter /
// ffn_gpus intermediate columns (as the AFD runtime splits it) over all
// tokens, MXFP8 slices of <= 4608 columns.
double dense_layer_s(afdk_ctx* ctx, int hidden, int ffn_gpus, int64_t tokens) {
  int cols = kDenseInter / ffn_gpus / 512 * 512;
  if (cols < 512) cols = 512;
  const int n_split = (cols + 4607) / 4608;
  const int Is = (cols / n_split) / 512 * 512;
  const int T = (int)std::min<int64_t>(tokens, 65536);
  const size_t w13n = (size_t)n_split * 2 * Is * hidden, w2n = (size_t)n_split * hidden * Is;
  DevBuf w13(w13n), w2(w2n), sf13(w13n / 32), sf2(w2n / 32), xq((size_t)T * hidden), xsf((size_t)T * hidden / 32),
      out((size_t)T * hidden * 2);
  fill(w13, w13n, 21, 1);
  fill(w2, w2n, 22, 1);
  fill(xq, (size_t)T * hidden, 23, 1);
  cudaMemset(sf13.p, 120, w13n / 32);
  cudaMemset(sf2.p, 120, w2n / 32);
  cudaMemset(xsf.p, 121, (size_t)T * hidden / 32);
  afdk_dense_mx_weights w{hidden, Is, n_split, w13.p, sf13.as<uint8_t>(), w2.p, sf2.as<uint8_t>()};
  return time_it([&] { ok(afdk_dense_ffn_mx(ctx, &w, T, xq.p, xsf.as<uint8_t>(), out.p, nullptr)); }) *
         (double)((tokens + T - 1) / T);
}

// Time one peer DMA of `bytes` from a second GPU into this one (the runtime's
// pull), or return 0 when no peer-capable second GPU is visible.
double peer_copy_s(size_t bytes) {
  int n = 0, cur = 0;
  if (bytes == 0 || cudaGetDeviceCount(&n) != cudaSuccess || n < 2) return 0.0;
  cudaGetDevice(&cur);
  const int peer = cur == 0 ? 1 : 0;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, cur, peer);
  if (!can) return 0.0;
  // direct NVLink copy-engine path (the AFD runtime maps its peers): without
  // peer access the driver stages the copy through host memory (~10 GB/s)
  const cudaError_t pe = cudaDeviceEnablePeerAccess(peer, 0);
  if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else if (pe != cudaSuccess) { cudaGetLastError(); return 0.0; }
  void *src = nullptr, *dst = nullptr;
  if (cudaMalloc(&dst, bytes) != cudaSuccess) return 0.0;
  cudaSetDevice(peer);
  const cudaError_t e = cudaMalloc(&src, bytes);
  cudaSetDevice(cur);
  if (e != cudaSuccess) { cudaFree(dst); return 0.0; }
  const double t = time_it([&] { cudaMemcpyPeerAsync(dst, cur, src, peer, bytes, nullptr); }, 2, 10);
  cudaFree(dst);
  cudaSetDevice(peer);
  cudaFree(src);
  cudaSetDevice(cur);
  return t;
}

struct Key {
  int attn_gpus, ffn_gpus, hidden;
  long long mb, ctx;
  double link;
  int fmt, kv;
  bool operator<(const Key& o) const {
    return std::tie(attn_gpus, ffn_gpus, hidden, mb, ctx, link, fmt, kv) <
           std::tie(o.attn_gpus, o.ffn_gpus, o.hidden, o.mb, o.ctx, o.link, o.fmt, o.kv);
  }
};

std::mutex g_mu;
std::map<Key, afdk_layer_times> g_cache;
afdk_ctx* g_ctx = nullptr;

}  // namespace

// Core measurement shared by the C++ and C entry points.
afdk_layer_times measure_core(afdk_ctx* ctx, const afdk_stage_plan& p) {
  if (p.attn_gpus < 1 || p.ffn_gpus < 1 || p.micro_batch < 1 || p.avg_ctx < 1 || p.hidden % 256)
    throw SpecError("measure_stage_times: need attn_gpus, ffn_gpus, micro_batch, avg_ctx >= 1 and hidden % 256 == 0");
  if (p.ffn_format < AFDK_FFN_FP8 || p.ffn_format > AFDK_FFN_BF16 || (p.kv_bytes != 0 && p.kv_bytes != 1 && p.kv_bytes != 2))
    throw SpecError("measure_stage_times: ffn_format must be AFDK_FFN_* and kv_bytes 0/1/2");
  if (p.ffn_format == AFDK_FFN_MX && p.hidden % 512)
    throw SpecError("measure_stage_times: the MXFP8 FFN needs hidden % 512 == 0");
  const bool kv8 = p.kv_bytes == 1;
  const Key key{p.attn_gpus, p.ffn_gpus, p.hidden, p.micro_batch, p.avg_ctx, p.link_gbs, p.ffn_format, kv8 ? 1 : 2};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) return it->second;
  }
  afdk_layer_times r{};
  r.attn_batch = (p.micro_batch + p.attn_gpus - 1) / p.attn_gpus;
  r.ffn_tokens = p.micro_batch;
  r.local_experts = (kExperts + p.ffn_gpus - 1) / p.ffn_gpus;
  r.attn_s = attention_layer_s(ctx, p.hidden, r.attn_batch, p.avg_ctx, p.ffn_format, kv8);
  const int64_t shared = (p.micro_batch + p.ffn_gpus - 1) / p.ffn_gpus;
  r.moe_ffn_s = ffn_layer_s(ctx, p.hidden, kInter, kExperts, kTopK, 0, r.local_experts, p.micro_batch, shared,
                            p.ffn_format);
  r.dense_ffn_s = dense_layer_s(ctx, p.hidden, p.ffn_gpus, p.micro_batch);
  // A->F per token: the dispatch row in the FFN format + its scales + top-k
  // (int32 id, fp32 weight); every attention GPU sends its tokens to every FFN
  // GPU (PAPER.md:654 broadcast).  F->A: the bf16 partial row.
  const double row = p.ffn_format == AFDK_FFN_BF16 ? 2.0 * p.hidden : (double)p.hidden;
  const double scales = p.ffn_format == AFDK_FFN_FP8 ? (p.hidden / 128) * 4.0
                        : p.ffn_format == AFDK_FFN_MX ? p.hidden / 32.0 : 0.0;
  const double tok_fwd = row + scales + kTopK * 8.0;
  const double tok_bwd = 2.0 * p.hidden;
  const double fwd = std::max((double)r.ffn_tokens * tok_fwd, (double)r.attn_batch * tok_fwd * p.ffn_gpus);
  const double bwd = std::max((double)r.ffn_tokens * tok_bwd, (double)r.attn_batch * tok_bwd * p.ffn_gpus);
  r.link_measured = 0;
  if (p.link_gbs > 0.0) {
    r.link_gbs = p.link_gbs;
    r.comm_fwd_s = fwd / (p.link_gbs * 1e9);
    r.comm_bwd_s = bwd / (p.link_gbs * 1e9);
  } else {
    const double tf = peer_copy_s((size_t)fwd), tb = peer_copy_s((size_t)bwd);
    if (tf > 0.0 && tb > 0.0) {  // the plan's actual payloads as real peer DMAs
      r.link_measured = 1;
      r.comm_fwd_s = tf;
      r.comm_bwd_s = tb;
      r.link_gbs = (fwd + bwd) / (tf + tb) / 1e9;
    } else {
      r.link_gbs = 770.0;  // measured peer copy on this pool (B200_PROFILING.md)
      r.comm_fwd_s = fwd / (r.link_gbs * 1e9);
      r.comm_bwd_s = bwd / (r.link_gbs * 1e9);
    }
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache[key] = r;
  return r;
}

void fill_stage_times(const afdk_layer_times& r, int L, double* attn, double* fwd, double* ffn, double* bwd) {
  for (int l = 0; l < L; ++l) {
    const bool dense = l < 4 || l == L - 1;  // builtin_catalog.cpp:248-250
    attn[l] = r.attn_s;
    fwd[l] = r.comm_fwd_s;
    ffn[l] = dense ? r.dense_ffn_s : r.moe_ffn_s;
    bwd[l] = r.comm_bwd_s;
  }
}

namespace {
int gpus_per_server(const Catalog& cat, const std::string& hw) {
  for (const auto& a : cat.accelerators)
    if (a.name == hw) return a.gpus_per_server > 0 ? a.gpus_per_server : 1;
  return 1;
}
afdk_ctx* shared_ctx() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx) {
    int dev = 0;
    cudaGetDevice(&dev);
    afdk_cfg cfg{dev, 0};
    ops::check(afdk_create(&g_ctx, &cfg));
  }
  return g_ctx;
}
afdk_stage_plan to_plan(const ModelSpec& m, const DeploymentPlan& p, const Workload& w, const Catalog& cat) {
  if (p.mode != PlanMode::afd) throw Error("stage times are defined for afd plans only");
  if (m.attention_groups.empty() || m.attention_groups[0].n_q_heads != kHeads ||
      m.attention_groups[0].qk_dim != kHeadDim || m.attention_groups[0].v_dim != kHeadDim)
    throw SpecError("measure_stage_times: model '" + m.name + "' is not MFA 64x256 (Step-3 geometry)");
  if (p.micro_batch < 1) throw SpecError("measure_stage_times: plan.micro_batch must be >= 1");
  afdk_stage_plan sp{};
  sp.attn_gpus = p.attn_instances * gpus_per_server(cat, p.attn_hw);
  sp.ffn_gpus = p.ffn_instances * gpus_per_server(cat, p.ffn_hw);
  sp.micro_batch = p.micro_batch;
  sp.avg_ctx = w.avg_ctx;
  sp.n_layers = m.n_layers;
  sp.hidden = m.hidden_dim;
  sp.link_gbs = 0.0;
  // the model card's quant scheme picks the formats (types.hpp:34-40):
  // 1-byte weights -> the block-scaled MXFP8 FFN, 2-byte -> bf16 experts;
  // kv_store_bytes 1 -> e4m3 KV cache (Step-3's 512 B/token), 2 -> bf16
  sp.ffn_format = m.quant.weight_bytes >= 2 ? AFDK_FFN_BF16 : AFDK_FFN_MX;
  sp.kv_bytes = m.quant.kv_store_bytes >= 2 ? 2 : 1;
  return sp;
}
}  // namespace

LayerMeasurement measure_layer(const ModelSpec& m, const DeploymentPlan& p, const Workload& w, const Catalog& cat) {
  const afdk_stage_plan sp = to_plan(m, p, w, cat);
  const afdk_layer_times r = measure_core(shared_ctx(), sp);
  LayerMeasurement out;
  out.attn_s = r.attn_s;
  out.moe_ffn_s = r.moe_ffn_s;
  out.dense_ffn_s = r.dense_ffn_s;
  out.comm_fwd_s = r.comm_fwd_s;
  out.comm_bwd_s = r.comm_bwd_s;
  out.attn_batch = r.attn_batch;
  out.ffn_tokens = r.ffn_tokens;
  out.local_experts = r.local_experts;
  out.link_gbs = r.link_gbs;
  out.link_source = r.link_measured ? "measured peer DMA of the payload" : "pool peer-copy figure 770 GB/s";
  return out;
}

void clear_measurement_cache() {
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache.clear();
}

}  // namespace b200

StageTimes measure_stage_times(const ModelSpec& model, const DeploymentPlan& plan, const Workload& w,
                               const Catalog& catalog) {
  const afdk_stage_plan sp = b200::to_plan(model, plan, w, catalog);
  const afdk_layer_times r = b200::measure_core(b200::shared_ctx(), sp);
  const int L = model.n_layers;
  StageTimes st;
  st.attn.resize(L);
  st.comm_fwd.resize(L);
  st.ffn.resize(L);
  st.comm_bwd.resize(L);
  b200::fill_stage_times(r, L, st.attn.data(), st.comm_fwd.data(), st.ffn.data(), st.comm_bwd.data());
  return st;
}

}  // namespace afd

extern "C" afdk_status afdk_measure_stage_times(afdk_ctx* ctx, const afdk_stage_plan* plan, double* attn,
                                                double* comm_fwd, double* ffn, double* comm_bwd,
                                                afdk_layer_times* detail) {
  if (!ctx || !plan || !attn || !comm_fwd || !ffn || !comm_bwd || plan->n_layers < 1) {
    afdk::set_error("afdk_measure_stage_times: NULL argument or n_layers < 1");
    return AFDK_ERR_INVALID;
  }
  try {
    const afdk_layer_times r = afd::b200::measure_core(ctx, *plan);
    afd::b200::fill_stage_times(r, plan->n_layers, attn, comm_fwd, ffn, comm_bwd);
    if (detail) *detail = r;
    return AFDK_OK;
  } catch (const afd::SpecError& e) {
    afdk::set_error(e.what());
    return AFDK_ERR_INVALID;
  } catch (const std::exception& e) {
    afdk::set_error(e.what());
    return AFDK_ERR_CUDA;
  }
}
