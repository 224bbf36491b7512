// afdk_internal.h — shared host-side state of the C-ABI implementation.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>

#include "linear.cuh"
#include "moe.cuh"

namespace afdk {

constexpr int kCounterSlots = 8192;  // [0,4096) GEMM tiles, [4096,8192) attention requests

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Ctx {
  int device = 0;
  int num_sms = 0;
  int sm_major = 0, sm_minor = 0;
  EncodeTiledFn encode = nullptr;
  void* ws = nullptr;  // grow-only device workspace
  size_t ws_bytes = 0;
  int* counters = nullptr;      // zeroed arrival counters (self-resetting kernels)
  bool pdl = true;               // launch chained kernels with programmatic dependent launch
  double* rope_freq = nullptr;  // NeoX inv_freq table (host-computed in double)
  int rope_dim = 0;
  float rope_theta = 0.0f;
};

// Entry points run on the context's device and hand the caller's current
// device back on return (a process may drive several GPUs from one thread).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Shape limits of the decode kernels, checked at the C-ABI (AFDK_ERR_INVALID):
// the per-request work prefix lives in shared memory (mfa_common.cuh
// kMaxBatch) and K3 merges at most kMfaMaxSplit parts per request
// (mfa_decode.cu), which must exceed the SM count.
constexpr int kMfaMaxBatch = 2048;
// CTAs of the decode core: every SM, or AFDK_MFA_GRID (experiments)
inline int mfa_grid(const Ctx& ctx, int batch) {
  static const int env = [] { const char* e = std::getenv("AFDK_MFA_GRID"); return e ? std::atoi(e) : 0; }();
  (void)batch;
  return (env > 0 && env < ctx.num_sms) ? env : ctx.num_sms;
}
constexpr int kMfaMaxSplit = 160;

// Returns a device workspace of at least `bytes` (grows; not graph-capturable
// the first time a larger size is requested).
void* workspace(Ctx& ctx, size_t bytes);

// Tiled tensor map, innermost dimension first; strides in bytes for dims 1..
bool encode_tma(Ctx& ctx, CUtensorMap* map, CUtensorMapDataType dt, int rank, void* base,
                const uint64_t* dims, const uint64_t* strides, const uint32_t* box,
                CUtensorMapSwizzle swizzle);

void set_error(const std::string& msg);

// Raise a kernel's dynamic shared-memory limit on the CURRENT device (function
// attributes are per device and a process may drive several GPUs); cached per
// (kernel, device) under a mutex.
cudaError_t ensure_smem_attr(const void* func, size_t bytes);
template <typename... KArgs>
cudaError_t ensure_smem(void (*kernel)(KArgs...), size_t bytes) {
  return ensure_smem_attr(reinterpret_cast<const void*>(kernel), bytes);
}

// cudaLaunchKernelEx with optional programmatic stream serialization (PDL).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Same, launched as thread-block clusters of `cluster_x` CTAs (CTA pairs for
// cta_group::2 tensor-core kernels).
template <typename... KArgs, typename... Args>
cudaError_t launch_cluster_k(bool pdl, int cluster_x, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct MfaDecodeArgs {
  int batch;
  const void* q;
  const void* k_cache;
  const void* v_cache;
  int num_pages;
  const int32_t* block_table;
  int max_pages;
  const int32_t* seq_lens;
  float softmax_scale;
  void* out;
  float* lse;
  void* workspace;
  float k_scale = 1.0f, v_scale = 1.0f;  // e4m3 caches only
};
size_t mfa_decode_workspace_bytes(int batch, int num_sms);
cudaError_t mfa_decode_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream);
// e4m3 KV cache variant (mfa_decode_fp8.cu): same args, k_cache/v_cache hold
// e4m3 codes [num_pages, 64, 256] dequantised by k_scale / v_scale
cudaError_t mfa_decode_fp8_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream);
// multi-token decode, mtp = 2 (mfa_decode_mtp.cu): q/out [B, 2, 64, 256], lse [B, 2, 64]
size_t mfa_decode_mtp_workspace_bytes(int batch, int num_sms);
cudaError_t mfa_decode_mtp_launch(Ctx& ctx, const MfaDecodeArgs& a, cudaStream_t stream);

LinearPlan make_linear_plan(int m_tok, int n_out, int k);
size_t linear_workspace_bytes(const LinearPlan& p, int num_sms);
// partials of y = x . w^T into `part` (linear_workspace_bytes); reduce with a
// SlotTable epilogue or linear_store_launch.  linear_grid = CTAs the GEMM uses.
int linear_grid(const Ctx& ctx, const LinearPlan& p);
// q_up with NeoX RoPE fused into the epilogue (one whole tile per CTA; pairs
// (i, i + head_dim/2) of a head in one tile): bf16 q out, no partials.
bool linear_rope_fusable(const Ctx& ctx, const LinearPlan& p, int head_dim);
cudaError_t linear_bf16_rope_launch(Ctx& ctx, const LinearPlan& p, const void* x, const void* w,
                                    __nv_bfloat16* q_out, const float2* rope_cs, int head_dim,
                                    cudaStream_t stream);
// w_dep: the weight operand is written by a predecessor kernel (no weight
// prefetch before the PDL wait)
cudaError_t linear_bf16_launch(Ctx& ctx, const LinearPlan& p, const void* x, const void* w, float* part,
                               cudaStream_t stream, bool w_dep = false);
// MXFP8 linear (linear_mx.cu): 128-element k-blocks, the same partial layout
LinearPlan make_linear_mx_plan(int m_tok, int n_out, int k);
cudaError_t linear_mx_launch(Ctx& ctx, const LinearPlan& p, const void* xq, const uint8_t* xsf, const void* wq,
                             const uint8_t* wsf, float* part, cudaStream_t stream, bool w_dep = false);
cudaError_t linear_store_launch(Ctx& ctx, const LinearPlan& p, const float* part, void* out, bool out_fp32,
                                cudaStream_t stream);

struct MfaLayerArgs {
  int batch, hidden, q_lora, n_heads, head_dim, page_size;
  const void *w_in_norm, *w_qkv, *w_q_norm, *w_q_up, *w_o, *w_post_norm;
  float rms_eps, rope_theta, softmax_scale;
  const void* x;
  void* k_cache;
  void* v_cache;
  int num_pages;
  const int32_t* block_table;
  int max_pages;
  const int32_t* seq_lens;
  void* h_res;
  void* h_norm;
  float k_scale = 0.0f, v_scale = 0.0f;  // > 0: e4m3 KV cache (mfa_decode_fp8.cu)
  int mtp = 1;  // query tokens per request: rows are (request, token), batch*mtp of them
  const void* w_o_mx = nullptr;     // optional MXFP8 o_proj weights (e4m3 [hidden, NQ]) ...
  const uint8_t* w_o_sf = nullptr;  // ... and their UE8M0 scales [hidden, NQ/32]
  const void* w_qup_mx = nullptr;     // optional MXFP8 q_up weights (e4m3 [NQ, q_lora]) ...
  const uint8_t* w_qup_sf = nullptr;  // ... and their UE8M0 scales [NQ, q_lora/32]
};
const double* rope_inv_freq(Ctx& ctx, int head_dim, float theta);
size_t mfa_layer_workspace_bytes(const MfaLayerArgs& a, int num_sms);
cudaError_t mfa_layer_launch(Ctx& ctx, const MfaLayerArgs& a, void* ws, cudaStream_t stream);

// ---------------------------------------------------------------- MoE FFN
size_t router_workspace_bytes(int H, int E, int num_sms);
cudaError_t router_launch(Ctx& ctx, const moe::RouterArgs& a, void* ws, cudaStream_t stream);
cudaError_t permute_launch(const moe::PermuteArgs& a, cudaStream_t stream, bool pdl);
cudaError_t gather_launch(const moe::GatherArgs& a, cudaStream_t stream, bool pdl);
cudaError_t combine_launch(const moe::CombineArgs& a, cudaStream_t stream, bool pdl);

struct MoeGemmArgs {
  const void* w;         // e4m3 [(n_local+1) * w_rows, K]
  const float* w_scale;  // [(n_local+1)][w_rows/128][K/128]
  const void* x;         // e4m3 [rows_pad, K] dispatch-ordered rows
  const float* xs_t;     // [K/128][rows_pad]
  const moe::Work* work;
  const int* n_work;
  int H, I, E, expert_lo, n_local, rows_pad;
  uint8_t* hq;           // GLU outputs
  float* hs_t;
  float* y;              // W2 output
};
cudaError_t moe_gemm_launch(Ctx& ctx, bool glu, const MoeGemmArgs& a, cudaStream_t stream);

struct MoeFfnArgs {
  int T, k, E, H, I;
  int expert_lo, expert_hi;
  const void* w13;
  const float* s13;
  const void* w2;
  const float* s2;
  const uint8_t* xq;
  const float* xs;
  const int32_t* ids;
  const float* weights;
  int shared_lo, shared_hi;
  void* out;
  const uint64_t* dst = nullptr;  // fused F->A return (CombineArgs::dst)
  int rows_per_dst = 0;
};
size_t moe_ffn_workspace_bytes(int T, int k, int E, int H, int I);
cudaError_t moe_ffn_launch(Ctx& ctx, const MoeFfnArgs& a, void* ws, cudaStream_t stream);

// MXFP8 path (hardware block-scaled MMA; moe_gemm_mx.cu)
cudaError_t quant_mx_launch(const moe::QuantMxArgs& a, cudaStream_t stream, bool pdl);
struct MoeGemmMxArgs {
  const void* w;         // e4m3 [(n_local+1) * w_rows, K]
  const uint8_t* w_sf;   // UE8M0 [(n_local+1) * w_rows, K/32]
  const void* x;         // e4m3 [rows_pad, K]
  const uint8_t* x_sf;   // UE8M0 [rows_pad, K/32]
  const moe::Work* work;
  const int* n_work;
  int H, I, E, expert_lo, n_local, rows_pad;
  uint8_t* hq;           // W13 outputs [rows_pad, I] + [rows_pad, I/32]
  uint8_t* hsf;
  float* y;              // W2 output [rows_pad, H]
  int chunk = 0;         // rows per work item (pair kernels: > 256 selects the two-accumulator form)
};
// decode-batch MoE: gate|up + down GEMMs in one persistent launch (dynamic
// item queue in sched[0], per-chunk gate|up completion counters in sched[1..])
cudaError_t moe_ffn_mx_fused_launch(Ctx& ctx, const MoeGemmMxArgs& g13, const MoeGemmMxArgs& g2, int* sched,
                                    cudaStream_t stream);
cudaError_t moe_gemm_mx_launch(Ctx& ctx, bool glu, const MoeGemmMxArgs& a, cudaStream_t stream);
cudaError_t moe_gemm_mx2_launch(Ctx& ctx, bool glu, const MoeGemmMxArgs& a, cudaStream_t stream);
// CTA-pair kernels once experts see enough rows (AFDK_MX_PAIR=0/1 forces)
bool moe_mx_use_pair(int T, int k, int E);
// rows per pair work item: 384 (two accumulators) when routed experts average
// 200-352 rows, else 256 (AFDK_MX_CHUNK=256/384 forces)
int moe_mx_pair_chunk(int T, int k, int E);
struct MoeFfnMxArgs {
  int T, k, E, H, I;
  int expert_lo, expert_hi;
  const void* w13;
  const uint8_t* sf13;
  const void* w2;
  const uint8_t* sf2;
  const uint8_t* xq;
  const uint8_t* xsf;
  const int32_t* ids;
  const float* weights;
  int shared_lo, shared_hi;
  void* out;
  const uint64_t* dst = nullptr;
  int rows_per_dst = 0;
};
size_t moe_ffn_mx_workspace_bytes(int T, int k, int E, int H, int I);
cudaError_t moe_ffn_mx_launch(Ctx& ctx, const MoeFfnMxArgs& a, void* ws, cudaStream_t stream);

// 16-bit experts (moe_gemm_bf16.cu, moe_ffn.cu): bf16 dispatch rows, bf16
// weights, bf16 SwiGLU intermediate, fp32 W2 outputs
struct MoeGemmBf16Args {
  const void* w;         // bf16 [(n_local+1) * w_rows, K]
  const void* x;         // bf16 [rows_pad, K]
  const moe::Work* work;
  const int* n_work;
  int H, I, E, expert_lo, n_local, rows_pad;
  __nv_bfloat16* h;      // W13 output [rows_pad, I]
  float* y;              // W2 output [rows_pad, H]
  int chunk = 128;       // token rows per work item (128 or 256)
};
cudaError_t moe_gemm_bf16_launch(Ctx& ctx, bool glu, const MoeGemmBf16Args& a, cudaStream_t stream);
struct MoeFfnBf16Args {
  int T, k, E, H, I;
  int expert_lo, expert_hi;
  const void* w13;
  const void* w2;
  const void* x;         // bf16 [T, H]
  const int32_t* ids;
  const float* weights;
  int shared_lo, shared_hi;
  void* out;
  const uint64_t* dst = nullptr;
  int rows_per_dst = 0;
};
size_t moe_ffn_bf16_workspace_bytes(int T, int k, int E, int H, int I);
cudaError_t moe_ffn_bf16_launch(Ctx& ctx, const MoeFfnBf16Args& a, void* ws, cudaStream_t stream);

// Dense FFN as n_split slices of the intermediate dimension ("virtual
// experts" every token visits with weight 1), MXFP8 (moe_ffn.cu)
struct DenseFfnMxArgs {
  int T, H, Is, n_split;  // Is = inter / n_split
  const void* w13;        // [n_split, 2*Is, H]
  const uint8_t* sf13;
  const void* w2;         // [n_split, H, Is]
  const uint8_t* sf2;
  const uint8_t* xq;      // [T, H]
  const uint8_t* xsf;     // [T, H/32]
  void* out;              // bf16 [T, H]
  const uint64_t* dst = nullptr;  // fused return (see moe::CombineArgs::dst)
  int rows_per_dst = 0;
};
size_t dense_ffn_mx_workspace_bytes(int T, int n_split, int H, int Is);
cudaError_t dense_ffn_mx_launch(Ctx& ctx, const DenseFfnMxArgs& a, void* ws, cudaStream_t stream);

// ---------------------------------------------------------- AFD exchange
bool exchange_available();
cudaError_t exchange_signal(uint32_t* flag, uint32_t value, cudaStream_t s);
cudaError_t exchange_wait(const uint32_t* flag, uint32_t value, cudaStream_t s);
cudaError_t add_partials_launch(const void* base, const void* const* parts_dev, int n, size_t count, void* out,
                                cudaStream_t s);

}  // namespace afdk
