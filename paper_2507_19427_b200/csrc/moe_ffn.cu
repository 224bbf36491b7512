// moe_ffn.cu — host orchestration of the FFN side of one Step-3 MoE layer:
// K6 permute -> dispatch gather -> K7 W13 (+SwiGLU +FP8 requant) -> K8 W2 ->
// K9 combine into this rank's bf16 partial (the attention side
// reduces EP partials of several FFN ranks).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "afdk_internal.h"
#include "moe.cuh"
#include "sm100.cuh"

namespace afdk {

size_t moe_ffn_workspace_bytes(int T, int k, int E, int H, int I) {
  const int rp = moe::rows_pad(T, k);
  size_t b = 0;
  b += align_up((size_t)(E + 1) * 4, 256);                       // offsets
  b += 2 * align_up((size_t)T * k * 4, 256);                     // perm, inv
  b += align_up((size_t)moe::max_work(T, k, E) * sizeof(moe::Work), 256);
  b += 256;                                                       // n_work
  b += align_up((size_t)rp * H, 256);                            // xp
  b += align_up((size_t)(H / 128) * rp * 4, 256);                // xs_t
  b += align_up((size_t)rp * I, 256);                            // hq
  b += align_up((size_t)(I / 128) * rp * 4, 256);                // hs_t
  b += align_up((size_t)rp * H * 4, 256);                        // y
  return b;
}

cudaError_t moe_ffn_launch(Ctx& ctx, const MoeFfnArgs& a, void* ws_base, cudaStream_t stream) {
  const int T = a.T, k = a.k, E = a.E, H = a.H, I = a.I;
  const int rp = moe::rows_pad(T, k);
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* offsets = static_cast<int32_t*>(take((size_t)(E + 1) * 4));
  auto* perm = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* inv = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* work = static_cast<moe::Work*>(take((size_t)moe::max_work(T, k, E) * sizeof(moe::Work)));
  auto* n_work = static_cast<int*>(take(256));
  auto* xp = static_cast<uint8_t*>(take((size_t)rp * H));
  auto* xs_t = static_cast<float*>(take((size_t)(H / 128) * rp * 4));
  auto* hq = static_cast<uint8_t*>(take((size_t)rp * I));
  auto* hs_t = static_cast<float*>(take((size_t)(I / 128) * rp * 4));
  auto* y = static_cast<float*>(take((size_t)rp * H * 4));
  const bool shared_local = a.shared_hi > a.shared_lo;
  cudaError_t e;
  // AFDK_DEBUG_SYNC=1: synchronise after every launch and name the failing kernel
  static const bool dbg = std::getenv("AFDK_DEBUG_SYNC") != nullptr;
  auto chk = [&](cudaError_t err, const char* what) {
    if (err == cudaSuccess && dbg) err = cudaStreamSynchronize(stream);
    if (err != cudaSuccess) set_error(std::string("moe_ffn/") + what + ": " + cudaGetErrorString(err));
    return err;
  };

  moe::PermuteArgs pa{a.ids, T, k, E, a.expert_lo, a.expert_hi, shared_local ? 1 : 0, a.shared_lo, a.shared_hi,
                      offsets, perm, inv, work, n_work, moe::kChunk};
  if ((e = chk(permute_launch(pa, stream, ctx.pdl), "permute")) != cudaSuccess) return e;
  moe::GatherArgs ga{a.xq, a.xs, perm, T, k, H, rp, xp, xs_t, nullptr, nullptr};
  if ((e = chk(gather_launch(ga, stream, ctx.pdl), "gather")) != cudaSuccess) return e;
  const int n_local = a.expert_hi - a.expert_lo;
  MoeGemmArgs g13{a.w13, a.s13, xp, xs_t, work, n_work, H, I, E, a.expert_lo, n_local, rp, hq, hs_t, nullptr};
  if ((e = chk(moe_gemm_launch(ctx, true, g13, stream), "gemm13")) != cudaSuccess) return e;
  MoeGemmArgs g2{a.w2, a.s2, hq, hs_t, work, n_work, H, I, E, a.expert_lo, n_local, rp, nullptr, nullptr, y};
  if ((e = chk(moe_gemm_launch(ctx, false, g2, stream), "gemm2")) != cudaSuccess) return e;
  moe::CombineArgs ca{y, a.ids, a.weights, inv, T, k, H, a.expert_lo, a.expert_hi, shared_local ? 1 : 0,
                      a.shared_lo, a.shared_hi, static_cast<__nv_bfloat16*>(a.out), a.dst, a.rows_per_dst};
  return chk(combine_launch(ca, stream, ctx.pdl), "combine");
}

// MXFP8 variant: same K6 -> gather -> K7 -> K8 -> K9 chain, operands with
// one UE8M0 scale per 32 elements, GEMMs on the block-scaled tensor-core path.
size_t moe_ffn_mx_workspace_bytes(int T, int k, int E, int H, int I) {
  const int rp = moe::rows_pad_mx(T, k);
  size_t b = 0;
  b += align_up((size_t)(E + 1) * 4, 256);
  b += 2 * align_up((size_t)T * k * 4, 256);
  b += align_up((size_t)moe::max_work(T, k, E) * sizeof(moe::Work), 256);
  b += 256;
  b += align_up((size_t)rp * H, 256);       // xp
  b += align_up((size_t)rp * (H / 32), 256);  // xsf_p
  b += align_up((size_t)rp * I, 256);       // hq
  b += align_up((size_t)rp * (I / 32), 256);  // hsf
  b += align_up((size_t)rp * H * 4, 256);   // y
  b += align_up((size_t)(1 + moe::max_work(T, k, E)) * 4, 256);  // fused kernel's queue
  return b;
}

// decode batches: gate|up and down GEMMs in one launch with a dynamic item
// queue (moe_ffn_mx_fused.cu); AFDK_MX_FUSED=0 runs the two launches
static bool moe_mx_fused() {
  static const bool on = [] { const char* e = std::getenv("AFDK_MX_FUSED"); return !(e && e[0] == '0'); }();
  return on;
}

bool moe_mx_use_pair(int T, int k, int E) {
  const char* env = std::getenv("AFDK_MX_PAIR");
  if (env && env[0] == '0') return false;
  if (env && env[0] == '1') return true;
  // >= 32 rows per routed expert on average (Step-3, MoE layer ms single / pair:
  // T=384 1.052 / 1.070, T=512 1.134 / 1.063, T=1024 1.356 / 1.169)
  return (long)T * k >= 32L * E;
}

int moe_mx_pair_chunk(int T, int k, int E) {
  if (const char* env = std::getenv("AFDK_MX_CHUNK")) return std::atoi(env) > moe::kChunkMX2 ? moe::kChunkMX2Two : moe::kChunkMX2;
  const long avg = (long)T * k / E;
  return (avg > 200 && avg <= 352) ? moe::kChunkMX2Two : moe::kChunkMX2;
}

cudaError_t moe_ffn_mx_launch(Ctx& ctx, const MoeFfnMxArgs& a, void* ws_base, cudaStream_t stream) {
  const int T = a.T, k = a.k, E = a.E, H = a.H, I = a.I;
  const int rp = moe::rows_pad_mx(T, k);
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* offsets = static_cast<int32_t*>(take((size_t)(E + 1) * 4));
  auto* perm = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* inv = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* work = static_cast<moe::Work*>(take((size_t)moe::max_work(T, k, E) * sizeof(moe::Work)));
  auto* n_work = static_cast<int*>(take(256));
  auto* xp = static_cast<uint8_t*>(take((size_t)rp * H));
  auto* xsf_p = static_cast<uint8_t*>(take((size_t)rp * (H / 32)));
  auto* hq = static_cast<uint8_t*>(take((size_t)rp * I));
  auto* hsf = static_cast<uint8_t*>(take((size_t)rp * (I / 32)));
  auto* y = static_cast<float*>(take((size_t)rp * H * 4));
  auto* sched = static_cast<int*>(take((size_t)(1 + moe::max_work(T, k, E)) * 4));
  const bool shared_local = a.shared_hi > a.shared_lo;
  const bool pair = moe_mx_use_pair(T, k, E);
  const bool fused = !pair && moe_mx_fused();
  const int chunk = pair ? moe_mx_pair_chunk(T, k, E) : moe::kChunkMX;
  auto gemm = pair ? moe_gemm_mx2_launch : moe_gemm_mx_launch;
  cudaError_t e;
  static const bool dbg = std::getenv("AFDK_DEBUG_SYNC") != nullptr;
  auto chk = [&](cudaError_t err, const char* what) {
    if (err == cudaSuccess && dbg) err = cudaStreamSynchronize(stream);
    if (err != cudaSuccess) set_error(std::string("moe_ffn_mx/") + what + ": " + cudaGetErrorString(err));
    return err;
  };
  moe::PermuteArgs pa{a.ids, T, k, E, a.expert_lo, a.expert_hi, shared_local ? 1 : 0, a.shared_lo, a.shared_hi,
                      offsets, perm, inv, work, n_work, chunk};
  if (fused) {
    pa.sched = sched;
    pa.sched_len = 1 + moe::max_work(T, k, E);
  }
  if ((e = chk(permute_launch(pa, stream, ctx.pdl), "permute")) != cudaSuccess) return e;
  moe::GatherArgs ga{a.xq, nullptr, perm, T, k, H, rp, xp, nullptr, a.xsf, xsf_p};
  if ((e = chk(gather_launch(ga, stream, ctx.pdl), "gather")) != cudaSuccess) return e;
  const int n_local = a.expert_hi - a.expert_lo;
  MoeGemmMxArgs g13{a.w13, a.sf13, xp, xsf_p, work, n_work, H, I, E, a.expert_lo, n_local, rp, hq, hsf, nullptr,
                    chunk};
  MoeGemmMxArgs g2{a.w2, a.sf2, hq, hsf, work, n_work, H, I, E, a.expert_lo, n_local, rp, nullptr, nullptr, y, chunk};
  if (fused) {
    if ((e = chk(moe_ffn_mx_fused_launch(ctx, g13, g2, sched, stream), "gemm13+2")) != cudaSuccess) return e;
  } else {
    if ((e = chk(gemm(ctx, true, g13, stream), "gemm13")) != cudaSuccess) return e;
    if ((e = chk(gemm(ctx, false, g2, stream), "gemm2")) != cudaSuccess) return e;
  }
  moe::CombineArgs ca{y, a.ids, a.weights, inv, T, k, H, a.expert_lo, a.expert_hi, shared_local ? 1 : 0,
                      a.shared_lo, a.shared_hi, static_cast<__nv_bfloat16*>(a.out), a.dst, a.rows_per_dst};
  return chk(combine_launch(ca, stream, ctx.pdl), "combine");
}

// 16-bit variant (QuantScheme with 2-byte FFN weights, types.hpp:34-40):
// bf16 dispatch rows gathered as 2H-byte rows, bf16 grouped GEMMs, the same
// permute / combine and partial semantics.
// 256-row items once routed experts average >= 128 rows (AFDK_BF16_CHUNK=128/256 forces)
static int moe_bf16_chunk(int T, int k, int E) {
  if (const char* env = std::getenv("AFDK_BF16_CHUNK")) return std::atoi(env) > 128 ? 256 : 128;
  return (long)T * k >= 128L * E ? 256 : 128;
}
static int rows_pad_bf16(int T, int k, int E) { return moe::rows_pad(T, k) + moe_bf16_chunk(T, k, E); }

size_t moe_ffn_bf16_workspace_bytes(int T, int k, int E, int H, int I) {
  const int rp = rows_pad_bf16(T, k, E);
  size_t b = 0;
  b += align_up((size_t)(E + 1) * 4, 256);
  b += 2 * align_up((size_t)T * k * 4, 256);
  b += align_up((size_t)moe::max_work(T, k, E) * sizeof(moe::Work), 256);
  b += 256;
  b += align_up((size_t)rp * H * 2, 256);  // xp
  b += align_up((size_t)rp * I * 2, 256);  // h
  b += align_up((size_t)rp * H * 4, 256);  // y
  return b;
}

cudaError_t moe_ffn_bf16_launch(Ctx& ctx, const MoeFfnBf16Args& a, void* ws_base, cudaStream_t stream) {
  const int T = a.T, k = a.k, E = a.E, H = a.H, I = a.I;
  const int rp = rows_pad_bf16(T, k, E);
  const int chunk = moe_bf16_chunk(T, k, E);
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* offsets = static_cast<int32_t*>(take((size_t)(E + 1) * 4));
  auto* perm = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* inv = static_cast<int32_t*>(take((size_t)T * k * 4));
  auto* work = static_cast<moe::Work*>(take((size_t)moe::max_work(T, k, E) * sizeof(moe::Work)));
  auto* n_work = static_cast<int*>(take(256));
  auto* xp = static_cast<uint8_t*>(take((size_t)rp * H * 2));
  auto* h = static_cast<__nv_bfloat16*>(take((size_t)rp * I * 2));
  auto* y = static_cast<float*>(take((size_t)rp * H * 4));
  const bool shared_local = a.shared_hi > a.shared_lo;
  cudaError_t e;
  static const bool dbg = std::getenv("AFDK_DEBUG_SYNC") != nullptr;
  auto chk = [&](cudaError_t err, const char* what) {
    if (err == cudaSuccess && dbg) err = cudaStreamSynchronize(stream);
    if (err != cudaSuccess) set_error(std::string("moe_ffn_bf16/") + what + ": " + cudaGetErrorString(err));
    return err;
  };
  moe::PermuteArgs pa{a.ids, T, k, E, a.expert_lo, a.expert_hi, shared_local ? 1 : 0, a.shared_lo, a.shared_hi,
                      offsets, perm, inv, work, n_work, chunk};
  if ((e = chk(permute_launch(pa, stream, ctx.pdl), "permute")) != cudaSuccess) return e;
  // rows of 2H bytes, no scales
  moe::GatherArgs ga{static_cast<const uint8_t*>(a.x), nullptr, perm, T, k, 2 * H, rp, xp, nullptr, nullptr, nullptr};
  if ((e = chk(gather_launch(ga, stream, ctx.pdl), "gather")) != cudaSuccess) return e;
  const int n_local = a.expert_hi - a.expert_lo;
  MoeGemmBf16Args g13{a.w13, xp, work, n_work, H, I, E, a.expert_lo, n_local, rp, h, nullptr, chunk};
  if ((e = chk(moe_gemm_bf16_launch(ctx, true, g13, stream), "gemm13")) != cudaSuccess) return e;
  MoeGemmBf16Args g2{a.w2, h, work, n_work, H, I, E, a.expert_lo, n_local, rp, nullptr, y, chunk};
  if ((e = chk(moe_gemm_bf16_launch(ctx, false, g2, stream), "gemm2")) != cudaSuccess) return e;
  moe::CombineArgs ca{y, a.ids, a.weights, inv, T, k, H, a.expert_lo, a.expert_hi, shared_local ? 1 : 0,
                      a.shared_lo, a.shared_hi, static_cast<__nv_bfloat16*>(a.out), a.dst, a.rows_per_dst};
  return chk(combine_launch(ca, stream, ctx.pdl), "combine");
}

// ------------------------------------------------------------- dense FFN
// The 5 dense Step-3 layers (inter 18432, builtin_catalog.cpp:248-250) run
// through the grouped MXFP8 GEMMs: slice j of the intermediate dimension is a
// "virtual expert" over ALL tokens (item rows come straight from the input,
// xrow0 = token row; intermediate / output rows at j*T + token), and the
// combine sums the slices in fixed order.  Slices held by different FFN GPUs
// give tensor-parallel partials reduced on the attention side like EP ones.
namespace moe {

__global__ void dense_work_kernel(int T, int n_split, int chunk, Work* work, int* n_work, int* sched, int sched_len) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  if (sched)  // the fused kernel's queue head and per-chunk counters
    for (int i = threadIdx.x; i < sched_len; i += blockDim.x) sched[i] = 0;
  if (threadIdx.x != 0) return;
  const int n_items = (T + chunk - 1) / chunk;
  const int per = ((T + n_items - 1) / n_items + 31) & ~31;
  int g = 0;
  for (int j = 0; j < n_split; ++j) {
    const int first = g;
    for (int r = 0; r < T; r += per) {
      work[g].group = j;
      work[g].row0 = j * T + r;
      work[g].rows = min(per, T - r);
      work[g].xrow0 = r;
      work[g].gfirst = first;
      work[g].gcnt = (T + per - 1) / per;
      ++g;
    }
  }
  *n_work = g;
}

__global__ void __launch_bounds__(256) dense_combine_kernel(const float* y, int T, int n_split, int H,
                                                            __nv_bfloat16* out, const uint64_t* dst, int rows_per_dst) {
  sm100::griddep_wait();
  sm100::griddep_launch();
  const int t = blockIdx.x;
  // fused TP return: row t straight into the attention GPU that owns it
  __nv_bfloat16* orow = dst ? reinterpret_cast<__nv_bfloat16*>(__ldg(dst + t / rows_per_dst)) +
                                  (size_t)(t % rows_per_dst) * H
                            : out + (size_t)t * H;
  for (int f = threadIdx.x * 4; f < H; f += blockDim.x * 4) {
    float4 acc = __ldcg(reinterpret_cast<const float4*>(y + (size_t)t * H + f));
    for (int j = 1; j < n_split; ++j) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(y + ((size_t)j * T + t) * H + f));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __nv_bfloat162 o0 = __floats2bfloat162_rn(acc.x, acc.y), o1 = __floats2bfloat162_rn(acc.z, acc.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&o0);
    o.y = *reinterpret_cast<uint32_t*>(&o1);
    *reinterpret_cast<uint2*>(orow + f) = o;
  }
}

}  // namespace moe

static inline int dense_rows_pad(int T, int n_split) { return ((n_split * T + 127) / 128) * 128 + moe::kChunkMX2; }
static inline int dense_max_work(int T, int n_split) { return n_split * (T / 32 + 2); }

size_t dense_ffn_mx_workspace_bytes(int T, int n_split, int H, int Is) {
  const int rp = dense_rows_pad(T, n_split);
  size_t b = align_up((size_t)dense_max_work(T, n_split) * sizeof(moe::Work), 256) + 256;
  b += align_up((size_t)rp * Is, 256);         // hq
  b += align_up((size_t)rp * (Is / 32), 256);  // hsf
  b += align_up((size_t)rp * H * 4, 256);      // y
  b += align_up((size_t)(1 + dense_max_work(T, n_split)) * 4, 256);  // fused kernel's queue
  return b;
}

// dense layers at small decode batches through the fused single-CTA kernel
// instead of the CTA-pair GEMMs (AFDK_DENSE_FUSED=1 / 0 forces).  ms fused /
// pair, best n_split: T=64 0.095 / 0.191, T=128 0.109 / 0.155, T=256 0.169 /
// 0.112 (every weight tile then serves two 128-row chunks: the pair's 256-row
// items win)
static bool dense_use_fused(int T) {
  if (const char* e = std::getenv("AFDK_DENSE_FUSED")) return e[0] == '1';
  return T < 192;
}

cudaError_t dense_ffn_mx_launch(Ctx& ctx, const DenseFfnMxArgs& a, void* ws_base, cudaStream_t stream) {
  const int rp = dense_rows_pad(a.T, a.n_split);
  uint8_t* ws = static_cast<uint8_t*>(ws_base);
  auto take = [&](size_t bytes) { void* p = ws; ws += align_up(bytes, 256); return p; };
  auto* work = static_cast<moe::Work*>(take((size_t)dense_max_work(a.T, a.n_split) * sizeof(moe::Work)));
  auto* n_work = static_cast<int*>(take(256));
  auto* hq = static_cast<uint8_t*>(take((size_t)rp * a.Is));
  auto* hsf = static_cast<uint8_t*>(take((size_t)rp * (a.Is / 32)));
  auto* y = static_cast<float*>(take((size_t)rp * a.H * 4));
  auto* sched = static_cast<int*>(take((size_t)(1 + dense_max_work(a.T, a.n_split)) * 4));
  const bool fused = dense_use_fused(a.T);
  const bool pair = !fused && moe_mx_use_pair(a.T, 1, 1);
  auto gemm = pair ? moe_gemm_mx2_launch : moe_gemm_mx_launch;
  static const bool dbg = std::getenv("AFDK_DEBUG_SYNC") != nullptr;
  auto chk = [&](cudaError_t err, const char* what) {
    if (err == cudaSuccess && dbg) err = cudaStreamSynchronize(stream);
    if (err != cudaSuccess) set_error(std::string("dense_ffn_mx/") + what + ": " + cudaGetErrorString(err));
    return err;
  };
  cudaError_t e;
  const int sched_len = 1 + dense_max_work(a.T, a.n_split);
  if ((e = chk(launch_k(ctx.pdl, moe::dense_work_kernel, dim3(1), dim3(32), 0, stream, a.T, a.n_split,
                        pair ? moe::kChunkMX2 : moe::kChunkMX, work, n_work, fused ? sched : nullptr, sched_len),
               "work")) != cudaSuccess)
    return e;
  // group j < E = n_split always: weight index j, never the shared slot
  MoeGemmMxArgs g13{a.w13, a.sf13, a.xq, a.xsf, work, n_work, a.H, a.Is, a.n_split, 0, a.n_split, a.T, hq, hsf,
                    nullptr};
  MoeGemmMxArgs g2{a.w2, a.sf2, hq, hsf, work, n_work, a.H, a.Is, a.n_split, 0, a.n_split, rp, nullptr, nullptr, y};
  if (fused) {
    if ((e = chk(moe_ffn_mx_fused_launch(ctx, g13, g2, sched, stream), "gemm13+2")) != cudaSuccess) return e;
  } else {
    if ((e = chk(gemm(ctx, true, g13, stream), "gemm13")) != cudaSuccess) return e;
    if ((e = chk(gemm(ctx, false, g2, stream), "gemm2")) != cudaSuccess) return e;
  }
  return chk(launch_k(ctx.pdl, moe::dense_combine_kernel, dim3(a.T), dim3(256), 0, stream, (const float*)y, a.T,
                      a.n_split, a.H, static_cast<__nv_bfloat16*>(a.out), a.dst, a.rows_per_dst),
             "combine");
}

}  // namespace afdk
