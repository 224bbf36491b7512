// moe_ffn.cu — host orchestration of the FFN side of one Step-3 MoE layer:
// K6 permute -> dispatch gather -> K7 W13 (+SwiGLU +FP8 requant) -> K8 W2 ->
// K9 combine into this rank's bf16 partial (the attention side
// reduces EP partials of several FFN ranks).
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "afdk_internal.h"
#include "moe.cuh"

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
                      a.shared_lo, a.shared_hi, static_cast<__nv_bfloat16*>(a.out)};
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
  return b;
}

bool moe_mx_use_pair(int T, int k, int E) {
  const char* env = std::getenv("AFDK_MX_PAIR");
  if (env && env[0] == '0') return false;
  if (env && env[0] == '1') return true;
  return (long)T * k >= 64L * E;  // >= 64 rows per routed expert on average
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
  const bool shared_local = a.shared_hi > a.shared_lo;
  const bool pair = moe_mx_use_pair(T, k, E);
  auto gemm = pair ? moe_gemm_mx2_launch : moe_gemm_mx_launch;
  cudaError_t e;
  static const bool dbg = std::getenv("AFDK_DEBUG_SYNC") != nullptr;
  auto chk = [&](cudaError_t err, const char* what) {
    if (err == cudaSuccess && dbg) err = cudaStreamSynchronize(stream);
    if (err != cudaSuccess) set_error(std::string("moe_ffn_mx/") + what + ": " + cudaGetErrorString(err));
    return err;
  };
  moe::PermuteArgs pa{a.ids, T, k, E, a.expert_lo, a.expert_hi, shared_local ? 1 : 0, a.shared_lo, a.shared_hi,
                      offsets, perm, inv, work, n_work, pair ? moe::kChunkMX2 : moe::kChunkMX};
  if ((e = chk(permute_launch(pa, stream, ctx.pdl), "permute")) != cudaSuccess) return e;
  moe::GatherArgs ga{a.xq, nullptr, perm, T, k, H, rp, xp, nullptr, a.xsf, xsf_p};
  if ((e = chk(gather_launch(ga, stream, ctx.pdl), "gather")) != cudaSuccess) return e;
  const int n_local = a.expert_hi - a.expert_lo;
  MoeGemmMxArgs g13{a.w13, a.sf13, xp, xsf_p, work, n_work, H, I, E, a.expert_lo, n_local, rp, hq, hsf, nullptr};
  if ((e = chk(gemm(ctx, true, g13, stream), "gemm13")) != cudaSuccess) return e;
  MoeGemmMxArgs g2{a.w2, a.sf2, hq, hsf, work, n_work, H, I, E, a.expert_lo, n_local, rp, nullptr, nullptr, y};
  if ((e = chk(gemm(ctx, false, g2, stream), "gemm2")) != cudaSuccess) return e;
  moe::CombineArgs ca{y, a.ids, a.weights, inv, T, k, H, a.expert_lo, a.expert_hi, shared_local ? 1 : 0,
                      a.shared_lo, a.shared_hi, static_cast<__nv_bfloat16*>(a.out)};
  return chk(combine_launch(ca, stream, ctx.pdl), "combine");
}

}  // namespace afdk
