/*
 * afd_oracle.h — CPU fp32 restatement of the Step-3 decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2507_19427_b200/,
 * include/) links, imports or calls this code; only tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() use it, and
 * only as the checker.
 *
 * Provenance and pinning:
 *   * The reference (/root/reference/proj, "afdsim") implements the *accounting*
 *     of this path, not its numerics.  The accounting is pinned by
 *     compiling the reference itself into oracle/_ref/libafdref.so (Makefile)
 *     and comparing these functions' byte/FLOP counts with its
 *     cost_breakdown()/ffn_net_bytes()/derive_stage_times()
 *     (costmodel.cpp:46-79, moeplan.cpp:17-20, pipesim.cpp:59-127).
 *   * Numerics: parity UNPINNED by the reference (it has no numeric kernels,
 *     SURVEY.md §8c).  Semantics follow the paper (PAPER.md:93-95 MFA
 *     structure, :649 router on the attention side, :654-655 FP8 dispatch /
 *     BF16 combine) and the public Step-3 decoder code shipped in this image
 *     (vllm/model_executor/models/step3_text.py: qkv_proj -> inter_norm -> wq
 *     -> neox RoPE -> attention(scale=head_dim^-0.5) -> o_proj; RMSNorm eps
 *     1e-5, rope_theta 5e5, softmax router with norm_expert_weight=False,
 *     SiLU-and-mul experts; configs/step3_vl.py defaults).  The restatement
 *     is cross-checked against an independent numpy implementation on the
 *     golden fixtures under tests/golden/ (tests/golden/make_golden.py).
 *
 * Conventions: row-major, all activations/weights passed as float (callers
 * widen bf16 / dequantize fp8 exactly), dot products accumulate in double.
 * Functions that model a GPU storage point take `round_bf16`: when non-zero
 * the result is rounded to bf16 (RNE) exactly where the B200 path stores bf16.
 */
#ifndef AFD_ORACLE_H
#define AFD_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- scalar formats ---------------------------------------------------- */
float orc_bf16_round(float x);              /* fp32 -> bf16 (RNE) -> fp32   */
uint16_t orc_f32_to_bf16_bits(float x);
float orc_bf16_bits_to_f32(uint16_t b);
uint8_t orc_f32_to_e4m3(float x);           /* RNE, saturate to +-448, NaN->0x7f */
float orc_e4m3_to_f32(uint8_t v);

/* ---- elementwise / linear ---------------------------------------------- */
/* out[r,:] = x[r,:] * rsqrt(mean(x[r,:]^2) + eps) * w  (step3_text.py RMSNorm) */
void orc_rmsnorm(const float* x, const float* w, int rows, int dim, float eps,
                 int round_bf16, float* out);
/* out[m,n] = sum_k x[m,k] * W[n,k]  (nn.Linear, weight [N,K]) */
void orc_linear(const float* x, const float* W, int M, int N, int K,
                int round_bf16, float* out);
/* NeoX-style rotary on n_vec vectors of length dim at position pos:
 * pairs (i, i+dim/2), inv_freq_i = theta^(-2i/dim). In place. */
void orc_rope_neox(float* x, int n_vec, int dim, int pos, float theta, int round_bf16);

/* ---- MFA decode attention core (K2/K3) ---------------------------------- */
/* q        [B, H, D]
 * k_cache  [num_pages, page, D], v_cache same; token t of request b lives in
 *          page block_table[b*max_pages + t/page], slot t%page
 * seq_lens [B]  (0 allowed: output zeros, lse = -inf)
 * out      [B, H, D];  lse [B, H] natural-log log-sum-exp of scaled scores
 * Exact two-pass softmax in double. Op counts equal group_core_flops
 * (costmodel.cpp:26-44): 2*H*(D+D)*ctx per request. */
void orc_mfa_decode_attention(const float* q, const float* k_cache, const float* v_cache,
                              const int32_t* block_table, int max_pages,
                              const int32_t* seq_lens, int B, int H, int D, int page,
                              float scale, int round_bf16, float* out, float* lse);

/* ---- full attention-side decode layer (K1 + K2 + K4 + post-norm) -------- */
typedef struct {
  int hidden, q_lora, n_heads, head_dim, page;
  float rms_eps, rope_theta, softmax_scale;
  /* e4m3 KV cache (0 = off): the caches hold DEQUANTISED values
   * e4m3(code)*scale; the appended token is stored as e4m3(x/scale) (x the
   * bf16-rounded post-RoPE k / v), and the query of every (request, head) is
   * quantised with a power-of-two scale (orc_quant_pow2, block = head_dim)
   * before the exact attention. */
  float kv_k_scale, kv_v_scale;
  /* o_mx != 0: the o_proj input (the attention output) is MXFP8-quantised
   * (orc_quant_mx) and dequantised before o_proj, as afdk_mfa_layer with
   * MXFP8 o_proj weights does (the caller passes the dequantised weights). */
  int o_mx;
  /* qup_mx != 0: likewise for the q_up input (the q-RMSNorm output). */
  int qup_mx;
} orc_mfa_dims;

/* x          [B, hidden]              layer input (residual stream)
 * w_in_norm  [hidden]
 * w_qkv      [q_lora + 2*head_dim, hidden]  rows: q_down | k | v
 * w_q_norm   [q_lora]
 * w_q_up     [n_heads*head_dim, q_lora]
 * w_o        [hidden, n_heads*head_dim]
 * w_post_norm[hidden]
 * k_cache/v_cache updated in place: the new token (position seq_lens[b]-1)
 * is written at its slot before attention reads the cache.
 * h_res  [B, hidden] = x + o_proj(attn)    (residual after attention)
 * h_norm [B, hidden] = RMSNorm(h_res)      (FFN input, pre-dispatch)      */
void orc_mfa_layer(const orc_mfa_dims* d, int B, const float* x,
                   const float* w_in_norm, const float* w_qkv, const float* w_q_norm,
                   const float* w_q_up, const float* w_o, const float* w_post_norm,
                   float* k_cache, float* v_cache, const int32_t* block_table,
                   int max_pages, const int32_t* seq_lens, int round_bf16,
                   float* h_res, float* h_norm);

/* ---- router / dispatch metadata (K5/K6) --------------------------------- */
/* logits [T,E] -> top-k ids/weights. Selection on logits, descending, ties to
 * the lower expert index; weights = softmax(logits)[id] (fp32, max-subtracted,
 * sum in index order); renormalize!=0 divides by the top-k sum. */
void orc_router_topk(const float* logits, int T, int E, int k, int renormalize,
                     int32_t* ids, float* weights);
/* Stable expert-major permutation: slot order (expert, token, j).
 * offsets [E+1] exclusive prefix of counts; perm [T*k] slot -> t*k+j;
 * inv [T*k] t*k+j -> slot. */
void orc_moe_permute(const int32_t* ids, int T, int k, int E, int32_t* offsets,
                     int32_t* perm, int32_t* inv);

/* ---- FP8 block quantization (A->F dispatch payload, K5 epilogue) -------- */
/* per row, per `block` contiguous elements: scale = max(amax,1e-10)/448,
 * q = e4m3_rne_sat(x / scale)  (IEEE fp32 division) */
void orc_quant_fp8_rowblock(const float* x, int rows, int cols, int block,
                            uint8_t* q, float* scales);
/* weight block quantization with [bm x bk] tiles (128x128 for experts) */
void orc_quant_fp8_tile(const float* w, int rows, int cols, int bm, int bk,
                        uint8_t* q, float* scales);

/* ---- MoE expert FFN (K7/K8) --------------------------------------------- */
/* One gated expert on `rows` dispatched tokens.
 * xq [rows, H] e4m3 + xs [rows, H/128]
 * w13 [2I, H] e4m3 (rows 0..I-1 gate, I..2I-1 up) + s13 [2I/128, H/128]
 * w2  [H, I]  e4m3 + s2 [H/128, I/128]
 * y [rows, H] fp32.  The SiLU(gate)*up intermediate is re-quantized to
 * e4m3 with 1x128 row blocks exactly as the B200 path does before W2. */
void orc_expert_ffn_fp8(const uint8_t* xq, const float* xs, int rows, int H, int I,
                        const uint8_t* w13, const float* s13,
                        const uint8_t* w2, const float* s2, float* y);

/* Whole MoE layer on T tokens: routed experts (ids/weights [T,k]) + one
 * shared expert (index E in the weight arrays, applied to every token).
 * w13_all [(E+1), 2I, H], s13_all [(E+1), 2I/128, H/128],
 * w2_all [(E+1), H, I], s2_all [(E+1), H/128, I/128].
 * out [T, H] = sum_j w_j * y_{ids_j}(t) + y_shared(t)   (fp32; round_bf16
 * applies the bf16 combine of PAPER.md:654). */
void orc_moe_layer_fp8(const uint8_t* xq, const float* xs, int T, int H, int I, int E,
                       int k, const int32_t* ids, const float* weights,
                       const uint8_t* w13_all, const float* s13_all,
                       const uint8_t* w2_all, const float* s2_all, int round_bf16,
                       float* out);

/* ---- MXFP8 (OCP MX, e4m3 elements + one UE8M0 scale per 32) ----------- */
/* Tensor-core block-scaled format used by the large-batch expert GEMMs.
 * Per 32-element block: e = smallest integer with amax <= 448 * 2^e
 * (amax == 0 -> e = -127), clamped to [-127, 127]; sf = e + 127 (UE8M0);
 * q = e4m3_rn_satfinite(x * 2^-e) (exact power-of-two scaling). */
int orc_mx_exponent(float amax);
void orc_quant_mx(const float* x, int rows, int cols, uint8_t* q, uint8_t* sf);
/* The same power-of-two rule over `block` contiguous elements: e per block
 * (orc_mx_exponent of the block amax), q = e4m3_rn_satfinite(x * 2^-e).
 * Used for the FP8-KV attention query (block = head_dim). */
void orc_quant_pow2(const float* x, int rows, int cols, int block, uint8_t* q, int32_t* e);
float orc_mx_scale(uint8_t sf); /* 2^(sf-127) */
/* One gated expert, all operands MXFP8: xq [rows,H] + xsf [rows,H/32],
 * w13 [2I,H] + sf13 [2I,H/32], w2 [H,I] + sf2 [H,I/32]; the SiLU(gate)*up
 * intermediate is re-quantised to MXFP8 before W2. y [rows,H] fp32. */
/* 16-bit (bf16) / unquantised fp32 gated expert and routed layer
 * (types.hpp:34-40,93-95; step3_text.py Step3TextMLP + SiluAndMul). */
void orc_expert_ffn_f32(const float* x, int rows, int H, int I, const float* w13,
                        const float* w2, int round_bf16, float* y);
void orc_moe_layer_f32(const float* x, int T, int H, int I, int E, int k, const int32_t* ids,
                       const float* weights, const float* w13_all, const float* w2_all,
                       int round_bf16, float* out);
void orc_expert_ffn_mx(const uint8_t* xq, const uint8_t* xsf, int rows, int H, int I,
                       const uint8_t* w13, const uint8_t* sf13, const uint8_t* w2,
                       const uint8_t* sf2, float* y);
/* Whole MoE layer in MXFP8 (weights of E routed + 1 shared expert stacked). */
void orc_moe_layer_mx(const uint8_t* xq, const uint8_t* xsf, int T, int H, int I, int E, int k,
                      const int32_t* ids, const float* weights, const uint8_t* w13_all,
                      const uint8_t* sf13_all, const uint8_t* w2_all, const uint8_t* sf2_all,
                      int round_bf16, float* out);

/* ---- accounting (must equal the reference's analytic model) ------------- */
/* attention-core FLOPs of one decode step for one request at ctx tokens */
double orc_mfa_core_flops(int n_heads, int head_dim, int64_t ctx);
/* KV bytes streamed by the core for one request (K and V, elt bytes each) */
double orc_mfa_kv_bytes(int head_dim, int64_t ctx, int elt_bytes);
/* parameters of the MFA projections (q_down, q_up, k, v, o) */
int64_t orc_mfa_linear_params(int hidden, int q_lora, int n_heads, int head_dim);
/* MoE FLOPs per token for (k routed + n_shared) gated experts */
double orc_moe_flops_per_token(int hidden, int inter, int k, int n_shared);
/* A->F + F->A bytes for T tokens (fp8 payload, bf16 return; scales and
 * routing metadata reported separately by orc_dispatch_meta_bytes) */
double orc_afd_wire_bytes(int hidden, int64_t T);
double orc_dispatch_meta_bytes(int hidden, int k, int64_t T);

/* threads used by the OpenMP-parallel oracle routines (1 if built without) */
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif /* AFD_ORACLE_H */
