/*
 * afdk.h — C-ABI of the B200-native Step-3 decode hot path.
 *
 * This is the drop-in boundary below the reference's C++ operator API
 * (/root/reference/proj/include/afdsim/*.hpp).  The reference *accounts* for
 * each operation analytically; every entry point here *executes* the
 * operation it accounts for, on an sm_100a GPU:
 *
 *   afdk_mfa_decode_attention   executes what kv_state_bytes / attn_core_flops
 *                               account for           (costmodel.cpp:10-58)
 *   afdk_mfa_layer              + attn_linear_flops    (costmodel.cpp:60-66,
 *                               params builtin_catalog.cpp:243-247)
 *   afdk_router_topk, afdk_quant_fp8, afdk_moe_permute,
 *   afdk_moe_ffn                what ffn_flops accounts for (costmodel.cpp:68-74,
 *                               params builtin_catalog.cpp:248-251)
 *   afdk_exchange_*             what ffn_net_bytes accounts for (moeplan.cpp:17-20)
 *   afdk_stage_times            the measured counterpart of derive_stage_times
 *                               (pipesim.cpp:59-127, pipesim.hpp:28-29)
 *
 * Conventions: plain pointers and sizes only.  Device
 * pointers are caller-owned and never freed here; the opaque afdk_ctx owns
 * workspaces and tensor-map state.  Every call returns an afdk_status; the
 * message of the last failure on the calling thread is afdk_last_error().
 * A context is used from one host thread at a time; work is enqueued on the
 * caller's CUDA stream (afdk_stream == cudaStream_t, NULL = legacy stream)
 * and calls do not synchronise the device unless stated.  Calls are CUDA-graph
 * capturable (kernels are chained with programmatic dependent launch); the
 * context's workspace grows on demand (cudaFree + cudaMalloc, synchronising),
 * so capture after a warm-up call of the largest shape, and recapture if a
 * later call needs a larger workspace.  One context per stream in flight
 * (the MFA merge kernel also synchronises with the main kernel through
 * self-re-arming arrival counters owned by the context).
 *
 * Tensor formats: bf16 = IEEE bfloat16 (uint16 storage), e4m3 = OCP FP8
 * E4M3FN (max 448), all tensors dense row-major unless stated.
 */
#ifndef AFDK_H
#define AFDK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AFDK_ABI_VERSION 1

typedef enum afdk_status {
  AFDK_OK = 0,
  AFDK_ERR_INVALID = 1,     /* bad argument / unsupported shape (afd::SpecError) */
  AFDK_ERR_CUDA = 2,        /* CUDA runtime/driver failure                       */
  AFDK_ERR_UNSUPPORTED = 3, /* device is not sm_100 / feature not built          */
  AFDK_ERR_NO_DEVICE = 4    /* no CUDA device visible                            */
} afdk_status;

typedef struct afdk_ctx afdk_ctx;
typedef void* afdk_stream; /* cudaStream_t */

typedef struct afdk_cfg {
  int device;  /* CUDA device ordinal */
  int num_sms; /* 0 = all SMs of the device */
} afdk_cfg;

int afdk_abi_version(void);
const char* afdk_last_error(void);
afdk_status afdk_create(afdk_ctx** out, const afdk_cfg* cfg);
void afdk_destroy(afdk_ctx* ctx);
/* SMs the persistent kernels of this context are sized for */
int afdk_num_sms(const afdk_ctx* ctx);
/* the CUDA device the context was created on (-1 for NULL) */
int afdk_ctx_device(const afdk_ctx* ctx);

/* ---------------------------------------------------------------- K2 + K3
 * MFA decode attention core.  One shared K head and one shared V head of
 * head_dim serve n_heads query heads.  Supported: n_heads 64,
 * head_dim 256, page_size 64, bf16 everywhere (Step-3, configs 2 and 4).
 *   q          [batch, n_heads, head_dim] bf16 (post-RoPE)
 *   k_cache    [num_pages, page_size, head_dim] bf16, v_cache same
 *   block_table[batch, max_pages] int32 page ids, seq_lens [batch] int32
 *   out        [batch, n_heads, head_dim] bf16
 *   lse        [batch, n_heads] fp32 natural-log LSE, optional (NULL)
 * Any seq_len >= 0 (ragged); the split-KV factor is chosen internally so
 * every SM streams the same number of pages (flash-decoding).            */
typedef struct afdk_mfa_decode_args {
  int batch, n_heads, head_dim, page_size;
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
} afdk_mfa_decode_args;

afdk_status afdk_mfa_decode_attention(afdk_ctx* ctx, const afdk_mfa_decode_args* a,
                                      afdk_stream stream);

/* Same core over an e4m3 KV cache (512 B per token per layer: the
 * kv_token_bytes the reference charges Step-3, builtin_catalog.cpp:11,242;
 * the paper's FP8 attention).  k_cache / v_cache hold e4m3
 * codes [num_pages, page_size, head_dim], dequantised by the per-tensor
 * k_scale / v_scale (> 0).  q stays bf16; the kernel quantises it per
 * (request, head) with a power-of-two scale 2^e (smallest e with
 * amax <= 448*2^e) and runs Q.K^T and P.V as FP8 tensor-core MMAs (P rounded
 * to e4m3); out/lse as above.                                              */
afdk_status afdk_mfa_decode_attention_fp8(afdk_ctx* ctx, const afdk_mfa_decode_args* a, float k_scale,
                                          float v_scale, afdk_stream stream);

/* Multi-token decode (MTP, mtp in {1, 2}): the mtp newest tokens of every
 * request (positions L-mtp .. L-1, already appended) query the bf16 cache
 * together; token j attends causally to positions <= L-mtp+j.  The
 * reference's mtp multiplier on attention FLOPs with KV bytes unchanged
 * (costmodel.cpp:46-58).  q/out [batch, mtp, n_heads, head_dim] bf16,
 * lse [batch, mtp, n_heads]; a token that sees no key gives zeros / -inf.
 * mtp = 2 runs one M=128 tensor-core contraction per KV page; batch <= 128. */
afdk_status afdk_mfa_decode_attention_mtp(afdk_ctx* ctx, const afdk_mfa_decode_args* a, int mtp,
                                          afdk_stream stream);

/* ------------------------------------------------------------ K1/K4 GEMM
 * y[m, n] = x[m, k] . w[n, k]^T, bf16 inputs, fp32 accumulate, decode-shaped
 * (1 <= m <= 512, k % 64 == 0).  out is bf16 (out_fp32 = 0) or fp32.      */
afdk_status afdk_linear(afdk_ctx* ctx, const void* x, const void* w, void* out, int m, int n, int k,
                        int out_fp32, afdk_stream stream);

/* The same projection with MXFP8 operands (the paper's FP8 attention GEMMs,
 * PAPER.md:774,781): xq e4m3 [m, k] + xsf UE8M0 [m, k/32], wq e4m3 [n, k] +
 * wsf UE8M0 [n, k/32] (afdk_quant_mx's format), y = dequant(xq) .
 * dequant(wq)^T with fp32 accumulation on the block-scaled tensor-core MMA.
 * 1 <= m <= 384 (above 256 tokens: two N/2 MMAs per k-block), k % 512 == 0
 * (the k/32-byte scale rows are TMA-loaded). */
afdk_status afdk_linear_mx(afdk_ctx* ctx, const void* xq, const uint8_t* xsf, const void* wq, const uint8_t* wsf,
                           void* out, int m, int n, int k, int out_fp32, afdk_stream stream);

/* --------------------------------------------- attention-side decode layer
 * input RMSNorm -> [q_down|k|v] -> q RMSNorm -> q_up -> NeoX RoPE(q, k)
 * -> paged KV append (position seq_lens[b]-1) -> MFA decode core -> o_proj
 * + residual -> post-attention RMSNorm.  Step-3 dims: hidden 7168, q_lora
 * 2048, 64 heads x 256 (builtin_catalog.cpp:241-247).   */
typedef struct afdk_mfa_weights {
  int hidden, q_lora, n_heads, head_dim;
  const void* in_norm;   /* bf16 [hidden]                                */
  const void* w_qkv;     /* bf16 [q_lora + 2*head_dim, hidden] q|k|v rows */
  const void* q_norm;    /* bf16 [q_lora]                                */
  const void* w_q_up;    /* bf16 [n_heads*head_dim, q_lora]              */
  const void* w_o;       /* bf16 [hidden, n_heads*head_dim]              */
  const void* post_norm; /* bf16 [hidden]                                */
  float rms_eps, rope_theta, softmax_scale;
  /* optional (NULL = bf16 w_o): o_proj as an MXFP8 GEMM (afdk_linear_mx) —
   * e4m3 [hidden, n_heads*head_dim] + UE8M0 [hidden, n_heads*head_dim/32];
   * the attention output is MXFP8-quantised on the way in.  batch <= 384. */
  const void* w_o_mx;
  const uint8_t* w_o_sf;
  /* optional (NULL = bf16 w_q_up): q_up as an MXFP8 GEMM — e4m3
   * [n_heads*head_dim, q_lora] + UE8M0 [n_heads*head_dim, q_lora/32]; the
   * q-RMSNorm output is MXFP8-quantised on the way in.  batch <= 384,
   * q_lora % 512 == 0 (the scale rows are TMA-loaded: 16-byte multiples). */
  const void* w_q_up_mx;
  const uint8_t* w_q_up_sf;
} afdk_mfa_weights;

typedef struct afdk_mfa_layer_args {
  int batch;
  const void* x;   /* bf16 [batch, hidden] layer input (residual stream)  */
  void* k_cache;   /* bf16 [num_pages, page_size, head_dim], appended     */
  void* v_cache;
  int num_pages, page_size;
  const int32_t* block_table; /* [batch, max_pages]                       */
  int max_pages;
  const int32_t* seq_lens;    /* [batch] lengths INCLUDING the new token  */
  void* h_res;     /* bf16 [batch, hidden] x + attention output           */
  void* h_norm;    /* bf16 [batch, hidden] RMSNorm(h_res): FFN input      */
} afdk_mfa_layer_args;

afdk_status afdk_mfa_layer(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a,
                           afdk_stream stream);

/* The same layer over e4m3 KV caches (see afdk_mfa_decode_attention_fp8):
 * the appended token is stored as e4m3_rn_satfinite(bf16(k_rope)/k_scale),
 * e4m3_rn_satfinite(bf16(v)/v_scale); the core runs on the FP8 path.      */
afdk_status afdk_mfa_layer_fp8(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a,
                               float k_scale, float v_scale, afdk_stream stream);

/* MTP decode layer (mtp in {1, 2}): every request carries its mtp newest
 * tokens (positions L-mtp .. L-1, L = seq_lens[b] counts them).  x, h_res and
 * h_norm have batch*mtp rows ordered (request, token); the projections run on
 * all rows, each row appends its K/V at its own position, and the core is
 * afdk_mfa_decode_attention_mtp (causal among the new tokens).
 * batch*mtp <= 256, batch <= 128 for mtp = 2 (afdk_mfa_layer[_fp8]: batch
 * <= 512; above 256 rows the projections run as two N/2 MMAs per weight k-block). */
afdk_status afdk_mfa_layer_mtp(afdk_ctx* ctx, const afdk_mfa_weights* w, const afdk_mfa_layer_args* a, int mtp,
                               afdk_stream stream);

/* ------------------------------------------------ K5 router + FP8 dispatch
 * Attention-side router: logits = h . gate_w^T (fp32), softmax,
 * top-k by logit (ties -> lower expert id), weights = softmax probability
 * (renormalize != 0 divides by their sum).  When xq != NULL the FP8 dispatch
 * payload is produced as well: per token and 128-feature
 * block, xs = max(amax, 1e-10)/448, xq = e4m3_rn_satfinite(h / xs).
 *   h [T, H] bf16, gate_w [E, H] bf16; logits [T, E] fp32 (optional);
 *   ids [T, k] int32; weights [T, k] fp32; xq [T, H] e4m3; xs [T, H/128] fp32.
 * Limits: E <= 64, k <= 8, H % 256 == 0.                                   */
afdk_status afdk_router_topk(afdk_ctx* ctx, const void* h, const void* gate_w, int T, int H, int E, int k,
                             int renormalize, float* logits, int32_t* ids, float* weights, void* xq,
                             float* xs, afdk_stream stream);

/* ---------------------------------------------- K6 expert distribution
 * Stable expert-major permutation of the [T, k] routing: offsets [E+1]
 * (exclusive prefix of per-expert counts), perm [T*k] (slot -> t*k+j in
 * (expert, token, j) order), inv [T*k] (t*k+j -> slot).                   */
afdk_status afdk_moe_permute(afdk_ctx* ctx, const int32_t* ids, int T, int k, int E, int32_t* offsets,
                             int32_t* perm, int32_t* inv, afdk_stream stream);

/* ----------------------------------------------- K7/K8/K9 MoE FFN (FP8)
 * One MoE layer on an FFN rank: dispatched FP8 tokens in, this rank's bf16
 * partial out = sum over its routed experts [expert_lo, expert_hi) of
 * w_j * expert(x) + the shared expert for tokens [shared_lo, shared_hi).
 * Gated experts (SiLU(gate) * up, then down), e4m3 weights with 128x128
 * fp32 block scales; the intermediate is re-quantised to e4m3 with 1x128
 * scales.  Weight tensors hold the local routed experts followed by the
 * shared expert (index n_local = expert_hi - expert_lo):
 *   w13 [(n_local+1), 2*inter, hidden] (rows: gate then up),
 *   s13 [(n_local+1), 2*inter/128, hidden/128],
 *   w2  [(n_local+1), hidden, inter],  s2 [(n_local+1), hidden/128, inter/128].
 * Limits: hidden % 128 == 0, inter % 128 == 0, E <= 64, k <= 8, T*k <= 65536. */
typedef struct afdk_moe_weights {
  int hidden, inter, n_experts, top_k;
  int expert_lo, expert_hi;
  const void* w13;
  const float* s13;
  const void* w2;
  const float* s2;
} afdk_moe_weights;

typedef struct afdk_moe_args {
  int T;
  const void* xq;        /* e4m3 [T, hidden] dispatch payload        */
  const float* xs;       /* [T, hidden/128] its scales               */
  const int32_t* ids;    /* [T, top_k]                               */
  const float* weights;  /* [T, top_k]                               */
  int shared_lo, shared_hi;
  void* out;             /* bf16 [T, hidden] this rank's partial     */
} afdk_moe_args;

afdk_status afdk_moe_ffn(afdk_ctx* ctx, const afdk_moe_weights* w, const afdk_moe_args* a, afdk_stream stream);

/* ------------------------------------- K5'/K7/K8/K9 MoE FFN (MXFP8 path)
 * The large-batch variant of afdk_moe_ffn: all GEMM operands in OCP MXFP8
 * (e4m3 + one UE8M0 scale per 32 elements along K), run on the hardware
 * block-scaled tensor-core MMA.  Same routing, shared-expert and partial-sum
 * semantics as afdk_moe_ffn (replaces the same ffn_flops accounting,
 * costmodel.cpp:68-74); the SiLU(gate)*up intermediate is re-quantised to
 * MXFP8.  Scale tensors are row-major with K/32 bytes per row:
 *   sf13 [(n_local+1), 2*inter, hidden/32], sf2 [(n_local+1), hidden, inter/32].
 * Limits: hidden % 512 == 0, inter % 512 == 0, E <= 64, k <= 8, T*k <= 65536. */
typedef struct afdk_moe_mx_weights {
  int hidden, inter, n_experts, top_k;
  int expert_lo, expert_hi;
  const void* w13;
  const uint8_t* sf13;
  const void* w2;
  const uint8_t* sf2;
} afdk_moe_mx_weights;

typedef struct afdk_moe_mx_args {
  int T;
  const void* xq;        /* e4m3 [T, hidden]                         */
  const uint8_t* xsf;    /* UE8M0 [T, hidden/32]                     */
  const int32_t* ids;    /* [T, top_k]                               */
  const float* weights;  /* [T, top_k]                               */
  int shared_lo, shared_hi;
  void* out;             /* bf16 [T, hidden] this rank's partial     */
} afdk_moe_mx_args;

afdk_status afdk_moe_ffn_mx(afdk_ctx* ctx, const afdk_moe_mx_weights* w, const afdk_moe_mx_args* a,
                            afdk_stream stream);

/* ---------------------------------- K7/K8/K9 MoE FFN (16-bit experts)
 * The FFN with 2-byte weights: QuantScheme.weight_bytes = 2 /
 * compute_kind f16 (types.hpp:34-40, effective_kind types.hpp:93-95), the
 * BF16 fallback of PAPER.md:279.  Same routing, shared-expert and
 * partial-sum semantics as afdk_moe_ffn; the dispatch payload is the bf16
 * token rows (dispatch_bytes 2 instead of 1 in ffn_net_bytes,
 * moeplan.cpp:17-20), the SiLU(gate)*up intermediate is stored bf16, GEMMs on
 * tcgen05 kind::f16 with fp32 accumulation:
 *   w13 bf16 [(n_local+1), 2*inter, hidden] (rows: gate then up),
 *   w2  bf16 [(n_local+1), hidden, inter].
 * Limits: hidden % 128 == 0, inter % 128 == 0, E <= 64, k <= 8, T*k <= 65536. */
typedef struct afdk_moe_bf16_weights {
  int hidden, inter, n_experts, top_k;
  int expert_lo, expert_hi;
  const void* w13;
  const void* w2;
} afdk_moe_bf16_weights;

typedef struct afdk_moe_bf16_args {
  int T;
  const void* x;         /* bf16 [T, hidden] dispatch payload        */
  const int32_t* ids;    /* [T, top_k]                               */
  const float* weights;  /* [T, top_k]                               */
  int shared_lo, shared_hi;
  void* out;             /* bf16 [T, hidden] this rank's partial     */
} afdk_moe_bf16_args;

afdk_status afdk_moe_ffn_bf16(afdk_ctx* ctx, const afdk_moe_bf16_weights* w, const afdk_moe_bf16_args* a,
                              afdk_stream stream);

/* ------------------------------------------------ dense FFN (MXFP8)
 * The dense Step-3 layers (first four and last, inter 18432,
 * builtin_catalog.cpp:248-250): out = SiLU(x.Wg^T) * (x.Wu^T) . W2^T as a sum
 * over n_split slices of the intermediate dimension, each a grouped MXFP8
 * GEMM pair over all T tokens (the MoE kernels with every slice a "virtual
 * expert" of weight 1).  A GPU holding only some slices returns their
 * partial; the attention side reduces partials like EP ones
 * (afdk_add_partials) — the FFN-tier tensor parallelism of PAPER.md:651.
 *   w13  e4m3 [n_split, 2*inter_split, hidden]: slice j = gate rows
 *        [j*inter_split, +inter_split) then the matching up rows
 *   sf13 UE8M0 [n_split, 2*inter_split, hidden/32]
 *   w2   e4m3 [n_split, hidden, inter_split] (columns of slice j)
 *   sf2  UE8M0 [n_split, hidden, inter_split/32]
 * xq/xsf: MXFP8 input [T, hidden] (afdk_quant_mx); out bf16 [T, hidden].
 * Limits: hidden % 512 == 0, inter_split % 512 == 0, 1 <= T <= 65536.     */
typedef struct afdk_dense_mx_weights {
  int hidden, inter_split, n_split;
  const void* w13;
  const uint8_t* sf13;
  const void* w2;
  const uint8_t* sf2;
} afdk_dense_mx_weights;

afdk_status afdk_dense_ffn_mx(afdk_ctx* ctx, const afdk_dense_mx_weights* w, int T, const void* xq,
                              const uint8_t* xsf, void* out, afdk_stream stream);

/* MXFP8 quantisation of the dispatch payload: x bf16 [T, H] -> q e4m3 [T, H]
 * + sf UE8M0 [T, H/32].  Per 32 elements: e = smallest integer with
 * amax <= 448 * 2^e (e = -127 for an all-zero block), sf = e + 127,
 * q = e4m3_rn_satfinite(x * 2^-e).  H % 32 == 0. */
afdk_status afdk_quant_mx(afdk_ctx* ctx, const void* x, int T, int H, void* q, uint8_t* sf, afdk_stream stream);

/* ------------------------------------- fused F->A return over NVLink
 * The same MoE layers with the combine kernel (K9) writing every token row
 * straight into the attention GPU that owns it: row t goes to
 * dst[t / rows_per_dst] + (t % rows_per_dst) * hidden (bf16), where dst is a
 * DEVICE array of n_dst pointers, typically peer buffers opened with
 * afdk_ipc_open.  The partial crosses NVLink as the combine produces it (no
 * separate copy); order a stream-ordered afdk_signal after the call, whose
 * implied system fence publishes the rows before the flag.               */
typedef struct afdk_row_scatter {
  int n_dst, rows_per_dst;
  const uint64_t* dst;
} afdk_row_scatter;

afdk_status afdk_moe_ffn_scatter(afdk_ctx* ctx, const afdk_moe_weights* w, const afdk_moe_args* a,
                                 const afdk_row_scatter* sc, afdk_stream stream);
afdk_status afdk_moe_ffn_mx_scatter(afdk_ctx* ctx, const afdk_moe_mx_weights* w, const afdk_moe_mx_args* a,
                                    const afdk_row_scatter* sc, afdk_stream stream);
afdk_status afdk_moe_ffn_bf16_scatter(afdk_ctx* ctx, const afdk_moe_bf16_weights* w, const afdk_moe_bf16_args* a,
                                      const afdk_row_scatter* sc, afdk_stream stream);
/* dense layer, this GPU's intermediate slices (tensor-parallel partial) */
afdk_status afdk_dense_ffn_mx_scatter(afdk_ctx* ctx, const afdk_dense_mx_weights* w, int T, const void* xq,
                                      const uint8_t* xsf, const afdk_row_scatter* sc, afdk_stream stream);

/* ------------------------------------------- C1/C2 AFD exchange (NVLink)
 * Zero-SM point-to-point transport between attention and FFN GPUs of one
 * box (the StepMesh pattern of PAPER.md:701-724 on NVLink 5 / NVSwitch):
 * buffers are registered once through CUDA IPC, data moves as copy-engine
 * DMA (afdk_copy: cudaMemcpyAsync on the stream; src/dst may be peer-mapped),
 * readiness travels as monotonically increasing 32-bit sequence flags
 * (afdk_signal writes a flag word, typically on a peer, after all prior work
 * of the stream; afdk_wait blocks the stream until a local flag >= value).
 * Together they carry ffn_net_bytes = (dispatch+combine)*H*T per layer
 * (moeplan.cpp:17-20).  IPC handles are 72 opaque bytes (the allocation's
 * CUDA IPC handle + the pointer's offset inside it); afdk_ipc_close takes
 * the pointer afdk_ipc_open returned.                                      */
afdk_status afdk_ipc_handle(afdk_ctx* ctx, const void* dev_ptr, void* handle72);
afdk_status afdk_ipc_open(afdk_ctx* ctx, const void* handle72, void** dev_ptr);
afdk_status afdk_ipc_close(afdk_ctx* ctx, void* dev_ptr);
afdk_status afdk_copy(afdk_ctx* ctx, void* dst, const void* src, size_t bytes, afdk_stream stream);
afdk_status afdk_signal(afdk_ctx* ctx, uint32_t* flag, uint32_t value, afdk_stream stream);
afdk_status afdk_wait(afdk_ctx* ctx, const uint32_t* flag, uint32_t value, afdk_stream stream);
/* EP reduction on the attention side: out = base + sum_i parts[i] (bf16, fp32
 * sum in index order); parts_dev is a DEVICE array of n device pointers;
 * base may be NULL; count % 8 == 0.                                        */
afdk_status afdk_add_partials(afdk_ctx* ctx, const void* base, const void* const* parts_dev, int n, size_t count,
                              void* out, afdk_stream stream);

/* -------------------------------------- NVLS in-switch reduction groups
 * The FFN-tier reduction of PAPER.md:651,654 (EP / TP partials summed for the
 * attention side) done by the NVSwitch: n_members GPUs (one process each)
 * bind one buffer each to a multicast object; afdk_nvls_reduce_bf16 reads
 * the element-wise sum over all members' buffers through the multicast
 * address (multimem.ld_reduce, fp32 accumulation in the switch).
 *   creator (creator_pid <= 0): creates the object and returns *export_fd;
 *   the others pass the creator's pid and export_fd (exchanged through the
 *   caller's rendezvous; imported with pidfd_getfd).  Every member then calls
 *   afdk_nvls_bind (blocks until all members were created/imported): uc_ptr
 *   = this member's buffer (write your contribution), mc_ptr = the multicast
 *   view (the reduce's input).  Order contributions before the reduce with
 *   the exchange flags (afdk_signal / afdk_wait).  AFDK_ERR_UNSUPPORTED when
 *   the device or system has no NVLS.                                      */
typedef struct afdk_nvls afdk_nvls;
int afdk_nvls_supported(afdk_ctx* ctx);
afdk_status afdk_nvls_create(afdk_ctx* ctx, int n_members, size_t bytes, int creator_pid, int creator_fd,
                             afdk_nvls** out, int* export_fd);
afdk_status afdk_nvls_bind(afdk_nvls* g, void** uc_ptr, void** mc_ptr);
size_t afdk_nvls_size(const afdk_nvls* g);
void afdk_nvls_destroy(afdk_nvls* g);
afdk_status afdk_nvls_reduce_bf16(afdk_ctx* ctx, const void* mc_ptr, void* out, size_t count, afdk_stream stream);

/* --------------------------------------------- AFD pipeline runtime (C++)
 * The A -> link -> F -> link schedule of a decode layer that
 * pipesim.cpp:155-237 models (ping-pong micro-batches, PAPER.md:690-724:
 * StepMesh's pattern, here on NVLink inside one box), as a host runtime in
 * C++ behind this C-ABI.  One afdk_afd per GPU (one process per GPU):
 * attention ranks [0, n_attn) hold their requests (DP attention,
 * PAPER.md:649), FFN ranks [n_attn, n_attn+n_ffn) hold experts
 * [f*E/nF, (f+1)*E/nF) and a 1/nF share of the shared expert's tokens
 * (expert parallel; dense layers: intermediate slices, tensor parallel).
 *
 * Ownership: the runtime owns the exchange buffers (A->F payload, F->A
 * partial rows, sequence flags), the h_res/h_norm scratch, its streams (one
 * per micro-batch + one copy stream) and the peer mappings; the caller owns
 * weights, KV caches and the layer activations x (read and overwritten by
 * afdk_afd_attn_layer).
 *
 * Rendezvous: afdk_afd_create calls allgather(user, mine, bytes, all) — any
 * transport (torch.distributed, MPI, sockets) that concatenates every rank's
 * `bytes` in rank order into `all` and returns 0 on success.  It is called
 * twice (allocation status + IPC handles; then a barrier once the peers are
 * mapped).  A rank that failed to allocate makes EVERY rank's create fail
 * before any peer is mapped, instead of leaving peers waiting on flags.
 *
 * Schedule of one layer at sequence number s (afdk_afd_plan returns the op
 * list the runtime executes; host only, no GPU needed):
 *   attention rank a, micro-batch m (stream m):
 *     ATTN(m) [mfa_layer in attn_chunk pieces; router + dispatch payload]
 *     -> SIGNAL(FFN f, slot a*n_micro+m, s) for every f
 *     -> WAIT(slot f*n_micro+m, s) [+ PULL f's partial rows if f2a=pull]
 *     -> REDUCE(m) [x = h_res + sum_f partial_f]
 *   FFN rank f, micro-batch m:
 *     copy stream: WAIT(slot a*n_micro+m, s) + PULL a's payload, every a
 *     -> JOIN(m) (compute stream waits for the copy stream)
 *     -> FFN(m) [push: its combine stores rows into the attention GPUs]
 *     -> SIGNAL(attention a, slot f*n_micro+m, s) for every a
 * Flags are monotone (s = 1, 2, ...), so every cross-layer buffer reuse is
 * ordered by a flag of the next layer (a payload is rewritten only after
 * the FFN signalled that it consumed it, and so on).                      */
#define AFDK_AFD_MAX_MICRO 4
enum { AFDK_FFN_FP8 = 0, AFDK_FFN_MX = 1, AFDK_FFN_BF16 = 2 };
enum { AFDK_LAYER_MOE = 0, AFDK_LAYER_DENSE = 1 };
enum { AFDK_F2A_PUSH = 0, AFDK_F2A_PULL = 1, AFDK_F2A_NVLS = 2 };
/* f2a: PUSH — each FFN rank's combine stores its partial rows into the
 * attention rank's receive buffer over NVLink, the attention side adds them;
 * PULL — the attention rank DMA-pulls them; NVLS — each FFN rank's combine
 * writes its rows into its OWN member buffer of an NVLS group per
 * (attention rank, micro-batch) whose attention member is h_res, and the
 * attention side reads x = h_res + sum of partials with one in-switch
 * multimem.ld_reduce (afdk_nvls_*; needs >= 1 GPU per rank on an NVSwitch
 * box and pidfd_getfd permission between the ranks' processes). */

typedef struct afdk_afd_cfg {
  int n_attn, n_ffn, n_micro;  /* n_micro <= AFDK_AFD_MAX_MICRO (2 = ping-pong)        */
  int T_mb;                    /* decode requests per micro-batch per attention rank  */
  int hidden, top_k, n_experts, inter;
  int dense_inter, dense_slices;  /* dense layers: inter and slices per FFN rank      */
  int ffn_format;              /* AFDK_FFN_*                                          */
  int layer_kind;              /* AFDK_LAYER_* (dense layers: MXFP8 slices)           */
  int f2a;                     /* AFDK_F2A_*                                          */
  int attn_chunk;              /* requests per attention-layer call, 1..512           */
} afdk_afd_cfg;

enum { AFDK_OP_ATTN = 0, AFDK_OP_SIGNAL = 1, AFDK_OP_WAIT = 2, AFDK_OP_PULL = 3, AFDK_OP_REDUCE = 4,
       AFDK_OP_JOIN = 5, AFDK_OP_FFN = 6 };
enum { AFDK_BUF_SEND = 0, AFDK_BUF_RECV = 1, AFDK_BUF_RX = 2, AFDK_BUF_OUT = 3 };

typedef struct afdk_afd_op {
  int kind;        /* AFDK_OP_*                                                  */
  int stream;      /* 0..n_micro-1: micro-batch streams; n_micro: copy stream    */
  int mb;          /* micro-batch                                                */
  int peer;        /* SIGNAL target / PULL source rank, else -1                  */
  int slot;        /* flag slot (on the peer for SIGNAL, local for WAIT)         */
  uint32_t value;  /* sequence number                                            */
  int src_buf, dst_buf;            /* PULL: peer buffer kind -> local buffer kind */
  size_t src_off, dst_off, bytes;  /* PULL byte range                            */
} afdk_afd_op;

/* payload section offsets/sizes of one A->F message (xq, scales, ids, wts;
 * 256-B aligned) and of the FFN's receive buffer (n_attn messages). */
typedef struct afdk_afd_layout {
  size_t off[4], size[4], total;        /* one attention rank's payload     */
  size_t rx_off[4], rx_total;           /* FFN receive buffer (n_attn each) */
  size_t part_bytes;                    /* one T_mb x hidden bf16 partial   */
} afdk_afd_layout;

afdk_status afdk_afd_check_cfg(const afdk_afd_cfg* cfg);
afdk_status afdk_afd_get_layout(const afdk_afd_cfg* cfg, afdk_afd_layout* out);
afdk_status afdk_afd_plan(const afdk_afd_cfg* cfg, int rank, uint32_t seq, afdk_afd_op* ops, int cap,
                          int* n_ops);

typedef int (*afdk_allgather_fn)(void* user, const void* mine, size_t bytes, void* all);
typedef struct afdk_afd afdk_afd;

/* ctxs: n_micro contexts on this rank's device (each micro-batch stream uses
 * its own workspace); rank in [0, n_attn + n_ffn). */
afdk_status afdk_afd_create(afdk_ctx* const* ctxs, const afdk_afd_cfg* cfg, int rank, afdk_allgather_fn allgather,
                            void* user, afdk_afd** out);
void afdk_afd_destroy(afdk_afd* afd);

/* attention rank: one layer for every micro-batch (enqueue only) */
typedef struct afdk_afd_attn_mb {
  void* x;                  /* bf16 [T_mb, hidden] in: layer input, out: next layer input */
  void* k_cache;            /* bf16 or e4m3 (k_scale > 0) [num_pages, page, head_dim]     */
  void* v_cache;
  int num_pages, page_size, max_pages;
  const int32_t* block_table;  /* [T_mb, max_pages] */
  const int32_t* seq_lens;     /* [T_mb]            */
  float k_scale, v_scale;      /* 0: bf16 KV; > 0: e4m3 KV with these per-tensor scales   */
} afdk_afd_attn_mb;
afdk_status afdk_afd_attn_layer(afdk_afd* afd, const afdk_mfa_weights* w, const void* gate_w,
                                const afdk_afd_attn_mb* mbs);

/* FFN rank: one layer for every micro-batch.  MoE: the local routed experts
 * then the shared expert (the afdk_moe_ffn* layouts of the format); dense:
 * this rank's dense_slices intermediate slices (afdk_dense_ffn_mx layout). */
typedef struct afdk_afd_ffn_weights {
  const void* w13;
  const void* s13;  /* fp8: fp32 128x128 scales; mx: UE8M0; bf16: NULL */
  const void* w2;
  const void* s2;
} afdk_afd_ffn_weights;
afdk_status afdk_afd_ffn_layer(afdk_afd* afd, const afdk_afd_ffn_weights* w);

/* the runtime's streams (i in [0, n_micro]: micro-batch streams, then the
 * copy stream) for event timing / joins; a runtime buffer (AFDK_BUF_*, or
 * 4 = h_res, 5 = h_norm) of micro-batch mb for inspection; sequence number
 * of the last enqueued layer; block the host until every stream is idle. */
afdk_stream afdk_afd_stream(afdk_afd* afd, int i);
void* afdk_afd_buffer(afdk_afd* afd, int which, int mb);
uint32_t afdk_afd_seq(const afdk_afd* afd);
afdk_status afdk_afd_sync(afdk_afd* afd);

/* Measured trace of the layers enqueued after afdk_afd_trace_start: CUDA
 * events around every op that occupies a resource (ATTN / REDUCE ->
 * attention, FFN -> ffn, the payload pulls of one (layer, micro-batch) ->
 * fwd_link on FFN ranks, partial pulls -> bwd_link on attention ranks; with
 * f2a = push the return transfer is inside the FFN op).  afdk_afd_trace_csv
 * (host-blocking) stops tracing and writes this rank's events in the
 * reference's trace_csv schema (pipesim.cpp:239-260: time_s relative to the
 * trace start, resource, layer, micro_batch, stage, duration_s; %.9f). */
afdk_status afdk_afd_trace_start(afdk_afd* afd);
afdk_status afdk_afd_trace_csv(afdk_afd* afd, char* buf, size_t cap, size_t* len);

/* ------------------------------------------------ measured stage times
 * The measured counterpart of derive_stage_times (pipesim.cpp:59-127): runs
 * one attention-tier layer (afdk_mfa_layer[_fp8] + router/dispatch in the FFN
 * format) at ceil(micro_batch / attn_gpus) requests and avg_ctx tokens, one
 * FFN-tier MoE layer (48/ffn_gpus local experts + the shared expert's token
 * share over micro_batch tokens) and one dense FFN layer as this GPU's
 * tensor-parallel share (dense_inter/ffn_gpus intermediate columns over all
 * micro_batch tokens, the AFD runtime's split), and the NVLink transfers,
 * then fills per-layer seconds for n_layers Step-3 layers (layers 0-3 and
 * n_layers-1 dense, builtin_catalog.cpp:248-250).
 *   ffn_format: AFDK_FFN_* (QuantScheme.weight_bytes 1 -> FP8, 2 -> BF16)
 *   kv_bytes:   1 = e4m3 KV cache, 2 (or 0) = bf16 (QuantScheme.kv_store_bytes)
 *   link_gbs <= 0: when a second GPU is visible, the A->F payload and the
 *   F->A partial of this plan are each timed as a real peer DMA of their
 *   byte count; otherwise bytes / the pool's measured 770 GB/s.           */
typedef struct afdk_stage_plan {
  int attn_gpus, ffn_gpus;
  long long micro_batch;
  long long avg_ctx;
  int n_layers;
  int hidden;
  double link_gbs;
  int ffn_format;
  int kv_bytes;
} afdk_stage_plan;

typedef struct afdk_layer_times {
  double attn_s, moe_ffn_s, dense_ffn_s, comm_fwd_s, comm_bwd_s, link_gbs;
  long long attn_batch, ffn_tokens;
  int local_experts, link_measured;
} afdk_layer_times;

afdk_status afdk_measure_stage_times(afdk_ctx* ctx, const afdk_stage_plan* plan, double* attn, double* comm_fwd,
                                     double* ffn, double* comm_bwd, afdk_layer_times* detail);

/* ------------------------------------------------- pipeline model (host)
 * simulate() of pipesim.cpp:155-237 evaluated on any StageTimes (typically
 * measured ones): tpot, tgs = total_batch / (tpot * total_gpus), per-resource
 * utilisation and bubbles (attention, fwd link, ffn, bwd link).  CPU only. */
typedef struct afdk_sim_plan {
  int n_micro;
  long long total_batch;
  int total_gpus;
  int token_steps;
  int shared_link;
} afdk_sim_plan;

typedef struct afdk_sim_result {
  double tpot, tgs;
  double utilization[4];
  double bubble_fraction[4];
} afdk_sim_result;

afdk_status afdk_simulate(const double* attn, const double* comm_fwd, const double* ffn, const double* comm_bwd,
                          int layers, const afdk_sim_plan* plan, afdk_sim_result* out);

/* trace_csv of the simulated run (pipesim.cpp:239-260 schema
 * "time_s,resource,layer,micro_batch,stage,duration_s", %.9f); *len = the
 * full text length; buf (may be NULL) receives up to cap-1 bytes + NUL. */
afdk_status afdk_trace_csv(const double* attn, const double* comm_fwd, const double* ffn, const double* comm_bwd,
                           int layers, const afdk_sim_plan* plan, char* buf, size_t cap, size_t* len);

/* vet_plan's stage check (planner.cpp:124-131) on given (typically measured)
 * per-layer attention / FFN stage times: stage_ok iff every layer's attn and
 * ffn <= budget = tpot_sla / pipeline_stages / n_model_layers
 * (stage_budget, sizing.cpp:9-11).  CPU only. */
typedef struct afdk_stage_check {
  int stage_ok, first_bad_layer;
  double budget_s, worst_attn_s, worst_ffn_s;
} afdk_stage_check;
afdk_status afdk_vet_stages(const double* attn, const double* ffn, int layers, double tpot_sla, int pipeline_stages,
                            int n_model_layers, afdk_stage_check* out);

#ifdef __cplusplus
}
#endif
#endif /* AFDK_H */
