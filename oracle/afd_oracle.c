/*
 * afd_oracle.c — CPU restatement of the Step-3 decode hot path (TEST ORACLE).
 *
 * Test infrastructure only: see afd_oracle.h for provenance, pinning status
 * ("numerics: parity unpinned by the reference; accounting pinned to
 * oracle/_ref") and the rule that the product never links this file.
 *
 * Each function cites what it restates:
 *   PAPER.md:93-95      MFA: q down 7168->2048, norm, up to 64x256; one shared
 *                       K and V head of 256
 *   PAPER.md:649        router runs on the attention side
 *   PAPER.md:654-655    FP8 dispatch + scales + expert distribution; BF16 return
 *   costmodel.cpp:26-44 core FLOPs 2*n_q*(qk+v)*ctx  (accounting helpers below)
 *   builtin_catalog.cpp:243-251  projection / expert parameter shapes
 *   moeplan.cpp:17-20   (dispatch + combine) * H * batch wire bytes
 */
#include "afd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ formats */
uint16_t orc_f32_to_bf16_bits(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_bf16_bits_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

float orc_bf16_round(float x) { return orc_bf16_bits_to_f32(orc_f32_to_bf16_bits(x)); }

static inline float maybe_bf16(float x, int r) { return r ? orc_bf16_round(x) : x; }

/* e4m3 "fn" variant: bias 7, max finite 448 (0x7e), 0x7f/0xff = NaN, no inf.
 * Round-to-nearest-even, saturating (cvt.rn.satfinite.e4m3x2.f32 semantics). */
uint8_t orc_f32_to_e4m3(float x) {
  if (isnan(x)) return 0x7f;
  uint8_t sign = signbit(x) ? 0x80 : 0x00;
  float a = fabsf(x);
  if (a >= 448.0f) return sign | 0x7e;
  if (a < 0.015625f) { /* below min normal 2^-6: subnormal grid 2^-9 */
    float q = nearbyintf(a * 512.0f); /* exact scaling, RNE */
    return sign | (uint8_t)q;          /* q==8 encodes min normal exactly */
  }
  int e;
  float m = frexpf(a, &e); /* a = m * 2^e, m in [0.5,1) */
  m *= 2.0f;
  e -= 1; /* m in [1,2) */
  float mant = nearbyintf((m - 1.0f) * 8.0f);
  if (mant >= 8.0f) { mant = 0.0f; e += 1; }
  int field = e + 7;
  if (field > 15 || (field == 15 && mant > 6.0f)) return sign | 0x7e;
  return sign | (uint8_t)((field << 3) | (int)mant);
}

float orc_e4m3_to_f32(uint8_t v) {
  int s = v & 0x80, field = (v >> 3) & 0xf, mant = v & 0x7;
  float r;
  if (field == 15 && mant == 7) return NAN;
  if (field == 0) r = ldexpf((float)mant, -9);
  else r = ldexpf(1.0f + mant / 8.0f, field - 7);
  return s ? -r : r;
}

/* ------------------------------------------------------------- elementwise */
/* step3_text.py: input_layernorm / inter_norm / post_attention_layernorm */
void orc_rmsnorm(const float* x, const float* w, int rows, int dim, float eps,
                 int round_bf16, float* out) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const float* xr = x + (size_t)r * dim;
    double ss = 0.0;
    for (int i = 0; i < dim; ++i) ss += (double)xr[i] * xr[i];
    const float inv = (float)(1.0 / sqrt(ss / dim + (double)eps));
    for (int i = 0; i < dim; ++i)
      out[(size_t)r * dim + i] = maybe_bf16((xr[i] * inv) * w[i], round_bf16);
  }
}

void orc_linear(const float* x, const float* W, int M, int N, int K, int round_bf16,
                float* out) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      const float* xr = x + (size_t)m * K;
      const float* wr = W + (size_t)n * K;
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += (double)xr[k] * wr[k];
      out[(size_t)m * N + n] = maybe_bf16((float)acc, round_bf16);
    }
}

/* step3_text.py: get_rope(head_dim, is_neox_style=True), rope_theta 5e5.
 * cos/sin evaluated in double from the exact angle; the B200 path reads a
 * host-built table of the same double-evaluated values (afdk_rope_table). */
void orc_rope_neox(float* x, int n_vec, int dim, int pos, float theta, int round_bf16) {
  const int half = dim / 2;
  for (int i = 0; i < half; ++i) {
    const double inv_freq = pow((double)theta, -(2.0 * i) / dim);
    const double ang = (double)pos * inv_freq;
    const float c = (float)cos(ang), s = (float)sin(ang);
    for (int v = 0; v < n_vec; ++v) {
      float* xv = x + (size_t)v * dim;
      const float x1 = xv[i], x2 = xv[i + half];
      xv[i] = maybe_bf16(x1 * c - x2 * s, round_bf16);
      xv[i + half] = maybe_bf16(x2 * c + x1 * s, round_bf16);
    }
  }
}

/* ----------------------------------------------------- MFA decode attention */
/* One shared K and V head serves all H query heads. */
void orc_mfa_decode_attention(const float* q, const float* k_cache, const float* v_cache,
                              const int32_t* block_table, int max_pages,
                              const int32_t* seq_lens, int B, int H, int D, int page,
                              float scale, int round_bf16, float* out, float* lse) {
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < H; ++h) {
      const int L = seq_lens[b];
      const float* qv = q + ((size_t)b * H + h) * D;
      float* o = out + ((size_t)b * H + h) * D;
      if (L <= 0) {
        for (int d = 0; d < D; ++d) o[d] = 0.0f;
        if (lse) lse[(size_t)b * H + h] = -INFINITY;
        continue;
      }
      double* s = (double*)malloc(sizeof(double) * (size_t)L);
      double mx = -INFINITY;
      for (int t = 0; t < L; ++t) {
        const int pg = block_table[(size_t)b * max_pages + t / page];
        const float* kv = k_cache + ((size_t)pg * page + (t % page)) * D;
        double acc = 0.0;
        for (int d = 0; d < D; ++d) acc += (double)qv[d] * kv[d];
        s[t] = acc * scale;
        if (s[t] > mx) mx = s[t];
      }
      double l = 0.0;
      double* acc = (double*)calloc((size_t)D, sizeof(double));
      for (int t = 0; t < L; ++t) {
        const double p = exp(s[t] - mx);
        l += p;
        const int pg = block_table[(size_t)b * max_pages + t / page];
        const float* vv = v_cache + ((size_t)pg * page + (t % page)) * D;
        for (int d = 0; d < D; ++d) acc[d] += p * vv[d];
      }
      for (int d = 0; d < D; ++d) o[d] = maybe_bf16((float)(acc[d] / l), round_bf16);
      if (lse) lse[(size_t)b * H + h] = (float)(mx + log(l));
      free(acc);
      free(s);
    }
}

/* ---------------------------------------------------- attention-side layer */
void orc_mfa_layer(const orc_mfa_dims* d, int B, const float* x,
                   const float* w_in_norm, const float* w_qkv, const float* w_q_norm,
                   const float* w_q_up, const float* w_o, const float* w_post_norm,
                   float* k_cache, float* v_cache, const int32_t* block_table,
                   int max_pages, const int32_t* seq_lens, int round_bf16,
                   float* h_res, float* h_norm) {
  const int Hd = d->hidden, QL = d->q_lora, NH = d->n_heads, D = d->head_dim;
  const int NQKV = QL + 2 * D, NQ = NH * D;
  float* xn = (float*)malloc(sizeof(float) * (size_t)B * Hd);
  float* qkv = (float*)malloc(sizeof(float) * (size_t)B * NQKV);
  float* qa_in = (float*)malloc(sizeof(float) * (size_t)B * QL);
  float* qa = (float*)malloc(sizeof(float) * (size_t)B * QL);
  float* q = (float*)malloc(sizeof(float) * (size_t)B * NQ);
  float* attn = (float*)malloc(sizeof(float) * (size_t)B * NQ);
  float* o = (float*)malloc(sizeof(float) * (size_t)B * Hd);

  orc_rmsnorm(x, w_in_norm, B, Hd, d->rms_eps, round_bf16, xn);       /* input_layernorm */
  orc_linear(xn, w_qkv, B, NQKV, Hd, round_bf16, qkv);                /* qkv_proj        */
  for (int b = 0; b < B; ++b)
    memcpy(qa_in + (size_t)b * QL, qkv + (size_t)b * NQKV, sizeof(float) * QL);
  orc_rmsnorm(qa_in, w_q_norm, B, QL, d->rms_eps, round_bf16, qa);    /* inter_norm      */
  if (d->qup_mx) { /* MXFP8 q_up input: e4m3 x 2^e per 32 q-latent elements */
    uint8_t* q8 = (uint8_t*)malloc((size_t)B * QL);
    uint8_t* sf = (uint8_t*)malloc((size_t)B * (QL / 32));
    orc_quant_mx(qa, B, QL, q8, sf);
    for (size_t i = 0; i < (size_t)B * QL; ++i) qa[i] = orc_e4m3_to_f32(q8[i]) * orc_mx_scale(sf[i / 32]);
    free(q8);
    free(sf);
  }
  orc_linear(qa, w_q_up, B, NQ, QL, round_bf16, q);                   /* wq              */
  for (int b = 0; b < B; ++b) {
    const int pos = seq_lens[b] - 1;
    float* kb = qkv + (size_t)b * NQKV + QL;
    float* vb = kb + D;
    orc_rope_neox(q + (size_t)b * NQ, NH, D, pos, d->rope_theta, round_bf16);
    orc_rope_neox(kb, 1, D, pos, d->rope_theta, round_bf16);
    const int pg = block_table[(size_t)b * max_pages + pos / d->page];
    float* kdst = k_cache + ((size_t)pg * d->page + pos % d->page) * D;
    float* vdst = v_cache + ((size_t)pg * d->page + pos % d->page) * D;
    if (d->kv_k_scale > 0.0f) { /* e4m3 cache: store the dequantised e4m3 value */
      for (int i = 0; i < D; ++i) {
        kdst[i] = orc_e4m3_to_f32(orc_f32_to_e4m3(kb[i] / d->kv_k_scale)) * d->kv_k_scale;
        vdst[i] = orc_e4m3_to_f32(orc_f32_to_e4m3(vb[i] / d->kv_v_scale)) * d->kv_v_scale;
      }
    } else {
      memcpy(kdst, kb, sizeof(float) * D);                             /* paged KV append */
      memcpy(vdst, vb, sizeof(float) * D);
    }
  }
  if (d->kv_k_scale > 0.0f) { /* per-(request, head) e4m3 query, power-of-two scale, as the fp8 kernel */
    for (size_t r = 0; r < (size_t)B * NH; ++r) {
      float* qr = q + r * D;
      float amax = 0.0f;
      for (int i = 0; i < D; ++i) amax = fmaxf(amax, fabsf(qr[i]));
      const int e = orc_mx_exponent(amax);
      for (int i = 0; i < D; ++i) qr[i] = ldexpf(orc_e4m3_to_f32(orc_f32_to_e4m3(qr[i] * ldexpf(1.0f, -e))), e);
    }
  }
  orc_mfa_decode_attention(q, k_cache, v_cache, block_table, max_pages, seq_lens, B, NH, D,
                           d->page, d->softmax_scale, round_bf16, attn, NULL);
  if (d->o_mx) { /* MXFP8 o_proj input: e4m3 x 2^e per 32 attention-output elements */
    uint8_t* q8 = (uint8_t*)malloc((size_t)B * NQ);
    uint8_t* sf = (uint8_t*)malloc((size_t)B * (NQ / 32));
    orc_quant_mx(attn, B, NQ, q8, sf);
    for (size_t i = 0; i < (size_t)B * NQ; ++i) attn[i] = orc_e4m3_to_f32(q8[i]) * orc_mx_scale(sf[i / 32]);
    free(q8);
    free(sf);
  }
  orc_linear(attn, w_o, B, Hd, NQ, 0, o);                             /* o_proj (fp32)   */
  for (size_t i = 0; i < (size_t)B * Hd; ++i) h_res[i] = maybe_bf16(x[i] + o[i], round_bf16);
  orc_rmsnorm(h_res, w_post_norm, B, Hd, d->rms_eps, round_bf16, h_norm);

  free(xn); free(qkv); free(qa_in); free(qa); free(q); free(attn); free(o);
}

/* ------------------------------------------------------------------ router */
/* FusedMoE(scoring softmax, renormalize=norm_expert_weight=False) semantics;
 * selection ties break to the lower expert id so indices are deterministic. */
void orc_router_topk(const float* logits, int T, int E, int k, int renormalize,
                     int32_t* ids, float* weights) {
  for (int t = 0; t < T; ++t) {
    const float* lg = logits + (size_t)t * E;
    float mx = lg[0];
    for (int e = 1; e < E; ++e) mx = lg[e] > mx ? lg[e] : mx;
    float sum = 0.0f;
    for (int e = 0; e < E; ++e) sum += expf(lg[e] - mx);
    unsigned char taken[1024] = {0};
    float wsum = 0.0f;
    for (int j = 0; j < k; ++j) {
      int best = -1;
      for (int e = 0; e < E; ++e) {
        if (taken[e]) continue;
        if (best < 0 || lg[e] > lg[best]) best = e;
      }
      taken[best] = 1;
      ids[(size_t)t * k + j] = best;
      weights[(size_t)t * k + j] = expf(lg[best] - mx) / sum;
      wsum += weights[(size_t)t * k + j];
    }
    if (renormalize)
      for (int j = 0; j < k; ++j) weights[(size_t)t * k + j] /= wsum;
  }
}

/* Expert distribution metadata of PAPER.md:655: counts -> exclusive offsets,
 * then a stable scatter in (expert, token, j) order. */
void orc_moe_permute(const int32_t* ids, int T, int k, int E, int32_t* offsets,
                     int32_t* perm, int32_t* inv) {
  int32_t* fill = (int32_t*)calloc((size_t)E, sizeof(int32_t));
  for (int e = 0; e <= E; ++e) offsets[e] = 0;
  for (int i = 0; i < T * k; ++i) offsets[ids[i] + 1]++;
  for (int e = 0; e < E; ++e) offsets[e + 1] += offsets[e];
  for (int i = 0; i < T * k; ++i) {
    const int e = ids[i];
    const int slot = offsets[e] + fill[e]++;
    perm[slot] = i;
    inv[i] = slot;
  }
  free(fill);
}

/* ------------------------------------------------------------ quantization */
void orc_quant_fp8_rowblock(const float* x, int rows, int cols, int block,
                            uint8_t* q, float* scales) {
  const int nb = cols / block;
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int b = 0; b < nb; ++b) {
      const float* xb = x + (size_t)r * cols + (size_t)b * block;
      float amax = 0.0f;
      for (int i = 0; i < block; ++i) amax = fmaxf(amax, fabsf(xb[i]));
      const float sc = fmaxf(amax, 1e-10f) / 448.0f;
      scales[(size_t)r * nb + b] = sc;
      for (int i = 0; i < block; ++i)
        q[(size_t)r * cols + (size_t)b * block + i] = orc_f32_to_e4m3(xb[i] / sc);
    }
}

void orc_quant_fp8_tile(const float* w, int rows, int cols, int bm, int bk,
                        uint8_t* q, float* scales) {
  const int nbr = rows / bm, nbc = cols / bk;
#pragma omp parallel for schedule(static)
  for (int br = 0; br < nbr; ++br)
    for (int bc = 0; bc < nbc; ++bc) {
      float amax = 0.0f;
      for (int r = 0; r < bm; ++r)
        for (int c = 0; c < bk; ++c)
          amax = fmaxf(amax, fabsf(w[((size_t)br * bm + r) * cols + (size_t)bc * bk + c]));
      const float sc = fmaxf(amax, 1e-10f) / 448.0f;
      scales[(size_t)br * nbc + bc] = sc;
      for (int r = 0; r < bm; ++r)
        for (int c = 0; c < bk; ++c) {
          const size_t i = ((size_t)br * bm + r) * cols + (size_t)bc * bk + c;
          q[i] = orc_f32_to_e4m3(w[i] / sc);
        }
    }
}

/* ------------------------------------------------------------- expert FFN */
static float silu(float g) { return g / (1.0f + expf(-g)); }

void orc_expert_ffn_fp8(const uint8_t* xq, const float* xs, int rows, int H, int I,
                        const uint8_t* w13, const float* s13,
                        const uint8_t* w2, const float* s2, float* y) {
  const int nbH = H / 128, nbI = I / 128;
  float lut[256];
  for (int i = 0; i < 256; ++i) lut[i] = orc_e4m3_to_f32((uint8_t)i);
  float* hbuf = (float*)malloc(sizeof(float) * (size_t)rows * I);
  uint8_t* hq = (uint8_t*)malloc((size_t)rows * I);
  float* hs = (float*)malloc(sizeof(float) * (size_t)rows * nbI);
  /* gate/up: per 128-wide K block, exact fp8 products, scaled block sums */
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < I; ++n) {
      double g = 0.0, u = 0.0;
      for (int kb = 0; kb < nbH; ++kb) {
        double ag = 0.0, au = 0.0;
        for (int c = kb * 128; c < kb * 128 + 128; ++c) {
          const double xv = lut[xq[(size_t)r * H + c]];
          ag += xv * lut[w13[(size_t)n * H + c]];
          au += xv * lut[w13[(size_t)(n + I) * H + c]];
        }
        const double sx = xs[(size_t)r * nbH + kb];
        g += ag * sx * s13[(size_t)(n / 128) * nbH + kb];
        u += au * sx * s13[(size_t)((n + I) / 128) * nbH + kb];
      }
      hbuf[(size_t)r * I + n] = silu((float)g) * (float)u;
    }
  orc_quant_fp8_rowblock(hbuf, rows, I, 128, hq, hs);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < H; ++n) {
      double acc = 0.0;
      for (int kb = 0; kb < nbI; ++kb) {
        double a = 0.0;
        for (int c = kb * 128; c < kb * 128 + 128; ++c)
          a += (double)lut[hq[(size_t)r * I + c]] * lut[w2[(size_t)n * I + c]];
        acc += a * hs[(size_t)r * nbI + kb] * s2[(size_t)(n / 128) * nbI + kb];
      }
      y[(size_t)r * H + n] = (float)acc;
    }
  free(hbuf); free(hq); free(hs);
}

void orc_moe_layer_fp8(const uint8_t* xq, const float* xs, int T, int H, int I, int E,
                       int k, const int32_t* ids, const float* weights,
                       const uint8_t* w13_all, const float* s13_all,
                       const uint8_t* w2_all, const float* s2_all, int round_bf16,
                       float* out) {
  const int nbH = H / 128, nbI = I / 128;
  const size_t w13_sz = (size_t)2 * I * H, w2_sz = (size_t)H * I;
  const size_t s13_sz = (size_t)(2 * I / 128) * nbH, s2_sz = (size_t)nbH * nbI;
  double* acc = (double*)calloc((size_t)T * H, sizeof(double));
  float* y = (float*)malloc(sizeof(float) * (size_t)T * H);
  uint8_t* gx = (uint8_t*)malloc((size_t)T * H);
  float* gs = (float*)malloc(sizeof(float) * (size_t)T * nbH);
  int32_t* rows_tok = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  float* rows_w = (float*)malloc(sizeof(float) * (size_t)T);
  for (int e = 0; e <= E; ++e) {
    int n = 0;
    for (int t = 0; t < T; ++t) {
      if (e == E) { rows_tok[n] = t; rows_w[n] = 1.0f; ++n; continue; }  /* shared */
      for (int j = 0; j < k; ++j)
        if (ids[(size_t)t * k + j] == e) { rows_tok[n] = t; rows_w[n] = weights[(size_t)t * k + j]; ++n; }
    }
    if (n == 0) continue;
    for (int r = 0; r < n; ++r) {
      memcpy(gx + (size_t)r * H, xq + (size_t)rows_tok[r] * H, (size_t)H);
      memcpy(gs + (size_t)r * nbH, xs + (size_t)rows_tok[r] * nbH, sizeof(float) * nbH);
    }
    orc_expert_ffn_fp8(gx, gs, n, H, I, w13_all + e * w13_sz, s13_all + e * s13_sz,
                       w2_all + e * w2_sz, s2_all + e * s2_sz, y);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < H; ++c)
        acc[(size_t)rows_tok[r] * H + c] += (double)rows_w[r] * y[(size_t)r * H + c];
  }
  for (size_t i = 0; i < (size_t)T * H; ++i) out[i] = maybe_bf16((float)acc[i], round_bf16);
  free(acc); free(y); free(gx); free(gs); free(rows_tok); free(rows_w);
}

/* ------------------------------------------------- 16-bit / fp32 experts */
/* QuantScheme with 2-byte FFN weights (types.hpp:34-40, effective_kind
 * types.hpp:93-95; "BF16 where FP8 is unavailable"): the gated
 * expert of step3_text.py Step3TextMLP — gate_up_proj rows [gate; up],
 * SiluAndMul, down_proj.  x and the weights are passed as float (bf16-widened
 * for the bf16 path, unquantised for the fp32 error budget).  round_bf16: the
 * SwiGLU intermediate is stored bf16 (the B200 path's storage point). */
void orc_expert_ffn_f32(const float* x, int rows, int H, int I, const float* w13,
                        const float* w2, int round_bf16, float* y) {
  float* hbuf = (float*)malloc(sizeof(float) * (size_t)rows * I);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < I; ++n) {
      const float* xr = x + (size_t)r * H;
      const float* wg = w13 + (size_t)n * H;
      const float* wu = w13 + (size_t)(n + I) * H;
      double g = 0.0, u = 0.0;
      for (int c = 0; c < H; ++c) { g += (double)xr[c] * wg[c]; u += (double)xr[c] * wu[c]; }
      hbuf[(size_t)r * I + n] = maybe_bf16(silu((float)g) * (float)u, round_bf16);
    }
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < H; ++n) {
      const float* hr = hbuf + (size_t)r * I;
      const float* wr = w2 + (size_t)n * I;
      double acc = 0.0;
      for (int c = 0; c < I; ++c) acc += (double)hr[c] * wr[c];
      y[(size_t)r * H + n] = (float)acc;
    }
  free(hbuf);
}

/* Routed layer over 16-bit/fp32 experts: same routing, shared-expert and
 * combine semantics as orc_moe_layer_fp8 (experts [0,E) routed, E shared). */
void orc_moe_layer_f32(const float* x, int T, int H, int I, int E, int k, const int32_t* ids,
                       const float* weights, const float* w13_all, const float* w2_all,
                       int round_bf16, float* out) {
  const size_t w13_sz = (size_t)2 * I * H, w2_sz = (size_t)H * I;
  double* acc = (double*)calloc((size_t)T * H, sizeof(double));
  float* y = (float*)malloc(sizeof(float) * (size_t)T * H);
  float* gx = (float*)malloc(sizeof(float) * (size_t)T * H);
  int32_t* rows_tok = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  float* rows_w = (float*)malloc(sizeof(float) * (size_t)T);
  for (int e = 0; e <= E; ++e) {
    int n = 0;
    for (int t = 0; t < T; ++t) {
      if (e == E) { rows_tok[n] = t; rows_w[n] = 1.0f; ++n; continue; }
      for (int j = 0; j < k; ++j)
        if (ids[(size_t)t * k + j] == e) { rows_tok[n] = t; rows_w[n] = weights[(size_t)t * k + j]; ++n; }
    }
    if (n == 0) continue;
    for (int r = 0; r < n; ++r) memcpy(gx + (size_t)r * H, x + (size_t)rows_tok[r] * H, sizeof(float) * H);
    orc_expert_ffn_f32(gx, n, H, I, w13_all + e * w13_sz, w2_all + e * w2_sz, round_bf16, y);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < H; ++c)
        acc[(size_t)rows_tok[r] * H + c] += (double)rows_w[r] * y[(size_t)r * H + c];
  }
  for (size_t i = 0; i < (size_t)T * H; ++i) out[i] = maybe_bf16((float)acc[i], round_bf16);
  free(acc); free(y); free(gx); free(rows_tok); free(rows_w);
}

/* ------------------------------------------------------------------ MXFP8 */
/* smallest e with amax <= 448 * 2^e, from the exact binary exponent/mantissa
 * of amax (448 = 1.75 * 2^8) */
int orc_mx_exponent(float amax) {
  if (!(amax > 0.0f)) return -127;
  uint32_t u;
  memcpy(&u, &amax, 4);
  const int E = (int)((u >> 23) & 0xff);
  const uint32_t M = u & 0x7fffffu;
  if (E == 0) return -127; /* subnormal amax */
  const int k = E - 127;
  int e = (M <= 6291456u) ? k - 8 : k - 7; /* mantissa 1.M <= 1.75 */
  if (e < -127) e = -127;
  if (e > 127) e = 127;
  return e;
}

float orc_mx_scale(uint8_t sf) { return ldexpf(1.0f, (int)sf - 127); }

void orc_quant_pow2(const float* x, int rows, int cols, int block, uint8_t* q, int32_t* eo) {
  const int nb = cols / block;
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int b = 0; b < nb; ++b) {
      const float* xb = x + (size_t)r * cols + (size_t)b * block;
      float amax = 0.0f;
      for (int i = 0; i < block; ++i) amax = fmaxf(amax, fabsf(xb[i]));
      const int e = orc_mx_exponent(amax);
      eo[(size_t)r * nb + b] = e;
      const float inv = ldexpf(1.0f, -e);
      for (int i = 0; i < block; ++i) q[(size_t)r * cols + (size_t)b * block + i] = orc_f32_to_e4m3(xb[i] * inv);
    }
}

void orc_quant_mx(const float* x, int rows, int cols, uint8_t* q, uint8_t* sf) {
  const int nb = cols / 32;
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int b = 0; b < nb; ++b) {
      const float* xb = x + (size_t)r * cols + (size_t)b * 32;
      float amax = 0.0f;
      for (int i = 0; i < 32; ++i) amax = fmaxf(amax, fabsf(xb[i]));
      const int e = orc_mx_exponent(amax);
      sf[(size_t)r * nb + b] = (uint8_t)(e + 127);
      const float inv = ldexpf(1.0f, -e);
      for (int i = 0; i < 32; ++i) q[(size_t)r * cols + (size_t)b * 32 + i] = orc_f32_to_e4m3(xb[i] * inv);
    }
}

void orc_expert_ffn_mx(const uint8_t* xq, const uint8_t* xsf, int rows, int H, int I,
                       const uint8_t* w13, const uint8_t* sf13, const uint8_t* w2,
                       const uint8_t* sf2, float* y) {
  float lut[256];
  for (int i = 0; i < 256; ++i) lut[i] = orc_e4m3_to_f32((uint8_t)i);
  const int nbH = H / 32, nbI = I / 32;
  float* hbuf = (float*)malloc(sizeof(float) * (size_t)rows * I);
  uint8_t* hq = (uint8_t*)malloc((size_t)rows * I);
  uint8_t* hsf = (uint8_t*)malloc((size_t)rows * nbI);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < I; ++n) {
      double g = 0.0, u = 0.0;
      for (int kb = 0; kb < nbH; ++kb) {
        double ag = 0.0, au = 0.0;
        for (int c = kb * 32; c < kb * 32 + 32; ++c) {
          const double xv = lut[xq[(size_t)r * H + c]];
          ag += xv * lut[w13[(size_t)n * H + c]];
          au += xv * lut[w13[(size_t)(n + I) * H + c]];
        }
        const double sx = orc_mx_scale(xsf[(size_t)r * nbH + kb]);
        g += ag * sx * orc_mx_scale(sf13[(size_t)n * nbH + kb]);
        u += au * sx * orc_mx_scale(sf13[(size_t)(n + I) * nbH + kb]);
      }
      hbuf[(size_t)r * I + n] = silu((float)g) * (float)u;
    }
  orc_quant_mx(hbuf, rows, I, hq, hsf);
#pragma omp parallel for collapse(2) schedule(static)
  for (int r = 0; r < rows; ++r)
    for (int n = 0; n < H; ++n) {
      double acc = 0.0;
      for (int kb = 0; kb < nbI; ++kb) {
        double a = 0.0;
        for (int c = kb * 32; c < kb * 32 + 32; ++c)
          a += (double)lut[hq[(size_t)r * I + c]] * lut[w2[(size_t)n * I + c]];
        acc += a * orc_mx_scale(hsf[(size_t)r * nbI + kb]) * orc_mx_scale(sf2[(size_t)n * nbI + kb]);
      }
      y[(size_t)r * H + n] = (float)acc;
    }
  free(hbuf); free(hq); free(hsf);
}

void orc_moe_layer_mx(const uint8_t* xq, const uint8_t* xsf, int T, int H, int I, int E, int k,
                      const int32_t* ids, const float* weights, const uint8_t* w13_all,
                      const uint8_t* sf13_all, const uint8_t* w2_all, const uint8_t* sf2_all,
                      int round_bf16, float* out) {
  const int nbH = H / 32;
  const size_t w13_sz = (size_t)2 * I * H, w2_sz = (size_t)H * I;
  const size_t sf13_sz = (size_t)2 * I * nbH, sf2_sz = (size_t)H * (I / 32);
  double* acc = (double*)calloc((size_t)T * H, sizeof(double));
  float* y = (float*)malloc(sizeof(float) * (size_t)T * H);
  uint8_t* gx = (uint8_t*)malloc((size_t)T * H);
  uint8_t* gs = (uint8_t*)malloc((size_t)T * nbH);
  int32_t* rows_tok = (int32_t*)malloc(sizeof(int32_t) * (size_t)T);
  float* rows_w = (float*)malloc(sizeof(float) * (size_t)T);
  for (int e = 0; e <= E; ++e) {
    int n = 0;
    for (int t = 0; t < T; ++t) {
      if (e == E) { rows_tok[n] = t; rows_w[n] = 1.0f; ++n; continue; }
      for (int j = 0; j < k; ++j)
        if (ids[(size_t)t * k + j] == e) { rows_tok[n] = t; rows_w[n] = weights[(size_t)t * k + j]; ++n; }
    }
    if (n == 0) continue;
    for (int r = 0; r < n; ++r) {
      memcpy(gx + (size_t)r * H, xq + (size_t)rows_tok[r] * H, (size_t)H);
      memcpy(gs + (size_t)r * nbH, xsf + (size_t)rows_tok[r] * nbH, (size_t)nbH);
    }
    orc_expert_ffn_mx(gx, gs, n, H, I, w13_all + e * w13_sz, sf13_all + e * sf13_sz, w2_all + e * w2_sz,
                      sf2_all + e * sf2_sz, y);
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < H; ++c)
        acc[(size_t)rows_tok[r] * H + c] += (double)rows_w[r] * y[(size_t)r * H + c];
  }
  for (size_t i = 0; i < (size_t)T * H; ++i) out[i] = maybe_bf16((float)acc[i], round_bf16);
  free(acc); free(y); free(gx); free(gs); free(rows_tok); free(rows_w);
}

/* -------------------------------------------------------------- accounting */
/* costmodel.cpp:26-44 (full attention): 2 * n_q * (qk + v) * ctx */
double orc_mfa_core_flops(int n_heads, int head_dim, int64_t ctx) {
  return 2.0 * n_heads * (double)(head_dim + head_dim) * (double)ctx;
}
/* one K row + one V row of head_dim per token (builtin_catalog.cpp:242 at 8-bit) */
double orc_mfa_kv_bytes(int head_dim, int64_t ctx, int elt_bytes) {
  return 2.0 * head_dim * (double)elt_bytes * (double)ctx;
}
/* builtin_catalog.cpp:243-247 per layer */
int64_t orc_mfa_linear_params(int hidden, int q_lora, int n_heads, int head_dim) {
  const int64_t h = hidden, q = q_lora, nd = (int64_t)n_heads * head_dim;
  return h * q + q * nd + 2 * h * head_dim + nd * h;
}
/* builtin_catalog.cpp:248-251: 3*h*inter params per gated expert */
double orc_moe_flops_per_token(int hidden, int inter, int k, int n_shared) {
  return 2.0 * 3.0 * hidden * (double)inter * (k + n_shared);
}
/* moeplan.cpp:17-20 with the fp8/bf16 element sizes of builtin_catalog.cpp:11 */
double orc_afd_wire_bytes(int hidden, int64_t T) { return (1.0 + 2.0) * hidden * (double)T; }
/* per token: one fp32 scale per 128 elements + k (int32 id, fp32 weight) */
double orc_dispatch_meta_bytes(int hidden, int k, int64_t T) {
  return ((double)(hidden / 128) * 4.0 + k * 8.0) * (double)T;
}
