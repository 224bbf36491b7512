"""numpy/ctypes view of the TEST ORACLES (liborc.so and _ref/libafdref.so).

Test infrastructure only: imported by tests/, bench.py's cpu_baseline /
--impl reference legs and __graft_entry__.smoke() as the checker — never by
the product package.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_longlong, c_uint8, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liborc.so")
REF_PATH = os.path.join(HERE, "_ref", "libafdref.so")

_orc = None
_ref = None


def _p(a, ct):
    return a.ctypes.data_as(POINTER(ct)) if a is not None else None


def orc() -> ctypes.CDLL:
    global _orc
    if _orc is None:
        # OpenMP workers must sleep between parallel regions: spinning workers
        # fight the other thread pools of the process (torch, OpenBLAS) and made
        # every small parallel region cost ~60 ms here.  Read by libgomp at load.
        os.environ.setdefault("OMP_WAIT_POLICY", "passive")
        if not os.path.exists(ORC_PATH):
            raise ImportError("oracle/liborc.so not built (make -C oracle)")
        _orc = ctypes.CDLL(ORC_PATH)
        _orc.orc_bf16_round.restype = c_float
        _orc.orc_bf16_round.argtypes = [c_float]
        _orc.orc_f32_to_e4m3.restype = c_uint8
        _orc.orc_f32_to_e4m3.argtypes = [c_float]
        _orc.orc_e4m3_to_f32.restype = c_float
        _orc.orc_e4m3_to_f32.argtypes = [c_uint8]
        for name in ("orc_mfa_core_flops", "orc_mfa_kv_bytes", "orc_moe_flops_per_token",
                     "orc_afd_wire_bytes", "orc_dispatch_meta_bytes"):
            getattr(_orc, name).restype = c_double
        _orc.orc_mfa_core_flops.argtypes = [c_int, c_int, c_longlong]
        _orc.orc_mfa_kv_bytes.argtypes = [c_int, c_longlong, c_int]
        _orc.orc_moe_flops_per_token.argtypes = [c_int, c_int, c_int, c_int]
        _orc.orc_afd_wire_bytes.argtypes = [c_int, c_longlong]
        _orc.orc_dispatch_meta_bytes.argtypes = [c_int, c_int, c_longlong]
        _orc.orc_mfa_linear_params.restype = c_longlong
        _orc.orc_mfa_linear_params.argtypes = [c_int, c_int, c_int, c_int]
        _orc.orc_num_threads.restype = c_int
    return _orc


def ref() -> ctypes.CDLL:
    """The reference's own analytic library (compiled from /root/reference)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise ImportError("oracle/_ref/libafdref.so not built (make -C oracle ref)")
        _ref = ctypes.CDLL(REF_PATH)
        _ref.ref_last_error.restype = c_char_p
        _ref.ref_trace_csv.restype = c_void_p
    return _ref


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------ formats
def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (RNE) -> fp32, vectorised restatement of orc_bf16_round."""
    u = _f32(x).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(x), np.float32(np.nan), out)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << 16).view(np.float32)


E4M3_LUT = None


def e4m3_to_f32(q: np.ndarray) -> np.ndarray:
    global E4M3_LUT
    if E4M3_LUT is None:
        E4M3_LUT = np.array([orc().orc_e4m3_to_f32(i) for i in range(256)], dtype=np.float32)
    return E4M3_LUT[np.asarray(q, dtype=np.uint8)]


# --------------------------------------------------------------- operators
def rmsnorm(x, w, eps=1e-5, round_bf16=True):
    x, w = _f32(x), _f32(w)
    out = np.empty_like(x)
    orc().orc_rmsnorm(_p(x, c_float), _p(w, c_float), c_int(x.shape[0]), c_int(x.shape[1]),
                      c_float(eps), c_int(int(round_bf16)), _p(out, c_float))
    return out


def linear(x, W, round_bf16=False):
    x, W = _f32(x), _f32(W)
    M, K = x.shape
    N = W.shape[0]
    out = np.empty((M, N), np.float32)
    orc().orc_linear(_p(x, c_float), _p(W, c_float), c_int(M), c_int(N), c_int(K),
                     c_int(int(round_bf16)), _p(out, c_float))
    return out


def mfa_decode_attention(q, k_cache, v_cache, block_table, seq_lens, scale, round_bf16=False):
    q, k_cache, v_cache = _f32(q), _f32(k_cache), _f32(v_cache)
    block_table, seq_lens = _i32(block_table), _i32(seq_lens)
    B, H, D = q.shape
    out = np.empty_like(q)
    lse = np.empty((B, H), np.float32)
    orc().orc_mfa_decode_attention(
        _p(q, c_float), _p(k_cache, c_float), _p(v_cache, c_float), _p(block_table, c_int32),
        c_int(block_table.shape[1]), _p(seq_lens, c_int32), c_int(B), c_int(H), c_int(D),
        c_int(k_cache.shape[1]), c_float(scale), c_int(int(round_bf16)), _p(out, c_float),
        _p(lse, c_float))
    return out, lse


def mfa_decode_attention_mtp(q, k_cache, v_cache, block_table, seq_lens, scale, round_bf16=False):
    """Multi-token decode (MTP what-if, costmodel.cpp:46-58 mtp factor).

    q [B, mtp, H, D]: the mtp newest tokens of every request (positions
    L-mtp .. L-1, all already in the KV cache).  Query j attends causally to
    keys at positions <= L-mtp+j; a query whose position is negative (L < mtp)
    yields zeros / -inf LSE.  Exact attention per query, as orc_mfa_decode_attention."""
    q = _f32(q)
    B, mtp, H, D = q.shape
    seq_lens = _i32(seq_lens)
    out = np.empty_like(q)
    lse = np.empty((B, mtp, H), np.float32)
    for j in range(mtp):
        sl = np.maximum(seq_lens - (mtp - 1 - j), 0).astype(np.int32)
        o, l = mfa_decode_attention(q[:, j], k_cache, v_cache, block_table, sl, scale, round_bf16=round_bf16)
        out[:, j], lse[:, j] = o, l
    return out, lse


def mfa_decode_attention_fp8(q, kq, vq, k_scale, v_scale, block_table, seq_lens, scale, round_bf16=False):
    """FP8-KV MFA decode (the paper's production setting).

    Semantics: K = e4m3(kq)*k_scale, V = e4m3(vq)*v_scale (per-tensor scales,
    512 B of KV per token, builtin_catalog.cpp:242); the query of every
    (request, head) is quantised with a power-of-two scale 2^e over its 256
    dims (the MXFP8 exponent rule, orc_quant_pow2); attention is then exact
    (double) on the dequantised Q/K/V.  The B200 kernel additionally
    rounds the softmax probabilities to e4m3 for the P.V tensor-core MMA
    (stated tolerance in tests/test_mfa_fp8_gpu.py)."""
    q = _f32(q)
    B, H, D = q.shape
    qq, qe = quant_pow2(q.reshape(B * H, D), block=D)
    qd = np.ldexp(e4m3_to_f32(qq), np.repeat(qe, D, axis=1)).astype(np.float32).reshape(B, H, D)
    kd = e4m3_to_f32(kq) * np.float32(k_scale)
    vd = e4m3_to_f32(vq) * np.float32(v_scale)
    return mfa_decode_attention(qd, kd, vd, block_table, seq_lens, scale, round_bf16=round_bf16)


class MfaDims(ctypes.Structure):
    _fields_ = [("hidden", c_int), ("q_lora", c_int), ("n_heads", c_int), ("head_dim", c_int),
                ("page", c_int), ("rms_eps", c_float), ("rope_theta", c_float),
                ("softmax_scale", c_float), ("kv_k_scale", c_float), ("kv_v_scale", c_float), ("o_mx", c_int),
                ("qup_mx", c_int)]


def mfa_layer(dims: dict, x, w, k_cache, v_cache, block_table, seq_lens, round_bf16=True):
    """Attention-side decode layer. `w` keys: in_norm, qkv, q_norm, q_up, o, post_norm.
    k_cache / v_cache (float32 copies) are updated in place with the new token."""
    d = MfaDims(dims["hidden"], dims["q_lora"], dims["n_heads"], dims["head_dim"], dims["page"],
                dims.get("rms_eps", 1e-5), dims.get("rope_theta", 5e5),
                dims.get("softmax_scale", dims["head_dim"] ** -0.5),
                dims.get("kv_k_scale", 0.0), dims.get("kv_v_scale", 0.0), int(dims.get("o_mx", 0)),
                int(dims.get("qup_mx", 0)))
    x = _f32(x)
    B = x.shape[0]
    ws = {k: _f32(v) for k, v in w.items()}
    assert k_cache.dtype == np.float32 and k_cache.flags.c_contiguous
    block_table, seq_lens = _i32(block_table), _i32(seq_lens)
    h_res = np.empty_like(x)
    h_norm = np.empty_like(x)
    orc().orc_mfa_layer(ctypes.byref(d), c_int(B), _p(x, c_float), _p(ws["in_norm"], c_float),
                        _p(ws["qkv"], c_float), _p(ws["q_norm"], c_float), _p(ws["q_up"], c_float),
                        _p(ws["o"], c_float), _p(ws["post_norm"], c_float), _p(k_cache, c_float),
                        _p(v_cache, c_float), _p(block_table, c_int32), c_int(block_table.shape[1]),
                        _p(seq_lens, c_int32), c_int(int(round_bf16)), _p(h_res, c_float),
                        _p(h_norm, c_float))
    return h_res, h_norm


def router_topk(logits, k, renormalize=False):
    logits = _f32(logits)
    T, E = logits.shape
    ids = np.empty((T, k), np.int32)
    wts = np.empty((T, k), np.float32)
    orc().orc_router_topk(_p(logits, c_float), c_int(T), c_int(E), c_int(k), c_int(int(renormalize)),
                          _p(ids, c_int32), _p(wts, c_float))
    return ids, wts


def moe_permute(ids, E):
    ids = _i32(ids)
    T, k = ids.shape
    offsets = np.empty(E + 1, np.int32)
    perm = np.empty(T * k, np.int32)
    inv = np.empty(T * k, np.int32)
    orc().orc_moe_permute(_p(ids, c_int32), c_int(T), c_int(k), c_int(E), _p(offsets, c_int32),
                          _p(perm, c_int32), _p(inv, c_int32))
    return offsets, perm, inv


def quant_fp8_rowblock(x, block=128):
    x = _f32(x)
    rows, cols = x.shape
    q = np.empty((rows, cols), np.uint8)
    s = np.empty((rows, cols // block), np.float32)
    orc().orc_quant_fp8_rowblock(_p(x, c_float), c_int(rows), c_int(cols), c_int(block),
                                 _p(q, c_uint8), _p(s, c_float))
    return q, s


def quant_fp8_tile(w, bm=128, bk=128):
    w = _f32(w)
    rows, cols = w.shape
    q = np.empty((rows, cols), np.uint8)
    s = np.empty((rows // bm, cols // bk), np.float32)
    orc().orc_quant_fp8_tile(_p(w, c_float), c_int(rows), c_int(cols), c_int(bm), c_int(bk),
                             _p(q, c_uint8), _p(s, c_float))
    return q, s


def expert_ffn_fp8(xq, xs, w13, s13, w2, s2):
    rows, H = xq.shape
    I = w2.shape[1]
    y = np.empty((rows, H), np.float32)
    orc().orc_expert_ffn_fp8(_p(np.ascontiguousarray(xq), c_uint8), _p(_f32(xs), c_float), c_int(rows),
                             c_int(H), c_int(I), _p(np.ascontiguousarray(w13), c_uint8), _p(_f32(s13), c_float),
                             _p(np.ascontiguousarray(w2), c_uint8), _p(_f32(s2), c_float), _p(y, c_float))
    return y


def moe_layer_fp8(xq, xs, ids, weights, w13_all, s13_all, w2_all, s2_all, round_bf16=True):
    T, H = xq.shape
    E = w13_all.shape[0] - 1
    I = w2_all.shape[2]
    k = ids.shape[1]
    out = np.empty((T, H), np.float32)
    orc().orc_moe_layer_fp8(
        _p(np.ascontiguousarray(xq), c_uint8), _p(_f32(xs), c_float), c_int(T), c_int(H), c_int(I),
        c_int(E), c_int(k), _p(_i32(ids), c_int32), _p(_f32(weights), c_float),
        _p(np.ascontiguousarray(w13_all), c_uint8), _p(_f32(s13_all), c_float),
        _p(np.ascontiguousarray(w2_all), c_uint8), _p(_f32(s2_all), c_float),
        c_int(int(round_bf16)), _p(out, c_float))
    return out


def mx_exponent(amax: float) -> int:
    orc().orc_mx_exponent.argtypes = [c_float]
    return orc().orc_mx_exponent(c_float(amax))


def quant_mx(x):
    """MXFP8: e4m3 codes [rows, cols] + UE8M0 scales [rows, cols/32]."""
    x = _f32(x)
    rows, cols = x.shape
    q = np.empty((rows, cols), np.uint8)
    sf = np.empty((rows, cols // 32), np.uint8)
    orc().orc_quant_mx(_p(x, c_float), c_int(rows), c_int(cols), _p(q, c_uint8), _p(sf, c_uint8))
    return q, sf


def quant_pow2(x, block):
    """e4m3 codes + per-block power-of-two exponents (orc_quant_pow2)."""
    x = _f32(x)
    rows, cols = x.shape
    q = np.empty((rows, cols), np.uint8)
    e = np.empty((rows, cols // block), np.int32)
    orc().orc_quant_pow2(_p(x, c_float), c_int(rows), c_int(cols), c_int(block), _p(q, c_uint8), _p(e, c_int32))
    return q, e


def mx_dequant(q, sf):
    q = np.asarray(q, np.uint8)
    return e4m3_to_f32(q) * np.exp2(np.repeat(np.asarray(sf, np.float64) - 127.0, 32, axis=-1)).astype(np.float32)


def expert_ffn_mx(xq, xsf, w13, sf13, w2, sf2):
    rows, H = xq.shape
    I = w2.shape[1]
    y = np.empty((rows, H), np.float32)
    c8 = lambda a: _p(np.ascontiguousarray(a, dtype=np.uint8), c_uint8)
    orc().orc_expert_ffn_mx(c8(xq), c8(xsf), c_int(rows), c_int(H), c_int(I), c8(w13), c8(sf13), c8(w2), c8(sf2),
                            _p(y, c_float))
    return y


def moe_layer_mx(xq, xsf, ids, weights, w13_all, sf13_all, w2_all, sf2_all, round_bf16=True):
    T, H = xq.shape
    E = w13_all.shape[0] - 1
    I = w2_all.shape[2]
    k = ids.shape[1]
    out = np.empty((T, H), np.float32)
    c8 = lambda a: _p(np.ascontiguousarray(a, dtype=np.uint8), c_uint8)
    orc().orc_moe_layer_mx(c8(xq), c8(xsf), c_int(T), c_int(H), c_int(I), c_int(E), c_int(k), _p(_i32(ids), c_int32),
                           _p(_f32(weights), c_float), c8(w13_all), c8(sf13_all), c8(w2_all), c8(sf2_all),
                           c_int(int(round_bf16)), _p(out, c_float))
    return out


def expert_ffn_f32(x, w13, w2, round_bf16=False):
    """Gated expert over float weights (orc_expert_ffn_f32): the bf16 FFN
    format with round_bf16=True (bf16-widened inputs), the unquantised fp32
    model with round_bf16=False."""
    x = _f32(x)
    rows, H = x.shape
    I = w2.shape[1]
    y = np.empty((rows, H), np.float32)
    orc().orc_expert_ffn_f32(_p(x, c_float), c_int(rows), c_int(H), c_int(I), _p(_f32(w13), c_float),
                             _p(_f32(w2), c_float), c_int(int(round_bf16)), _p(y, c_float))
    return y


def moe_layer_f32(x, ids, weights, w13_all, w2_all, round_bf16=False):
    x = _f32(x)
    T, H = x.shape
    E = w13_all.shape[0] - 1
    I = w2_all.shape[2]
    k = ids.shape[1]
    out = np.empty((T, H), np.float32)
    orc().orc_moe_layer_f32(_p(x, c_float), c_int(T), c_int(H), c_int(I), c_int(E), c_int(k),
                            _p(_i32(ids), c_int32), _p(_f32(weights), c_float), _p(_f32(w13_all), c_float),
                            _p(_f32(w2_all), c_float), c_int(int(round_bf16)), _p(out, c_float))
    return out


def moe_layer_by_expert(ids, weights, n_experts, expert_fn, tokens=None, round_bf16=True):
    """Routed layer restricted to a token subset, one expert at a time.

    Same semantics as orc_moe_layer_* (experts [0,E) routed, E = shared, out =
    sum_k w_k y_k + shared, bf16-rounded): a token's output depends only on its
    own row, so the oracle can check a fixed subset of a full-size layer.
    expert_fn(e, token_rows) -> y [len(rows), H] float32 runs expert e (the
    caller fetches that expert's weights only, keeping host memory small)."""
    ids = np.asarray(ids)
    T = ids.shape[0]
    tokens = np.arange(T) if tokens is None else np.asarray(tokens)
    acc = None
    for e in range(n_experts + 1):
        if e == n_experts:
            rows, w = tokens, np.ones(len(tokens), np.float64)
        else:
            hit = ids[tokens] == e
            sel = hit.any(axis=1)
            rows = tokens[sel]
            w = np.asarray(weights)[rows][hit[sel]].astype(np.float64)
        if len(rows) == 0:
            continue
        y = expert_fn(e, rows).astype(np.float64)
        if acc is None:
            acc = np.zeros((len(tokens), y.shape[1]), np.float64)
        pos = np.searchsorted(tokens, rows) if np.all(np.diff(tokens) > 0) else \
            np.array([int(np.where(tokens == r)[0][0]) for r in rows])
        np.add.at(acc, pos, w[:, None] * y)
    out = acc.astype(np.float32)
    return bf16_round(out) if round_bf16 else out


def num_threads() -> int:
    return orc().orc_num_threads()


# ---------------------------------------------------- reference accounting
STEP3 = b"step3"


def ref_model_card(model=STEP3):
    out = (c_longlong * 9)()
    _ref_check(ref().ref_model_card(c_char_p(model), out))
    keys = ["n_layers", "hidden", "n_q_heads", "qk_dim", "v_dim", "kv_token_bytes",
            "attn_linear_params", "ffn_activated_params", "ffn_total_weight_bytes"]
    return dict(zip(keys, list(out)))


def ref_cost_breakdown(ctx, kvq=1.0, mtp=1.0, model=STEP3):
    out = (c_double * 4)()
    _ref_check(ref().ref_cost_breakdown(c_char_p(model), c_longlong(ctx), c_double(kvq), c_double(mtp), out))
    return dict(kv_state_bytes=out[0], attn_core_flops=out[1], attn_linear_flops=out[2], ffn_flops=out[3])


def ref_ffn_net_bytes(batch, model=STEP3):
    out = c_double()
    _ref_check(ref().ref_ffn_net_bytes(c_char_p(model), c_longlong(batch), ctypes.byref(out)))
    return out.value


def ref_b_dense_moe(f16, f8, bw, model=STEP3):
    out = (c_longlong * 3)()
    _ref_check(ref().ref_b_dense_moe(c_char_p(model), c_double(f16), c_double(f8), c_double(bw), out))
    return tuple(out)


def ref_derive_stage_times(hw: dict, attn_inst, ffn_inst, micro_batch, n_micro, ctx, model=STEP3, L=61):
    arrs = [(c_double * L)() for _ in range(4)]
    _ref_check(ref().ref_derive_stage_times(
        c_char_p(model), c_char_p(hw["name"].encode()), c_double(hw["f16"]), c_double(hw.get("f8", 0.0)),
        c_double(hw["bw"]), c_double(hw["net"]), c_int(hw.get("gps", 1)), c_double(hw.get("net_eff", 1.0)),
        c_int(attn_inst), c_int(ffn_inst), c_longlong(micro_batch), c_int(n_micro), c_longlong(ctx),
        *arrs, c_int(L)))
    return [np.array(a[:]) for a in arrs]  # attn, fwd, ffn, bwd


def ref_simulate(attn, fwd, ffn, bwd, n_micro, total_batch, total_gpus, token_steps=3, shared_link=False):
    L = len(attn)
    cs = [(c_double * L)(*map(float, v)) for v in (attn, fwd, ffn, bwd)]
    out = (c_double * 10)()
    _ref_check(ref().ref_simulate(*cs, c_int(L), c_int(n_micro), c_longlong(total_batch), c_int(total_gpus),
                                  c_int(token_steps), c_int(int(shared_link)), out))
    return dict(tpot=out[0], tgs=out[1], utilization=list(out[2:6]), bubble=list(out[6:10]))


def ref_analytic_tpot_bound(attn, fwd, ffn, bwd, n_micro):
    L = len(attn)
    cs = [(c_double * L)(*map(float, v)) for v in (attn, fwd, ffn, bwd)]
    out = c_double()
    _ref_check(ref().ref_analytic_tpot_bound(*cs, c_int(L), c_int(n_micro), ctypes.byref(out)))
    return out.value


def ref_trace_csv(attn, fwd, ffn, bwd, n_micro, total_batch, total_gpus) -> str:
    L = len(attn)
    cs = [(c_double * L)(*map(float, v)) for v in (attn, fwd, ffn, bwd)]
    p = ref().ref_trace_csv(*cs, c_int(L), c_int(n_micro), c_longlong(total_batch), c_int(total_gpus))
    s = ctypes.string_at(p).decode()
    ref().ref_free(c_void_p(p))
    return s


def ref_vet_plan(hw: dict, attn_inst, ffn_inst, micro_batch, n_micro, ctx, tpot=0.05, stages=3, model=STEP3):
    """The reference's vet_plan flags (planner.cpp:111-137)."""
    flags = (c_int * 3)()
    _ref_check(ref().ref_vet_plan(
        c_char_p(model), c_char_p(hw["name"].encode()), c_double(hw["f16"]), c_double(hw.get("f8", 0.0)),
        c_double(hw["bw"]), c_double(hw["net"]), c_int(hw.get("gps", 1)), c_double(hw.get("net_eff", 1.0)),
        c_int(attn_inst), c_int(ffn_inst), c_longlong(micro_batch), c_int(n_micro), c_longlong(ctx),
        c_double(tpot), c_int(stages), flags))
    return dict(sparsity_ok=bool(flags[0]), net_ok=bool(flags[1]), stage_ok=bool(flags[2]))


def ref_stage_budget(tpot, stages, layers):
    out = c_double()
    _ref_check(ref().ref_stage_budget(c_double(tpot), c_int(stages), c_int(layers), ctypes.byref(out)))
    return out.value


def _ref_check(rc):
    if rc != 0:
        raise RuntimeError(ref().ref_last_error().decode())


def ref_dump_builtin_catalog() -> str:
    ref().ref_dump_builtin_catalog.restype = c_void_p
    p = ref().ref_dump_builtin_catalog()
    if not p:
        raise RuntimeError(ref().ref_last_error().decode())
    s = ctypes.string_at(p).decode()
    ref().ref_free(ctypes.c_void_p(p))
    return s


def ref_catalog_accel(text: str, name: str) -> dict:
    """The reference's own catalog loader (parse_catalog + validate) on `text`."""
    out = (c_double * 6)()
    _ref_check(ref().ref_catalog_accel(c_char_p(text.encode()), c_char_p(name.encode()), out))
    keys = ["flops_16bit", "flops_8bit", "mem_bw", "net_bw_per_server", "gpus_per_server", "net_efficiency"]
    return dict(zip(keys, list(out)))
