"""ctypes binding of include/afdk.h (the C-ABI of the B200 decode hot path).

This is the Python view of the same entry points the C++ host layer
(afd::ops, csrc/afd_ops.cpp) calls.  It carries no fallback: if
libafdk.so is missing or the device is not sm_100, every call raises.
Device tensors are passed as raw pointers (torch is only the allocator).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_float, c_int, c_int32, c_size_t, c_uint32, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AFDK_LIB") or os.path.join(HERE, "libafdk.so")

AFDK_OK = 0
_STATUS = {1: "AFDK_ERR_INVALID", 2: "AFDK_ERR_CUDA", 3: "AFDK_ERR_UNSUPPORTED", 4: "AFDK_ERR_NO_DEVICE"}


class AfdkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class SpecError(AfdkError):
    """Mirrors afd::SpecError (types.hpp:23): a shape/argument invariant failed."""


class Cfg(Structure):
    _fields_ = [("device", c_int), ("num_sms", c_int)]


class MfaDecodeArgs(Structure):
    _fields_ = [
        ("batch", c_int), ("n_heads", c_int), ("head_dim", c_int), ("page_size", c_int),
        ("q", c_void_p), ("k_cache", c_void_p), ("v_cache", c_void_p),
        ("num_pages", c_int), ("block_table", c_void_p), ("max_pages", c_int),
        ("seq_lens", c_void_p), ("softmax_scale", c_float), ("out", c_void_p), ("lse", c_void_p),
    ]


class MfaWeights(Structure):
    _fields_ = [
        ("hidden", c_int), ("q_lora", c_int), ("n_heads", c_int), ("head_dim", c_int),
        ("in_norm", c_void_p), ("w_qkv", c_void_p), ("q_norm", c_void_p), ("w_q_up", c_void_p),
        ("w_o", c_void_p), ("post_norm", c_void_p),
        ("rms_eps", c_float), ("rope_theta", c_float), ("softmax_scale", c_float),
        ("w_o_mx", c_void_p), ("w_o_sf", c_void_p),  # optional MXFP8 o_proj (NULL: bf16 w_o)
        ("w_q_up_mx", c_void_p), ("w_q_up_sf", c_void_p),  # optional MXFP8 q_up (NULL: bf16 w_q_up)
    ]


class MfaLayerArgs(Structure):
    _fields_ = [
        ("batch", c_int), ("x", c_void_p), ("k_cache", c_void_p), ("v_cache", c_void_p),
        ("num_pages", c_int), ("page_size", c_int), ("block_table", c_void_p), ("max_pages", c_int),
        ("seq_lens", c_void_p), ("h_res", c_void_p), ("h_norm", c_void_p),
    ]


class MoeWeights(Structure):
    _fields_ = [
        ("hidden", c_int), ("inter", c_int), ("n_experts", c_int), ("top_k", c_int),
        ("expert_lo", c_int), ("expert_hi", c_int),
        ("w13", c_void_p), ("s13", c_void_p), ("w2", c_void_p), ("s2", c_void_p),
    ]


class MoeArgs(Structure):
    _fields_ = [
        ("T", c_int), ("xq", c_void_p), ("xs", c_void_p), ("ids", c_void_p), ("weights", c_void_p),
        ("shared_lo", c_int), ("shared_hi", c_int), ("out", c_void_p),
    ]


class MoeMxWeights(Structure):
    _fields_ = [
        ("hidden", c_int), ("inter", c_int), ("n_experts", c_int), ("top_k", c_int),
        ("expert_lo", c_int), ("expert_hi", c_int),
        ("w13", c_void_p), ("sf13", c_void_p), ("w2", c_void_p), ("sf2", c_void_p),
    ]


class MoeMxArgs(Structure):
    _fields_ = [
        ("T", c_int), ("xq", c_void_p), ("xsf", c_void_p), ("ids", c_void_p), ("weights", c_void_p),
        ("shared_lo", c_int), ("shared_hi", c_int), ("out", c_void_p),
    ]


class MoeBf16Weights(Structure):
    _fields_ = [
        ("hidden", c_int), ("inter", c_int), ("n_experts", c_int), ("top_k", c_int),
        ("expert_lo", c_int), ("expert_hi", c_int), ("w13", c_void_p), ("w2", c_void_p),
    ]


class MoeBf16Args(Structure):
    _fields_ = [
        ("T", c_int), ("x", c_void_p), ("ids", c_void_p), ("weights", c_void_p),
        ("shared_lo", c_int), ("shared_hi", c_int), ("out", c_void_p),
    ]


class DenseMxWeights(Structure):
    _fields_ = [("hidden", c_int), ("inter_split", c_int), ("n_split", c_int),
                ("w13", c_void_p), ("sf13", c_void_p), ("w2", c_void_p), ("sf2", c_void_p)]


class RowScatter(Structure):
    _fields_ = [("n_dst", c_int), ("rows_per_dst", c_int), ("dst", c_void_p)]


class StagePlan(Structure):
    _fields_ = [("attn_gpus", c_int), ("ffn_gpus", c_int), ("micro_batch", ctypes.c_longlong),
                ("avg_ctx", ctypes.c_longlong), ("n_layers", c_int), ("hidden", c_int), ("link_gbs", ctypes.c_double),
                ("ffn_format", c_int), ("kv_bytes", c_int)]


class LayerTimes(Structure):
    _fields_ = [("attn_s", ctypes.c_double), ("moe_ffn_s", ctypes.c_double), ("dense_ffn_s", ctypes.c_double),
                ("comm_fwd_s", ctypes.c_double), ("comm_bwd_s", ctypes.c_double), ("link_gbs", ctypes.c_double),
                ("attn_batch", ctypes.c_longlong), ("ffn_tokens", ctypes.c_longlong), ("local_experts", c_int),
                ("link_measured", c_int)]


class SimPlan(Structure):
    _fields_ = [("n_micro", c_int), ("total_batch", ctypes.c_longlong), ("total_gpus", c_int),
                ("token_steps", c_int), ("shared_link", c_int)]


class StageCheck(Structure):
    _fields_ = [("stage_ok", c_int), ("first_bad_layer", c_int), ("budget_s", ctypes.c_double),
                ("worst_attn_s", ctypes.c_double), ("worst_ffn_s", ctypes.c_double)]


class SimResult(Structure):
    _fields_ = [("tpot", ctypes.c_double), ("tgs", ctypes.c_double), ("utilization", ctypes.c_double * 4),
                ("bubble_fraction", ctypes.c_double * 4)]


# exported symbol -> (restype, argtypes); the CPU test checks every symbol of
# include/afdk.h is present in the built library
SIGNATURES = {
    "afdk_abi_version": (c_int, []),
    "afdk_last_error": (c_char_p, []),
    "afdk_create": (c_int, [POINTER(c_void_p), POINTER(Cfg)]),
    "afdk_destroy": (None, [c_void_p]),
    "afdk_num_sms": (c_int, [c_void_p]),
    "afdk_ctx_device": (c_int, [c_void_p]),
    "afdk_mfa_decode_attention": (c_int, [c_void_p, POINTER(MfaDecodeArgs), c_void_p]),
    "afdk_linear": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]),
    "afdk_linear_mx": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                               c_void_p]),
    "afdk_mfa_layer": (c_int, [c_void_p, POINTER(MfaWeights), POINTER(MfaLayerArgs), c_void_p]),
    "afdk_router_topk": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "afdk_moe_permute": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "afdk_moe_ffn": (c_int, [c_void_p, POINTER(MoeWeights), POINTER(MoeArgs), c_void_p]),
    "afdk_mfa_layer_mtp": (c_int, [c_void_p, POINTER(MfaWeights), POINTER(MfaLayerArgs), c_int, c_void_p]),
    "afdk_mfa_layer_fp8": (c_int, [c_void_p, POINTER(MfaWeights), POINTER(MfaLayerArgs), c_float, c_float,
                                   c_void_p]),
    "afdk_mfa_decode_attention_mtp": (c_int, [c_void_p, POINTER(MfaDecodeArgs), c_int, c_void_p]),
    "afdk_mfa_decode_attention_fp8": (c_int, [c_void_p, POINTER(MfaDecodeArgs), c_float, c_float, c_void_p]),
    "afdk_moe_ffn_scatter": (c_int, [c_void_p, POINTER(MoeWeights), POINTER(MoeArgs), POINTER(RowScatter),
                                     c_void_p]),
    "afdk_moe_ffn_mx_scatter": (c_int, [c_void_p, POINTER(MoeMxWeights), POINTER(MoeMxArgs), POINTER(RowScatter),
                                        c_void_p]),
    "afdk_moe_ffn_mx": (c_int, [c_void_p, POINTER(MoeMxWeights), POINTER(MoeMxArgs), c_void_p]),
    "afdk_moe_ffn_bf16": (c_int, [c_void_p, POINTER(MoeBf16Weights), POINTER(MoeBf16Args), c_void_p]),
    "afdk_moe_ffn_bf16_scatter": (c_int, [c_void_p, POINTER(MoeBf16Weights), POINTER(MoeBf16Args),
                                          POINTER(RowScatter), c_void_p]),
    "afdk_dense_ffn_mx": (c_int, [c_void_p, POINTER(DenseMxWeights), c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "afdk_dense_ffn_mx_scatter": (c_int, [c_void_p, POINTER(DenseMxWeights), c_int, c_void_p, c_void_p,
                                          POINTER(RowScatter), c_void_p]),
    "afdk_quant_mx": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "afdk_ipc_handle": (c_int, [c_void_p, c_void_p, c_void_p]),
    "afdk_ipc_open": (c_int, [c_void_p, c_void_p, POINTER(c_void_p)]),
    "afdk_ipc_close": (c_int, [c_void_p, c_void_p]),
    "afdk_copy": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "afdk_signal": (c_int, [c_void_p, c_void_p, ctypes.c_uint32, c_void_p]),
    "afdk_wait": (c_int, [c_void_p, c_void_p, ctypes.c_uint32, c_void_p]),
    "afdk_add_partials": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_size_t, c_void_p, c_void_p]),
    "afdk_measure_stage_times": (c_int, [c_void_p, POINTER(StagePlan), c_void_p, c_void_p, c_void_p, c_void_p,
                                         POINTER(LayerTimes)]),
    "afdk_simulate": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, POINTER(SimPlan), POINTER(SimResult)]),
    "afdk_trace_csv": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, POINTER(SimPlan), c_void_p, c_size_t,
                               POINTER(c_size_t)]),
    "afdk_vet_stages": (c_int, [c_void_p, c_void_p, c_int, ctypes.c_double, c_int, c_int, POINTER(StageCheck)]),
}

# ------------------------------------------------ AFD runtime (afdk_afd_*)
class AfdCfg(Structure):
    _fields_ = [("n_attn", c_int), ("n_ffn", c_int), ("n_micro", c_int), ("T_mb", c_int), ("hidden", c_int),
                ("top_k", c_int), ("n_experts", c_int), ("inter", c_int), ("dense_inter", c_int),
                ("dense_slices", c_int), ("ffn_format", c_int), ("layer_kind", c_int), ("f2a", c_int),
                ("attn_chunk", c_int)]


class AfdOp(Structure):
    _fields_ = [("kind", c_int), ("stream", c_int), ("mb", c_int), ("peer", c_int), ("slot", c_int),
                ("value", c_uint32), ("src_buf", c_int), ("dst_buf", c_int), ("src_off", c_size_t),
                ("dst_off", c_size_t), ("bytes", c_size_t)]


class AfdLayout(Structure):
    _fields_ = [("off", c_size_t * 4), ("size", c_size_t * 4), ("total", c_size_t), ("rx_off", c_size_t * 4),
                ("rx_total", c_size_t), ("part_bytes", c_size_t)]


class AfdAttnMb(Structure):
    _fields_ = [("x", c_void_p), ("k_cache", c_void_p), ("v_cache", c_void_p), ("num_pages", c_int),
                ("page_size", c_int), ("max_pages", c_int), ("block_table", c_void_p), ("seq_lens", c_void_p),
                ("k_scale", c_float), ("v_scale", c_float)]


class AfdFfnWeights(Structure):
    _fields_ = [("w13", c_void_p), ("s13", c_void_p), ("w2", c_void_p), ("s2", c_void_p)]


ALLGATHER = ctypes.CFUNCTYPE(c_int, c_void_p, c_void_p, c_size_t, c_void_p)

_SIGS = {
    "afdk_nvls_supported": (c_int, [c_void_p]),
    "afdk_nvls_create": (c_int, [c_void_p, c_int, c_size_t, c_int, c_int, POINTER(c_void_p), POINTER(c_int)]),
    "afdk_nvls_bind": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "afdk_nvls_size": (c_size_t, [c_void_p]),
    "afdk_nvls_destroy": (None, [c_void_p]),
    "afdk_nvls_reduce_bf16": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "afdk_afd_check_cfg": (c_int, [POINTER(AfdCfg)]),
    "afdk_afd_get_layout": (c_int, [POINTER(AfdCfg), POINTER(AfdLayout)]),
    "afdk_afd_plan": (c_int, [POINTER(AfdCfg), c_int, c_uint32, c_void_p, c_int, POINTER(c_int)]),
    "afdk_afd_create": (c_int, [POINTER(c_void_p), POINTER(AfdCfg), c_int, ALLGATHER, c_void_p, POINTER(c_void_p)]),
    "afdk_afd_destroy": (None, [c_void_p]),
    "afdk_afd_attn_layer": (c_int, [c_void_p, POINTER(MfaWeights), c_void_p, POINTER(AfdAttnMb)]),
    "afdk_afd_ffn_layer": (c_int, [c_void_p, POINTER(AfdFfnWeights)]),
    "afdk_afd_stream": (c_void_p, [c_void_p, c_int]),
    "afdk_afd_buffer": (c_void_p, [c_void_p, c_int, c_int]),
    "afdk_afd_seq": (c_uint32, [c_void_p]),
    "afdk_afd_sync": (c_int, [c_void_p]),
    "afdk_afd_trace_start": (c_int, [c_void_p]),
    "afdk_afd_trace_csv": (c_int, [c_void_p, c_void_p, c_size_t, POINTER(c_size_t)]),
}
SIGNATURES.update(_SIGS)



_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != AFDK_OK:
        msg = load().afdk_last_error().decode()
        raise (SpecError if status == 1 else AfdkError)(status, msg)


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return 0 if t is None else int(t.data_ptr())


def simulate(attn, fwd, ffn, bwd, n_micro, total_batch, total_gpus, token_steps=3, shared_link=False) -> dict:
    """Pipeline model (pipesim.cpp:155-237 semantics) on given per-layer stage times; CPU only."""
    L = len(attn)
    arrs = [(ctypes.c_double * L)(*map(float, v)) for v in (attn, fwd, ffn, bwd)]
    out = SimResult()
    check(load().afdk_simulate(*[ctypes.cast(a, c_void_p) for a in arrs], L,
                               ctypes.byref(SimPlan(n_micro, total_batch, total_gpus, token_steps, int(shared_link))),
                               ctypes.byref(out)))
    return dict(tpot=out.tpot, tgs=out.tgs, utilization=list(out.utilization), bubble=list(out.bubble_fraction))


def trace_csv(attn, fwd, ffn, bwd, n_micro, total_batch, total_gpus, token_steps=3, shared_link=False) -> str:
    """trace_csv (pipesim.cpp:239-260 schema) of the product's simulate; CPU only."""
    L = len(attn)
    arrs = [ctypes.cast((ctypes.c_double * L)(*map(float, v)), c_void_p) for v in (attn, fwd, ffn, bwd)]
    plan = SimPlan(n_micro, total_batch, total_gpus, token_steps, int(shared_link))
    n = c_size_t(0)
    check(load().afdk_trace_csv(*arrs, L, ctypes.byref(plan), None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    check(load().afdk_trace_csv(*arrs, L, ctypes.byref(plan), buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def vet_stages(attn, ffn, tpot_sla=0.05, pipeline_stages=3, n_model_layers=None) -> dict:
    """vet_plan's stage_ok (planner.cpp:124-131) on given per-layer attn/ffn stage seconds; CPU only."""
    L = len(attn)
    a = (ctypes.c_double * L)(*map(float, attn))
    f = (ctypes.c_double * L)(*map(float, ffn))
    out = StageCheck()
    check(load().afdk_vet_stages(a, f, L, tpot_sla, pipeline_stages, n_model_layers or L, ctypes.byref(out)))
    return dict(stage_ok=bool(out.stage_ok), first_bad_layer=out.first_bad_layer, budget_s=out.budget_s,
                worst_attn_s=out.worst_attn_s, worst_ffn_s=out.worst_ffn_s)


class Context:
    """RAII wrapper of afdk_ctx (afdk_create / afdk_destroy)."""

    def __init__(self, device: int = 0, num_sms: int = 0):
        self.lib = load()
        h = c_void_p()
        check(self.lib.afdk_create(ctypes.byref(h), ctypes.byref(Cfg(device, num_sms))))
        self.handle = h

    @property
    def num_sms(self) -> int:
        return self.lib.afdk_num_sms(self.handle)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.afdk_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- K2 + K3
    def mfa_decode_attention(self, q, k_cache, v_cache, block_table, seq_lens, out,
                             softmax_scale: float, lse=None, stream: int = 0) -> None:
        B, H, D = q.shape
        a = MfaDecodeArgs(B, H, D, k_cache.shape[1], ptr(q), ptr(k_cache), ptr(v_cache),
                          k_cache.shape[0], ptr(block_table), block_table.shape[1], ptr(seq_lens),
                          softmax_scale, ptr(out), ptr(lse))
        check(self.lib.afdk_mfa_decode_attention(self.handle, ctypes.byref(a), c_void_p(stream)))

    def mfa_decode_attention_mtp(self, q, k_cache, v_cache, block_table, seq_lens, out, softmax_scale: float,
                                 lse=None, stream: int = 0) -> None:
        """q/out [B, mtp, H, D]: the mtp newest tokens of each request (causal among them)."""
        B, mtp, H, D = q.shape
        a = MfaDecodeArgs(B, H, D, k_cache.shape[1], ptr(q), ptr(k_cache), ptr(v_cache),
                          k_cache.shape[0], ptr(block_table), block_table.shape[1], ptr(seq_lens),
                          softmax_scale, ptr(out), ptr(lse))
        check(self.lib.afdk_mfa_decode_attention_mtp(self.handle, ctypes.byref(a), mtp, c_void_p(stream)))

    def mfa_decode_attention_fp8(self, q, k_cache, v_cache, block_table, seq_lens, out, softmax_scale: float,
                                 k_scale: float, v_scale: float, lse=None, stream: int = 0) -> None:
        """e4m3 KV cache (uint8 codes) dequantised by per-tensor k_scale / v_scale."""
        B, H, D = q.shape
        a = MfaDecodeArgs(B, H, D, k_cache.shape[1], ptr(q), ptr(k_cache), ptr(v_cache),
                          k_cache.shape[0], ptr(block_table), block_table.shape[1], ptr(seq_lens),
                          softmax_scale, ptr(out), ptr(lse))
        check(self.lib.afdk_mfa_decode_attention_fp8(self.handle, ctypes.byref(a), c_float(k_scale),
                                                     c_float(v_scale), c_void_p(stream)))

    # ------------------------------------------------------------ K1/K4
    def linear(self, x, w, out, stream: int = 0) -> None:
        import torch

        m, k = x.shape
        n = w.shape[0]
        check(self.lib.afdk_linear(self.handle, ptr(x), ptr(w), ptr(out), m, n, k,
                                   int(out.dtype == torch.float32), c_void_p(stream)))

    def linear_mx(self, xq, xsf, wq, wsf, out, stream: int = 0) -> None:
        """MXFP8 projection: xq/wq e4m3 codes (uint8), xsf/wsf UE8M0 [rows, K/32]."""
        import torch

        m, k = xq.shape
        n = wq.shape[0]
        check(self.lib.afdk_linear_mx(self.handle, ptr(xq), ptr(xsf), ptr(wq), ptr(wsf), ptr(out), m, n, k,
                                      int(out.dtype == torch.float32), c_void_p(stream)))

    def mfa_layer(self, w: dict, x, k_cache, v_cache, block_table, seq_lens, h_res, h_norm,
                  rms_eps=1e-5, rope_theta=5e5, softmax_scale=None, stream: int = 0, kv_scales=None,
                  mtp: int = 1) -> None:
        """Attention-side decode layer; `w` holds bf16 device tensors
        in_norm, qkv, q_norm, q_up, o, post_norm (shapes as in include/afdk.h)."""
        hidden = x.shape[1]
        q_lora = w["q_norm"].shape[0]
        head_dim = k_cache.shape[2]
        n_heads = (w["q_up"] if "q_up" in w else w["q_up_mx"]).shape[0] // head_dim
        scale = head_dim ** -0.5 if softmax_scale is None else softmax_scale
        mw = MfaWeights(hidden, q_lora, n_heads, head_dim, ptr(w["in_norm"]), ptr(w["qkv"]), ptr(w["q_norm"]),
                        ptr(w["q_up"]) if "q_up" in w else None, ptr(w["o"]) if "o" in w else None, ptr(w["post_norm"]),
                        rms_eps, rope_theta, scale, ptr(w["o_mx"]) if "o_mx" in w else None,
                        ptr(w["o_sf"]) if "o_sf" in w else None, ptr(w["q_up_mx"]) if "q_up_mx" in w else None,
                        ptr(w["q_up_sf"]) if "q_up_sf" in w else None)
        a = MfaLayerArgs(x.shape[0] // mtp, ptr(x), ptr(k_cache), ptr(v_cache), k_cache.shape[0], k_cache.shape[1],
                         ptr(block_table), block_table.shape[1], ptr(seq_lens), ptr(h_res), ptr(h_norm))
        if mtp != 1:  # x / h_res / h_norm rows are (request, token)
            check(self.lib.afdk_mfa_layer_mtp(self.handle, ctypes.byref(mw), ctypes.byref(a), mtp, c_void_p(stream)))
        elif kv_scales is None:
            check(self.lib.afdk_mfa_layer(self.handle, ctypes.byref(mw), ctypes.byref(a), c_void_p(stream)))
        else:  # e4m3 caches (uint8 codes) with per-tensor (k_scale, v_scale)
            check(self.lib.afdk_mfa_layer_fp8(self.handle, ctypes.byref(mw), ctypes.byref(a),
                                              c_float(kv_scales[0]), c_float(kv_scales[1]), c_void_p(stream)))

    # -------------------------------------------------------- K5/K6/K7-K9
    def router_topk(self, h, gate_w, k, ids, weights, logits=None, xq=None, xs=None, renormalize=False,
                    stream: int = 0) -> None:
        T, Hd = h.shape
        E = gate_w.shape[0]
        check(self.lib.afdk_router_topk(self.handle, ptr(h), ptr(gate_w), T, Hd, E, k, int(renormalize),
                                        ptr(logits), ptr(ids), ptr(weights), ptr(xq), ptr(xs), c_void_p(stream)))

    def moe_permute(self, ids, n_experts, offsets, perm, inv, stream: int = 0) -> None:
        T, k = ids.shape
        check(self.lib.afdk_moe_permute(self.handle, ptr(ids), T, k, n_experts, ptr(offsets), ptr(perm),
                                        ptr(inv), c_void_p(stream)))

    def moe_ffn(self, w: dict, xq, xs, ids, weights, out, expert_lo=0, expert_hi=None, shared=(0, None),
                stream: int = 0, scatter=None) -> None:
        """w: n_experts, w13, s13, w2, s2 (local experts then the shared one)."""
        T, Hd = xq.shape
        k = ids.shape[1]
        inter = w["w2"].shape[2]
        E = w["n_experts"]
        hi = E if expert_hi is None else expert_hi
        sh_lo, sh_hi = shared[0], (T if shared[1] is None else shared[1])
        mw = MoeWeights(Hd, inter, E, k, expert_lo, hi, ptr(w["w13"]), ptr(w["s13"]), ptr(w["w2"]), ptr(w["s2"]))
        a = MoeArgs(T, ptr(xq), ptr(xs), ptr(ids), ptr(weights), sh_lo, sh_hi, ptr(out))
        if scatter is None:
            check(self.lib.afdk_moe_ffn(self.handle, ctypes.byref(mw), ctypes.byref(a), c_void_p(stream)))
        else:  # (dst device int64 tensor of peer row-block pointers, rows_per_dst)
            sc = RowScatter(scatter[0].numel(), scatter[1], ptr(scatter[0]))
            check(self.lib.afdk_moe_ffn_scatter(self.handle, ctypes.byref(mw), ctypes.byref(a), ctypes.byref(sc),
                                                c_void_p(stream)))

    def moe_ffn_mx(self, w: dict, xq, xsf, ids, weights, out, expert_lo=0, expert_hi=None, shared=(0, None),
                   stream: int = 0, scatter=None) -> None:
        """MXFP8 path. w: n_experts, w13, sf13, w2, sf2 (local experts then the shared one)."""
        T, Hd = xq.shape
        k = ids.shape[1]
        inter = w["w2"].shape[2]
        E = w["n_experts"]
        hi = E if expert_hi is None else expert_hi
        sh_lo, sh_hi = shared[0], (T if shared[1] is None else shared[1])
        mw = MoeMxWeights(Hd, inter, E, k, expert_lo, hi, ptr(w["w13"]), ptr(w["sf13"]), ptr(w["w2"]), ptr(w["sf2"]))
        a = MoeMxArgs(T, ptr(xq), ptr(xsf), ptr(ids), ptr(weights), sh_lo, sh_hi, ptr(out))
        if scatter is None:
            check(self.lib.afdk_moe_ffn_mx(self.handle, ctypes.byref(mw), ctypes.byref(a), c_void_p(stream)))
        else:
            sc = RowScatter(scatter[0].numel(), scatter[1], ptr(scatter[0]))
            check(self.lib.afdk_moe_ffn_mx_scatter(self.handle, ctypes.byref(mw), ctypes.byref(a), ctypes.byref(sc),
                                                   c_void_p(stream)))

    def moe_ffn_bf16(self, w: dict, x, ids, weights, out, expert_lo=0, expert_hi=None, shared=(0, None),
                     stream: int = 0, scatter=None) -> None:
        """16-bit experts. w: n_experts, w13 [n+1, 2I, H] bf16, w2 [n+1, H, I] bf16; x bf16 [T, H]."""
        T, Hd = x.shape
        k = ids.shape[1]
        inter = w["w2"].shape[2]
        E = w["n_experts"]
        hi = E if expert_hi is None else expert_hi
        sh_lo, sh_hi = shared[0], (T if shared[1] is None else shared[1])
        mw = MoeBf16Weights(Hd, inter, E, k, expert_lo, hi, ptr(w["w13"]), ptr(w["w2"]))
        a = MoeBf16Args(T, ptr(x), ptr(ids), ptr(weights), sh_lo, sh_hi, ptr(out))
        if scatter is None:
            check(self.lib.afdk_moe_ffn_bf16(self.handle, ctypes.byref(mw), ctypes.byref(a), c_void_p(stream)))
        else:
            sc = RowScatter(scatter[0].numel(), scatter[1], ptr(scatter[0]))
            check(self.lib.afdk_moe_ffn_bf16_scatter(self.handle, ctypes.byref(mw), ctypes.byref(a),
                                                     ctypes.byref(sc), c_void_p(stream)))

    def dense_ffn_mx(self, w: dict, xq, xsf, out, stream: int = 0, scatter=None) -> None:
        """Dense FFN in slice layout: w13 [n_split, 2*Is, H], sf13, w2 [n_split, H, Is], sf2."""
        T, Hd = xq.shape
        n_split, _, Is = w["w2"].shape
        dw = DenseMxWeights(Hd, Is, n_split, ptr(w["w13"]), ptr(w["sf13"]), ptr(w["w2"]), ptr(w["sf2"]))
        if scatter is None:
            check(self.lib.afdk_dense_ffn_mx(self.handle, ctypes.byref(dw), T, ptr(xq), ptr(xsf), ptr(out),
                                             c_void_p(stream)))
        else:
            sc = RowScatter(scatter[0].numel(), scatter[1], ptr(scatter[0]))
            check(self.lib.afdk_dense_ffn_mx_scatter(self.handle, ctypes.byref(dw), T, ptr(xq), ptr(xsf),
                                                     ctypes.byref(sc), c_void_p(stream)))

    @staticmethod
    def dense_split_layout(w13, sf13, w2, sf2, n_split):
        """Re-lay standard dense weights (w13 [2I, H] gate rows then up rows,
        w2 [H, I]) into the slice layout of afdk_dense_ffn_mx (torch or numpy)."""
        I = w2.shape[1]
        Is = I // n_split

        def cat(a, b):
            import numpy as np
            return np.concatenate([a, b]) if isinstance(a, np.ndarray) else __import__("torch").cat([a, b])

        def stack(parts):
            import numpy as np
            return np.stack(parts) if isinstance(parts[0], np.ndarray) else __import__("torch").stack(parts)

        out = {}
        for name, t, blk in (("w13", w13, 1), ("sf13", sf13, 1)):
            out[name] = stack([cat(t[j * Is:(j + 1) * Is], t[I + j * Is:I + (j + 1) * Is]) for j in range(n_split)])
        out["w2"] = stack([w2[:, j * Is:(j + 1) * Is] for j in range(n_split)])
        out["sf2"] = stack([sf2[:, j * Is // 32:(j + 1) * Is // 32] for j in range(n_split)])
        for k in out:
            out[k] = out[k].contiguous() if hasattr(out[k], "contiguous") else out[k]
        return out

    def quant_mx(self, x, q, sf, stream: int = 0) -> None:
        T, Hd = x.shape
        check(self.lib.afdk_quant_mx(self.handle, ptr(x), T, Hd, ptr(q), ptr(sf), c_void_p(stream)))

    # ------------------------------------------------------- C1/C2 exchange
    def ipc_handle(self, t) -> bytes:
        buf = ctypes.create_string_buffer(72)
        check(self.lib.afdk_ipc_handle(self.handle, ptr(t), buf))
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        out = c_void_p()
        check(self.lib.afdk_ipc_open(self.handle, ctypes.create_string_buffer(handle, 72), ctypes.byref(out)))
        return out.value

    def ipc_close(self, dev_ptr: int) -> None:
        check(self.lib.afdk_ipc_close(self.handle, c_void_p(dev_ptr)))

    def copy(self, dst: int, src: int, nbytes: int, stream: int = 0) -> None:
        check(self.lib.afdk_copy(self.handle, c_void_p(dst), c_void_p(src), nbytes, c_void_p(stream)))

    def signal(self, flag_ptr: int, value: int, stream: int = 0) -> None:
        check(self.lib.afdk_signal(self.handle, c_void_p(flag_ptr), value, c_void_p(stream)))

    def wait(self, flag_ptr: int, value: int, stream: int = 0) -> None:
        check(self.lib.afdk_wait(self.handle, c_void_p(flag_ptr), value, c_void_p(stream)))

    def add_partials(self, base, parts_dev, n: int, out, stream: int = 0) -> None:
        check(self.lib.afdk_add_partials(self.handle, ptr(base), ptr(parts_dev), n, out.numel(), ptr(out),
                                         c_void_p(stream)))

    # -------------------------------------------------- measured stage times
    def measure_stage_times(self, attn_gpus, ffn_gpus, micro_batch, avg_ctx, n_layers=61, hidden=7168,
                            link_gbs=0.0, ffn_format="fp8", kv="bf16") -> dict:
        """ffn_format: fp8 (1x128) / mx / bf16; kv: bf16 / e4m3 (afdk_stage_plan)."""
        L = n_layers
        arrs = [(ctypes.c_double * L)() for _ in range(4)]
        det = LayerTimes()
        fmt = {"fp8": 0, "mx": 1, "bf16": 2}[ffn_format]
        sp = StagePlan(attn_gpus, ffn_gpus, micro_batch, avg_ctx, L, hidden, link_gbs, fmt, 1 if kv == "e4m3" else 2)
        check(self.lib.afdk_measure_stage_times(
            self.handle, ctypes.byref(sp),
            *[ctypes.cast(a, c_void_p) for a in arrs], ctypes.byref(det)))
        names = ["attn", "comm_fwd", "ffn", "comm_bwd"]
        res = {n: list(a) for n, a in zip(names, arrs)}
        res["detail"] = {f: getattr(det, f) for f, _ in LayerTimes._fields_}
        return res
