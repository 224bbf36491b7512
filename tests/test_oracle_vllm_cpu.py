"""The oracle's numeric semantics vs the public Step-3 decoder (vLLM).

tests/golden/vllm_step3.npz was produced by tests/golden/make_vllm_golden.py
from vLLM's own Step-3 building blocks (RMSNorm.forward_native, get_rope NeoX
forward_native, SiluAndMul.forward_native, the torch router select_experts,
Step3TextConfig defaults), so these tests pin eps, RoPE style/theta, softmax
scale, router renormalisation and the SwiGLU/shared-expert combine to an
implementation the builder did not write (VERDICT r1 "parity unpinned").

Bars: fp32 vLLM vs the oracle's double accumulation: rel <= 2e-5 on the layer
outputs and the appended K/V; router ids bit-exact, weights abs <= 1e-6.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import rel_err

FIX = os.path.join(os.path.dirname(__file__), "golden", "vllm_step3.npz")


@pytest.fixture(scope="module")
def g():
    return dict(np.load(FIX))


def test_config_defaults_match_oracle(g):
    """Step3TextConfig defaults == the constants the oracle and kernels use
    (builtin_catalog.cpp:232-255 for the dims)."""
    assert float(g["eps"]) == 1e-5
    assert float(g["theta"]) == 5e5
    assert not bool(g["renorm"])  # norm_expert_weight=False: no top-k renormalisation
    assert int(g["top_k"]) == 3 and int(g["n_experts"]) == 48
    assert int(g["head_dim"]) == 256 and int(g["share_q_dim"]) == 2048
    assert int(g["hidden"]) == 7168 and int(g["moe_inter"]) == 5120 and int(g["share_expert_dim"]) == 5120


def test_mfa_layer_matches_vllm(g):
    HID, QL, NH, HD, PAGE = (int(v) for v in g["dims"])
    dims = dict(hidden=HID, q_lora=QL, n_heads=NH, head_dim=HD, page=PAGE, rms_eps=float(g["eps"]),
                rope_theta=float(g["theta"]), softmax_scale=float(g["scaling"]))
    w = {n: g["w_" + n] for n in ("in_norm", "qkv", "q_norm", "q_up", "o", "post_norm")}
    kc, vc = g["k_cache"].copy(), g["v_cache"].copy()
    h_res, h_norm = orc.mfa_layer(dims, g["x"], w, kc, vc, g["block_table"], g["seq_lens"], round_bf16=False)
    assert rel_err(h_res, g["h_res"]) <= 2e-5, rel_err(h_res, g["h_res"])
    assert rel_err(h_norm, g["h_norm"]) <= 2e-5, rel_err(h_norm, g["h_norm"])
    assert rel_err(kc, g["k_cache_out"]) <= 2e-5  # RoPE(k) at position L-1, appended
    assert rel_err(vc, g["v_cache_out"]) <= 2e-5


def test_mfa_layer_default_dims_are_vllm_semantics(g):
    """The oracle's defaults (eps, theta, scale = head_dim^-0.5) without overrides."""
    HID, QL, NH, HD, PAGE = (int(v) for v in g["dims"])
    dims = dict(hidden=HID, q_lora=QL, n_heads=NH, head_dim=HD, page=PAGE)
    w = {n: g["w_" + n] for n in ("in_norm", "qkv", "q_norm", "q_up", "o", "post_norm")}
    kc, vc = g["k_cache"].copy(), g["v_cache"].copy()
    h_res, _ = orc.mfa_layer(dims, g["x"], w, kc, vc, g["block_table"], g["seq_lens"], round_bf16=False)
    assert rel_err(h_res, g["h_res"]) <= 2e-5


def test_router_matches_vllm_select_experts(g):
    ids, wts = orc.router_topk(g["logits"], int(g["top_k"]), renormalize=bool(g["renorm"]))
    vid, vw = g["topk_ids"], g["topk_w"]
    # torch.topk(sorted=False) order is unspecified: compare per-token (id -> weight) maps
    for t in range(ids.shape[0]):
        o1, o2 = np.argsort(ids[t]), np.argsort(vid[t])
        np.testing.assert_array_equal(ids[t][o1], vid[t][o2])
        np.testing.assert_allclose(wts[t][o1], vw[t][o2], rtol=0, atol=1e-6)


def test_moe_layer_swiglu_shared_matches_vllm(g):
    """SiluAndMul experts, top-k weights from the softmax router, shared expert
    added with weight 1 (share_output + moe_output)."""
    out = orc.moe_layer_f32(g["moe_x"], g["moe_ids"], g["moe_wts"], g["moe_w13"], g["moe_w2"], round_bf16=False)
    assert rel_err(out, g["moe_out"]) <= 2e-5, rel_err(out, g["moe_out"])


def test_moe_by_expert_subset_equals_whole_layer(g):
    """The subset oracle used by the full-size GPU tests equals the C layer."""
    x, ids, w = g["moe_x"], g["moe_ids"], g["moe_wts"]
    E = g["moe_w13"].shape[0] - 1
    whole = orc.moe_layer_f32(x, ids, w, g["moe_w13"], g["moe_w2"], round_bf16=True)
    sub = np.array([1, 4, 7])
    got = orc.moe_layer_by_expert(ids, w, E, lambda e, rows: orc.expert_ffn_f32(x[rows], g["moe_w13"][e],
                                                                                 g["moe_w2"][e], True),
                                  tokens=sub)
    np.testing.assert_array_equal(got, whole[sub])
