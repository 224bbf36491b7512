"""CPU suite for the test oracles.

1. The C oracle reproduces the committed golden fixtures and agrees with the
   independent numpy restatement (tests/golden/np_reference.py).
2. Scalar formats (bf16 RNE, e4m3 RNE-saturating) agree with torch.
3. Accounting parity: the oracle's per-layer bytes/FLOPs equal the numbers
   of the reference itself (oracle/_ref/libafdref.so built from
   /root/reference/proj/src), pinning SURVEY.md §8c's accounting rows.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden import make_golden as mg
from tests.golden import np_reference as npr

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIX = json.load(open(os.path.join(GOLD, "fixtures.json")))


# ---------------------------------------------------------------- goldens
@pytest.mark.parametrize("name,dims", [("mfa_tiny", mg.TINY), ("mfa_small", mg.SMALL)])
def test_mfa_layer_golden(name, dims):
    f = np.load(os.path.join(GOLD, f"{name}.npz"))
    x, w, kc, vc, bt, sl = mg.layer_inputs(dims, FIX[name]["seq_lens"], FIX[name]["seed"])
    h_res, h_norm = orc.mfa_layer(dims, x, w, kc, vc, bt, sl)
    np.testing.assert_array_equal(h_res, f["h_res"])
    np.testing.assert_array_equal(h_norm, f["h_norm"])


def test_mfa_layer_numpy_second_implementation():
    dims = mg.TINY
    x, w, kc, vc, bt, sl = mg.layer_inputs(dims, [3, 33, 17, 48], 99)
    k1, v1, k2, v2 = kc.copy(), vc.copy(), kc.copy(), vc.copy()
    a_res, a_norm = orc.mfa_layer(dims, x, w, k1, v1, bt, sl)
    b_res, b_norm = npr.mfa_layer(dims, x, w, k2, v2, bt, sl)
    assert np.max(np.abs(a_res - b_res)) <= 1e-2 * np.max(np.abs(a_res))
    np.testing.assert_array_equal(k1, k2)  # appended K (post-RoPE, bf16) bit-identical
    np.testing.assert_array_equal(v1, v2)


def test_attention_golden():
    f = np.load(os.path.join(GOLD, "attn_small.npz"))
    fx = FIX["attn_small"]
    _, _, kc, vc, bt, sl = mg.layer_inputs(mg.SMALL, fx["seq_lens"], fx["layer_seed"])
    q = npr.bf16(np.random.default_rng(fx["q_seed"]).standard_normal((4, 64, 256)).astype(np.float32))
    out, lse = orc.mfa_decode_attention(q, kc, vc, bt, sl, 256 ** -0.5)
    np.testing.assert_allclose(out, f["out"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(lse, f["lse"], rtol=0, atol=1e-6)


def test_attention_empty_and_single_token():
    rng = np.random.default_rng(0)
    q = rng.standard_normal((2, 4, 8)).astype(np.float32)
    kc = rng.standard_normal((2, 4, 8)).astype(np.float32)
    vc = rng.standard_normal((2, 4, 8)).astype(np.float32)
    bt = np.array([[0], [1]], np.int32)
    out, lse = orc.mfa_decode_attention(q, kc, vc, bt, np.array([0, 1], np.int32), 0.3)
    assert np.all(out[0] == 0) and np.all(np.isneginf(lse[0]))
    np.testing.assert_allclose(out[1], np.broadcast_to(vc[1, 0], (4, 8)), rtol=1e-6)


def test_router_golden_bit_exact():
    f = np.load(os.path.join(GOLD, "router.npz"))
    logits = mg.router_inputs(64, 48, FIX["router"]["seed"])
    ids, wts = orc.router_topk(logits, 3)
    np.testing.assert_array_equal(ids, f["ids"])
    np.testing.assert_array_equal(wts, f["weights"])
    assert list(ids[0]) == [5, 9, 30]  # 3-way tie resolves to ascending expert id
    assert list(ids[1]) == [0, 1, 2]   # all-equal row
    offsets, perm, inv = orc.moe_permute(ids, 48)
    np.testing.assert_array_equal(offsets, f["offsets"])
    np.testing.assert_array_equal(perm, f["perm"])
    np.testing.assert_array_equal(inv, f["inv"])


def test_permutation_is_stable_expert_major():
    rng = np.random.default_rng(5)
    ids = np.stack([rng.permutation(48)[:3] for _ in range(257)]).astype(np.int32)
    offsets, perm, inv = orc.moe_permute(ids, 48)
    flat = ids.reshape(-1)
    assert offsets[-1] == flat.size
    experts = flat[perm]
    assert np.all(np.diff(experts) >= 0)
    for e in range(48):
        seg = perm[offsets[e]:offsets[e + 1]]
        assert np.all(np.diff(seg) > 0)  # token-major (then j) inside an expert
    np.testing.assert_array_equal(inv[perm], np.arange(flat.size))


def test_quant_golden_and_numpy():
    f = np.load(os.path.join(GOLD, "quant.npz"))
    codes = np.array([orc.orc().orc_f32_to_e4m3(float(v)) for v in f["probe"]], np.uint8)
    np.testing.assert_array_equal(codes, f["codes"])
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(20000) * np.exp(rng.uniform(-12, 7, 20000))).astype(np.float32)
    mine = np.array([orc.orc().orc_f32_to_e4m3(float(v)) for v in x], np.uint8)
    np.testing.assert_array_equal(mine, npr.quant_e4m3(x))


def test_e4m3_and_bf16_vs_torch():
    import torch

    rng = np.random.default_rng(4)
    x = (rng.standard_normal(50000) * np.exp(rng.uniform(-10, 6, 50000))).astype(np.float32)
    x = x[np.abs(x) < 448]
    mine = np.array([orc.orc().orc_f32_to_e4m3(float(v)) for v in x], np.uint8)
    theirs = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    np.testing.assert_array_equal(mine, theirs)
    back = orc.e4m3_to_f32(mine)
    np.testing.assert_array_equal(back, torch.from_numpy(mine).view(torch.float8_e4m3fn).float().numpy())
    np.testing.assert_array_equal(orc.bf16_round(x), torch.from_numpy(x).to(torch.bfloat16).float().numpy())


def test_expert_golden_and_numpy():
    f = np.load(os.path.join(GOLD, "expert_fp8.npz"))
    xq, xs, w13, s13, w2, s2 = mg.ffn_inputs(5, 256, 256, FIX["expert_fp8"]["seed"])
    y = orc.expert_ffn_fp8(xq, xs, w13, s13, w2, s2)
    np.testing.assert_allclose(y, f["y"], rtol=0, atol=1e-6)
    ny = npr.expert_ffn_fp8(xq, xs, w13, s13, w2, s2)
    assert np.max(np.abs(ny - y)) <= 1e-2 * np.max(np.abs(y))


def test_moe_layer_matches_per_expert_sum():
    H, I, E, k, T = 256, 128, 4, 2, 9
    rng = np.random.default_rng(8)
    x = rng.standard_normal((T, H)).astype(np.float32)
    xq, xs = orc.quant_fp8_rowblock(x)
    w13 = np.zeros((E + 1, 2 * I, H), np.uint8)
    s13 = np.zeros((E + 1, 2 * I // 128, H // 128), np.float32)
    w2 = np.zeros((E + 1, H, I), np.uint8)
    s2 = np.zeros((E + 1, H // 128, I // 128), np.float32)
    for e in range(E + 1):
        w13[e], s13[e] = orc.quant_fp8_tile(rng.standard_normal((2 * I, H)).astype(np.float32) / 16)
        w2[e], s2[e] = orc.quant_fp8_tile(rng.standard_normal((H, I)).astype(np.float32) / 11)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    ids, wts = orc.router_topk(logits, k)
    out = orc.moe_layer_fp8(xq, xs, ids, wts, w13, s13, w2, s2, round_bf16=False)
    ref = np.zeros((T, H))
    for t in range(T):
        ref[t] += orc.expert_ffn_fp8(xq[t:t + 1], xs[t:t + 1], w13[E], s13[E], w2[E], s2[E])[0]
        for j in range(k):
            e = ids[t, j]
            ref[t] += wts[t, j] * orc.expert_ffn_fp8(xq[t:t + 1], xs[t:t + 1], w13[e], s13[e], w2[e], s2[e])[0]
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)


# ----------------------------------------------------------------- MXFP8
def _np_mx_quant(x):
    """independent restatement: smallest e with amax <= 448*2^e by search"""
    rows, cols = x.shape
    xb = x.reshape(rows, cols // 32, 32).astype(np.float64)
    amax = np.abs(xb).max(axis=2)
    e = np.full(amax.shape, -127, np.int64)
    nz = amax > 0
    e0 = np.floor(np.log2(np.where(nz, amax, 1.0))).astype(np.int64) - 10
    for _ in range(4):
        bump = nz & (amax > 448.0 * np.exp2(e0.astype(np.float64)))
        e0 = e0 + bump
    e = np.where(nz, np.clip(e0, -127, 127), -127)
    scaled = (xb * np.exp2(-e.astype(np.float64))[..., None]).astype(np.float32).reshape(rows, cols)
    return npr.quant_e4m3(scaled).reshape(rows, cols), (e + 127).astype(np.uint8)


def test_mx_quant_vs_independent_numpy():
    rng = np.random.default_rng(11)
    x = (rng.standard_normal((64, 512)) * np.exp2(rng.integers(-30, 30, (64, 1)))).astype(np.float32)
    x[0, :32] = 0.0
    x[1, :32] = 448.0
    x[2, 5] = 448.0 * 1.0000001
    q, sf = orc.quant_mx(x)
    nq, nsf = _np_mx_quant(x)
    np.testing.assert_array_equal(sf, nsf)
    np.testing.assert_array_equal(q, nq)
    assert sf[0, 0] == 0 and sf[1, 0] == 127 and sf[2, 0] == 128
    d = orc.mx_dequant(q, sf)
    blk = np.abs(x).reshape(64, 16, 32).max(axis=2, keepdims=True)
    assert np.all(np.abs(d - x).reshape(64, 16, 32) <= blk * 2.0 ** -4 + 1e-30)


def test_expert_mx_vs_numpy_dequant():
    rng = np.random.default_rng(12)
    rows, H, I = 6, 256, 128
    xq, xsf = orc.quant_mx(rng.standard_normal((rows, H)).astype(np.float32))
    w13, sf13 = orc.quant_mx((rng.standard_normal((2 * I, H)) / 16).astype(np.float32))
    w2, sf2 = orc.quant_mx((rng.standard_normal((H, I)) / 11).astype(np.float32))
    y = orc.expert_ffn_mx(xq, xsf, w13, sf13, w2, sf2)
    xd = orc.mx_dequant(xq, xsf).astype(np.float64)
    gu = xd @ orc.mx_dequant(w13, sf13).astype(np.float64).T
    g, u = gu[:, :I], gu[:, I:]
    h = (g / (1 + np.exp(-g)) * u).astype(np.float32)
    hq, hsf = _np_mx_quant(h)
    ny = orc.mx_dequant(hq, hsf).astype(np.float64) @ orc.mx_dequant(w2, sf2).astype(np.float64).T
    assert np.max(np.abs(ny - y)) <= 1e-2 * np.max(np.abs(ny))


def test_moe_layer_mx_matches_per_expert_sum():
    H, I, E, k, T = 256, 128, 4, 2, 9
    rng = np.random.default_rng(13)
    xq, xsf = orc.quant_mx(rng.standard_normal((T, H)).astype(np.float32))
    w13 = np.zeros((E + 1, 2 * I, H), np.uint8)
    sf13 = np.zeros((E + 1, 2 * I, H // 32), np.uint8)
    w2 = np.zeros((E + 1, H, I), np.uint8)
    sf2 = np.zeros((E + 1, H, I // 32), np.uint8)
    for e in range(E + 1):
        w13[e], sf13[e] = orc.quant_mx((rng.standard_normal((2 * I, H)) / 16).astype(np.float32))
        w2[e], sf2[e] = orc.quant_mx((rng.standard_normal((H, I)) / 11).astype(np.float32))
    ids, wts = orc.router_topk(rng.standard_normal((T, E)).astype(np.float32), k)
    out = orc.moe_layer_mx(xq, xsf, ids, wts, w13, sf13, w2, sf2, round_bf16=False)
    ref = np.zeros((T, H))
    for t in range(T):
        one = lambda e: orc.expert_ffn_mx(xq[t:t + 1], xsf[t:t + 1], w13[e], sf13[e], w2[e], sf2[e])[0]
        ref[t] += one(E)
        for j in range(k):
            ref[t] += wts[t, j] * one(ids[t, j])
    np.testing.assert_allclose(out, ref, rtol=1e-5, atol=1e-5)


# ------------------------------------------------------ accounting parity
STEP3 = dict(hidden=7168, q_lora=2048, n_heads=64, head_dim=256, inter=5120, dense_inter=18432,
             layers=61, moe_layers=56, experts=48, topk=3)


def test_model_card_matches_reference():
    card = orc.ref_model_card()
    assert card["n_layers"] == STEP3["layers"] and card["hidden"] == STEP3["hidden"]
    assert card["n_q_heads"] == STEP3["n_heads"]
    assert card["qk_dim"] == card["v_dim"] == STEP3["head_dim"]
    assert card["kv_token_bytes"] == 512  # one K + one V head of 256 at 8 bit
    per_layer = orc.orc().orc_mfa_linear_params(7168, 2048, 64, 256)
    assert card["attn_linear_params"] == STEP3["layers"] * per_layer == 10_330_046_464


@pytest.mark.parametrize("ctx", [1, 4096, 8192, 32768])
def test_attention_accounting_matches_reference(ctx):
    c = orc.ref_cost_breakdown(ctx)
    L = STEP3["layers"]
    assert c["attn_core_flops"] / L == orc.orc().orc_mfa_core_flops(64, 256, ctx)
    assert c["kv_state_bytes"] / L == orc.orc().orc_mfa_kv_bytes(256, ctx, 1)      # 8-bit KV
    assert 2 * c["kv_state_bytes"] / L == orc.orc().orc_mfa_kv_bytes(256, ctx, 2)  # bf16 KV
    assert c["attn_linear_flops"] / L == 2 * orc.orc().orc_mfa_linear_params(7168, 2048, 64, 256)


def test_ffn_accounting_matches_reference():
    c = orc.ref_cost_breakdown(4096)
    dense = 2.0 * 3 * 7168 * 18432
    moe = orc.orc().orc_moe_flops_per_token(7168, 5120, 3, 1)
    assert c["ffn_flops"] == 5 * dense + 56 * moe
    assert moe == 880_803_840


@pytest.mark.parametrize("T", [1, 256, 2048, 4096])
def test_wire_bytes_match_reference(T):
    assert orc.ref_ffn_net_bytes(T) == orc.orc().orc_afd_wire_bytes(7168, T)


def test_b200_batching_thresholds():
    """b_dense / b_moe (moeplan.cpp:7-15) with datasheet B200 peaks."""
    bd8, bd16, bm = orc.ref_b_dense_moe(2.25e15, 4.5e15, 8e12)
    assert (bd8, bd16, bm) == (282, 141, 3455)


def test_quant_pow2_matches_mx_rule():
    """orc_quant_pow2 (the FP8-KV attention query quantiser) is the MXFP8 rule
    over an arbitrary block: at block 32 it equals orc_quant_mx exactly."""
    rng = np.random.default_rng(14)
    x = (rng.standard_normal((16, 256)) * np.exp2(rng.integers(-20, 20, (16, 1)))).astype(np.float32)
    x[0] = 0.0
    q32, e32 = orc.quant_pow2(x, 32)
    qm, sf = orc.quant_mx(x)
    np.testing.assert_array_equal(q32, qm)
    np.testing.assert_array_equal(e32 + 127, sf.astype(np.int32))
    q, e = orc.quant_pow2(x, 256)
    amax = np.abs(x).max(axis=1)
    nz = amax > 0
    assert np.all(amax[nz] <= 448.0 * np.exp2(e[nz, 0].astype(np.float64)))
    assert np.all(amax[nz] > 448.0 * np.exp2(e[nz, 0].astype(np.float64) - 1))
    assert e[0, 0] == -127
