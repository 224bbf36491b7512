"""Independent numpy restatement of the Step-3 decode semantics.

A second implementation (the pattern of ReferenceEngine,
test_pipesim.cpp:39-107) used only to cross-check the C oracle
(oracle/afd_oracle.c) when the golden fixtures are generated and in the CPU
test suite.  Written from the same semantic sources (
vllm step3_text.py) without sharing code with the C oracle: vectorised
float64 math, explicit bf16 rounding at the B200 storage points.
"""
from __future__ import annotations

import numpy as np


def bf16(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


def rmsnorm(x, w, eps=1e-5):
    x = np.asarray(x, np.float32)
    inv = (1.0 / np.sqrt(np.mean(x.astype(np.float64) ** 2, axis=-1, keepdims=True) + eps)).astype(np.float32)
    return (x * inv) * np.asarray(w, np.float32)


def rope_neox(x, pos, theta):
    d = x.shape[-1]
    half = d // 2
    inv = theta ** (-(2.0 * np.arange(half)) / d)
    ang = pos * inv
    c = np.cos(ang).astype(np.float32)
    s = np.sin(ang).astype(np.float32)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def gather_kv(cache, block_table_row, L, page):
    idx = np.arange(L)
    return cache[block_table_row[idx // page], idx % page]


def mfa_attention(q, k_cache, v_cache, block_table, seq_lens, scale):
    B, H, D = q.shape
    page = k_cache.shape[1]
    out = np.zeros((B, H, D), np.float64)
    lse = np.full((B, H), -np.inf)
    for b in range(B):
        L = int(seq_lens[b])
        if L == 0:
            continue
        K = gather_kv(k_cache, block_table[b], L, page).astype(np.float64)
        V = gather_kv(v_cache, block_table[b], L, page).astype(np.float64)
        s = (q[b].astype(np.float64) @ K.T) * scale  # [H, L]
        m = s.max(axis=1, keepdims=True)
        p = np.exp(s - m)
        l = p.sum(axis=1, keepdims=True)
        out[b] = (p @ V) / l
        lse[b] = (m + np.log(l))[:, 0]
    return out, lse


def mfa_layer(dims, x, w, k_cache, v_cache, block_table, seq_lens):
    """Returns (h_res, h_norm); updates the float32 caches in place."""
    QL, NH, D, page = dims["q_lora"], dims["n_heads"], dims["head_dim"], dims["page"]
    eps, theta = dims.get("rms_eps", 1e-5), dims.get("rope_theta", 5e5)
    scale = dims.get("softmax_scale", D ** -0.5)
    B = x.shape[0]
    xn = bf16(rmsnorm(x, w["in_norm"], eps))
    qkv = bf16((xn.astype(np.float64) @ w["qkv"].T.astype(np.float64)).astype(np.float32))
    qa = bf16(rmsnorm(qkv[:, :QL], w["q_norm"], eps))
    q = bf16((qa.astype(np.float64) @ w["q_up"].T.astype(np.float64)).astype(np.float32)).reshape(B, NH, D)
    k = qkv[:, QL:QL + D]
    v = qkv[:, QL + D:QL + 2 * D]
    for b in range(B):
        pos = int(seq_lens[b]) - 1
        q[b] = bf16(rope_neox(q[b], pos, theta))
        kb = bf16(rope_neox(k[b:b + 1], pos, theta))[0]
        pg = block_table[b, pos // page]
        k_cache[pg, pos % page] = kb
        v_cache[pg, pos % page] = v[b]
    attn, _ = mfa_attention(q, k_cache, v_cache, block_table, seq_lens, scale)
    attn = bf16(attn.astype(np.float32)).reshape(B, NH * D)
    o = (attn.astype(np.float64) @ w["o"].T.astype(np.float64)).astype(np.float32)
    h_res = bf16(x + o)
    h_norm = bf16(rmsnorm(h_res, w["post_norm"], eps))
    return h_res, h_norm


def router_topk(logits, k):
    logits = np.asarray(logits, np.float32)
    T, E = logits.shape
    # stable descending sort: ties keep the lower expert index first
    order = np.argsort(-logits, axis=1, kind="stable")[:, :k].astype(np.int32)
    m = logits.max(axis=1, keepdims=True)
    e = np.exp((logits - m).astype(np.float64))
    p = e / e.sum(axis=1, keepdims=True)
    return order, np.take_along_axis(p, order, axis=1).astype(np.float32)


def moe_permute(ids, E):
    flat = np.asarray(ids).reshape(-1)
    counts = np.bincount(flat, minlength=E)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    perm = np.argsort(flat, kind="stable").astype(np.int32)  # (expert, token, j) order
    inv = np.empty_like(perm)
    inv[perm] = np.arange(flat.size, dtype=np.int32)
    return offsets, perm, inv


E4M3_MAX = 448.0


def e4m3_grid():
    vals = []
    for code in range(256):
        s = -1.0 if code & 0x80 else 1.0
        e = (code >> 3) & 0xF
        m = code & 7
        if e == 15 and m == 7:
            vals.append(np.nan)
        elif e == 0:
            vals.append(s * m / 8.0 * 2.0 ** -6)
        else:
            vals.append(s * (1 + m / 8.0) * 2.0 ** (e - 7))
    return np.array(vals)


def quant_e4m3(x):
    """Nearest-even e4m3 code of each value, saturating at 448 (brute force)."""
    grid = e4m3_grid()
    pos_codes = np.arange(0, 127)  # 0x00..0x7e non-negative finite
    pos_vals = grid[pos_codes]
    a = np.minimum(np.abs(np.asarray(x, np.float64)), E4M3_MAX)
    idx = np.searchsorted(pos_vals, a)
    idx = np.clip(idx, 1, len(pos_vals) - 1)
    lo, hi = pos_vals[idx - 1], pos_vals[idx]
    pick_hi = (a - lo > hi - a) | ((a - lo == hi - a) & (pos_codes[idx] % 2 == 0))
    code = np.where(pick_hi, pos_codes[idx], pos_codes[idx - 1])
    code = np.where(a == 0, 0, code)
    return (code | np.where(np.signbit(x), 0x80, 0)).astype(np.uint8)


def quant_rowblock(x, block=128):
    x = np.asarray(x, np.float32)
    R, C = x.shape
    xb = x.reshape(R, C // block, block)
    scale = (np.maximum(np.abs(xb).max(axis=2), np.float32(1e-10)) / np.float32(448.0)).astype(np.float32)
    q = quant_e4m3((xb / scale[:, :, None]).astype(np.float32)).reshape(R, C)
    return q, scale


def expert_ffn_fp8(xq, xs, w13, s13, w2, s2):
    grid = e4m3_grid()
    I = w2.shape[1]
    x = grid[xq] * np.repeat(xs, 128, axis=1)
    W13 = grid[w13] * np.repeat(np.repeat(s13, 128, axis=0), 128, axis=1)
    gu = x @ W13.T
    g, u = gu[:, :I].astype(np.float32), gu[:, I:].astype(np.float32)
    h = (g / (1.0 + np.exp(-g))) * u
    hq, hs = quant_rowblock(h.astype(np.float32))
    W2 = grid[w2] * np.repeat(np.repeat(s2, 128, axis=0), 128, axis=1)
    return (grid[hq] * np.repeat(hs, 128, axis=1)) @ W2.T
