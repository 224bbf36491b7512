"""Generate the golden fixtures under tests/golden/ (committed).

Inputs are regenerated from seeds (numpy PCG64 is bit-stable across
platforms), so a fixture holds seeds, shapes and the expected OUTPUTS only.
Outputs come from the C oracle (oracle/afd_oracle.c); before a fixture is
written the independent numpy restatement (np_reference.py) must agree with
it, so a fixture pins two independent implementations of the semantics.

    python tests/golden/make_golden.py          # rewrite fixtures
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from tests.golden import np_reference as npr  # noqa: E402

TINY = dict(hidden=64, q_lora=32, n_heads=4, head_dim=32, page=16)
SMALL = dict(hidden=1024, q_lora=256, n_heads=64, head_dim=256, page=64)  # B200 kernel head layout


def layer_inputs(dims, seq_lens, seed):
    """bf16-representable layer inputs (float32 arrays) from a seed."""
    rng = np.random.default_rng(seed)
    H, QL, NH, D, P = dims["hidden"], dims["q_lora"], dims["n_heads"], dims["head_dim"], dims["page"]
    B = len(seq_lens)

    def w(shape, fan_in):
        return npr.bf16((rng.standard_normal(shape) / np.sqrt(fan_in)).astype(np.float32))

    weights = {
        "in_norm": npr.bf16((1.0 + 0.1 * rng.standard_normal(H)).astype(np.float32)),
        "qkv": w((QL + 2 * D, H), H),
        "q_norm": npr.bf16((1.0 + 0.1 * rng.standard_normal(QL)).astype(np.float32)),
        "q_up": w((NH * D, QL), QL),
        "o": w((H, NH * D), NH * D),
        "post_norm": npr.bf16((1.0 + 0.1 * rng.standard_normal(H)).astype(np.float32)),
    }
    x = npr.bf16(rng.standard_normal((B, H)).astype(np.float32))
    need = [(L + P - 1) // P for L in seq_lens]
    num_pages = sum(need) + 2
    perm = rng.permutation(num_pages).astype(np.int32)
    bt = np.zeros((B, max(need)), np.int32)
    k = 0
    for b, n in enumerate(need):
        bt[b, :n] = perm[k:k + n]
        k += n
    kc = npr.bf16(rng.standard_normal((num_pages, P, D)).astype(np.float32))
    vc = npr.bf16(rng.standard_normal((num_pages, P, D)).astype(np.float32))
    return x, weights, kc, vc, bt, np.array(seq_lens, np.int32)


def router_inputs(T, E, seed):
    rng = np.random.default_rng(seed)
    logits = rng.standard_normal((T, E)).astype(np.float32)
    logits[0, 5] = logits[0, 9] = logits[0, 30] = 3.0  # exact 3-way tie at the top
    logits[1, :] = 0.25                                 # all-equal row
    logits[2, 7] = logits[2, 8] = logits[0].max() + 1  # tie for first
    return logits


QUANT_PROBE = np.array([0.0, -0.0, 1.0, -1.0, 448.0, 449.0, 464.0, 500.0, -1e9, 0.0009765625,
                        0.001953125, 0.0029296875, 0.015625, 0.0146484375, 1.0625, 1.1875,
                        1.125 + 1e-7, 240.0, 232.0, 3.0e-7, 17.0, 18.0, 19.0, 0.33], np.float32)


def ffn_inputs(rows, H, I, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, H)).astype(np.float32)
    xq, xs = orc.quant_fp8_rowblock(x)
    w13q, s13 = orc.quant_fp8_tile((rng.standard_normal((2 * I, H)) / np.sqrt(H)).astype(np.float32))
    w2q, s2 = orc.quant_fp8_tile((rng.standard_normal((H, I)) / np.sqrt(I)).astype(np.float32))
    return xq, xs, w13q, s13, w2q, s2


def main():
    fixtures = {}
    # ---- MFA layer, tiny and GPU-shaped small dims
    for name, dims, seq_lens, seed in [("mfa_tiny", TINY, [5, 16, 40], 11),
                                       ("mfa_small", SMALL, [70, 130], 12)]:
        x, w, kc, vc, bt, sl = layer_inputs(dims, seq_lens, seed)
        kc1, vc1 = kc.copy(), vc.copy()
        h_res, h_norm = orc.mfa_layer(dims, x, w, kc1, vc1, bt, sl)
        kc2, vc2 = kc.copy(), vc.copy()
        n_res, n_norm = npr.mfa_layer(dims, x, w, kc2, vc2, bt, sl)
        d_res = float(np.max(np.abs(n_res - h_res)) / np.max(np.abs(h_res)))
        d_norm = float(np.max(np.abs(n_norm - h_norm)) / np.max(np.abs(h_norm)))
        assert d_res < 1e-2 and d_norm < 2e-2, (name, d_res, d_norm)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), h_res=h_res, h_norm=h_norm,
                            seq_lens=sl, seed=seed)
        fixtures[name] = dict(dims=dims, seq_lens=seq_lens, seed=seed, numpy_vs_c=[d_res, d_norm])
    # ---- attention core (K2) at the GPU head layout
    x, w, kc, vc, bt, sl = layer_inputs(SMALL, [1, 64, 65, 300], 13)
    rng = np.random.default_rng(14)
    q = npr.bf16(rng.standard_normal((4, 64, 256)).astype(np.float32))
    out, lse = orc.mfa_decode_attention(q, kc, vc, bt, sl, 256 ** -0.5)
    nout, nlse = npr.mfa_attention(q, kc, vc, bt, sl, 256 ** -0.5)
    assert np.max(np.abs(nout - out)) < 1e-5 and np.max(np.abs(nlse - lse)) < 1e-5
    np.savez_compressed(os.path.join(HERE, "attn_small.npz"), out=out, lse=lse)
    fixtures["attn_small"] = dict(seq_lens=[1, 64, 65, 300], layer_seed=13, q_seed=14)
    # ---- router top-k + permutation (bit-exact)
    logits = router_inputs(64, 48, 21)
    ids, wts = orc.router_topk(logits, 3)
    nids, nwts = npr.router_topk(logits, 3)
    assert np.array_equal(ids, nids) and np.max(np.abs(wts - nwts)) < 1e-6
    offsets, perm, inv = orc.moe_permute(ids, 48)
    no, npm, ni = npr.moe_permute(ids, 48)
    assert np.array_equal(offsets, no) and np.array_equal(perm, npm) and np.array_equal(inv, ni)
    np.savez_compressed(os.path.join(HERE, "router.npz"), ids=ids, weights=wts, offsets=offsets,
                        perm=perm, inv=inv)
    fixtures["router"] = dict(T=64, E=48, k=3, seed=21)
    # ---- FP8 quantization probe values (bit-exact codes)
    codes = np.array([orc.orc().orc_f32_to_e4m3(float(v)) for v in QUANT_PROBE], np.uint8)
    assert np.array_equal(codes, npr.quant_e4m3(QUANT_PROBE)), (codes, npr.quant_e4m3(QUANT_PROBE))
    np.savez_compressed(os.path.join(HERE, "quant.npz"), probe=QUANT_PROBE, codes=codes)
    # ---- one FP8 expert (K7 semantics)
    xq, xs, w13, s13, w2, s2 = ffn_inputs(5, 256, 256, 31)
    y = orc.expert_ffn_fp8(xq, xs, w13, s13, w2, s2)
    ny = npr.expert_ffn_fp8(xq, xs, w13, s13, w2, s2)
    d = float(np.max(np.abs(ny - y)) / np.max(np.abs(y)))
    assert d < 1e-2, d
    np.savez_compressed(os.path.join(HERE, "expert_fp8.npz"), y=y)
    fixtures["expert_fp8"] = dict(rows=5, H=256, I=256, seed=31, numpy_vs_c=d)
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump(fixtures, f, indent=1)
    print(json.dumps(fixtures, indent=1))


if __name__ == "__main__":
    main()
