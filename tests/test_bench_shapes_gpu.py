"""Parity at the EXACT shapes bench.py times (VERDICT r1 "next" item 1).

The split-KV partition, the per-request K3 publish counters, the stream-K
GEMM split and the MoE work list all depend on (B, ctx, E, T), so the
configurations behind the reported numbers are checked here, not just
smaller stand-ins:

  * config 2: the attention-side layer at full Step-3 dims, B=64 x 4K, bf16
    KV and e4m3 KV; the MFA core alone at the same shape;
  * config 4: the MFA core at B=32 x 32K (split-KV), bf16 and e4m3 KV;
  * config 3: the MoE layer with all 48 routed experts + the shared expert,
    top-3, T=256 (and the T=4096 / 8192 tensor-bound points), fp8 1x128 and
    MXFP8, with the kernels' default selection (as bench.py runs them).  The
    GPU computes all T tokens; the oracle checks a fixed token subset (a
    token's output depends only on its own row, and the per-row dispatch /
    intermediate quantisation is row-local), fetching one expert's weights at
    a time (oracle.moe_layer_by_expert).

Bars are the same as the small-shape tests (stated there): layer h_res/h_norm
2e-2 (bf16 KV) / 3e-2 (e4m3 KV); core 1e-2 (bf16) / 3e-2 (e4m3); MoE 5e-3
(fp8 1x128) / 1e-2 (MXFP8).  Measured errors go to $PARITY_LOG.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import test_mfa_decode_gpu as core_bf16
from tests import test_mfa_fp8_gpu as core_fp8
from tests import test_mfa_layer_gpu as layer
from tests.helpers import record, rel_err

H, INTER, E, TOPK = 7168, 5120, 48, 3


# ------------------------------------------------------------ attention side
@pytest.mark.gpu
def test_config2_layer_bf16_kv(ctx):
    res = layer.run_layer(ctx, layer.STEP3, [4096] * 64, 2)
    record("config2_layer_bf16", h_res=rel_err(res[0], res[4]), h_norm=rel_err(res[1], res[5]))
    layer.check(res, 64)


@pytest.mark.gpu
def test_config2_layer_e4m3_kv(ctx):
    g_res, g_norm, gk, gv, r_res, r_norm, rk, rv, bt, sl, _ = layer.run_layer_fp8(ctx, layer.STEP3, [4096] * 64, 3)
    record("config2_layer_e4m3", h_res=rel_err(g_res, r_res), h_norm=rel_err(g_norm, r_norm))
    assert rel_err(g_res, r_res) <= 3e-2, rel_err(g_res, r_res)
    assert rel_err(g_norm, r_norm) <= 3e-2, rel_err(g_norm, r_norm)


@pytest.mark.gpu
@pytest.mark.parametrize("B,L", [(64, 4096), (32, 32768)], ids=["config2", "config4"])
def test_core_bf16_bench_shape(ctx, B, L):
    got, lse, ref, ref_lse = core_bf16.run_case(ctx, [L] * B, seed=B, poison=False)
    record(f"core_bf16_B{B}_L{L}", out=rel_err(got, ref), lse=np.max(np.abs(lse - ref_lse)))
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)
    np.testing.assert_allclose(lse, ref_lse, rtol=2e-3, atol=2e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("B,L", [(64, 4096), (32, 32768)], ids=["config2", "config4"])
def test_core_e4m3_bench_shape(ctx, B, L):
    got, lse, ref, ref_lse = core_fp8.run_case(ctx, [L] * B, seed=B, poison=False)
    record(f"core_e4m3_B{B}_L{L}", out=rel_err(got, ref), lse=np.max(np.abs(lse - ref_lse)))
    assert rel_err(got, ref) <= 3e-2, rel_err(got, ref)
    assert np.max(np.abs(lse - ref_lse)) <= 2e-2


# ------------------------------------------------------------------ FFN side
def dev_e4m3(torch, shape, gen):
    """random finite e4m3 codes generated on the device (5.4 GB of experts)."""
    mag = torch.randint(0x18, 0x40, shape, generator=gen, dtype=torch.int32, device="cuda")
    sgn = torch.randint(0, 2, shape, generator=gen, dtype=torch.int32, device="cuda") * 0x80
    return (mag | sgn).to(torch.uint8)


def full_layer_case(ctx, fmt, T, n_check, seed):
    import torch

    gen = torch.Generator(device="cuda").manual_seed(seed)
    n = E + 1
    w = {"n_experts": E, "w13": dev_e4m3(torch, (n, 2 * INTER, H), gen), "w2": dev_e4m3(torch, (n, H, INTER), gen)}
    x = torch.randn(T, H, generator=gen, device="cuda").cpu().numpy()
    logits = torch.randn(T, E, generator=gen, device="cuda").cpu().numpy()
    ids_np, w_np = orc.router_topk(logits, TOPK)
    if fmt == "mx":
        b13, b2 = 127 - 7 - 1, 127 - 6 - 1  # ~1/sqrt(K) so activations stay O(1)
        w["sf13"] = torch.randint(b13 - 1, b13 + 2, (n, 2 * INTER, H // 32), generator=gen, device="cuda").to(torch.uint8)
        w["sf2"] = torch.randint(b2 - 1, b2 + 2, (n, H, INTER // 32), generator=gen, device="cuda").to(torch.uint8)
        xq_np, xs_np = orc.quant_mx(x)
        run = ctx.moe_ffn_mx
    else:
        w["s13"] = (torch.rand(n, 2 * INTER // 128, H // 128, generator=gen, device="cuda") * 0.5 + 0.5) / H ** 0.5
        w["s2"] = (torch.rand(n, H // 128, INTER // 128, generator=gen, device="cuda") * 0.5 + 0.5) / INTER ** 0.5
        xq_np, xs_np = orc.quant_fp8_rowblock(x)
        run = ctx.moe_ffn
    dev = torch.device("cuda:0")
    out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    run(w, torch.from_numpy(xq_np).to(dev), torch.from_numpy(xs_np).to(dev), torch.from_numpy(ids_np).to(dev),
        torch.from_numpy(w_np).to(dev), out)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    assert np.isfinite(got).all()
    rng = np.random.default_rng(seed)
    tokens = np.sort(rng.choice(T, size=n_check, replace=False))

    def expert(e, rows):
        if fmt == "mx":
            return orc.expert_ffn_mx(xq_np[rows], xs_np[rows], w["w13"][e].cpu().numpy(), w["sf13"][e].cpu().numpy(),
                                     w["w2"][e].cpu().numpy(), w["sf2"][e].cpu().numpy())
        return orc.expert_ffn_fp8(xq_np[rows], xs_np[rows], w["w13"][e].cpu().numpy(), w["s13"][e].cpu().numpy(),
                                  w["w2"][e].cpu().numpy(), w["s2"][e].cpu().numpy())

    ref = orc.moe_layer_by_expert(ids_np, w_np, E, expert, tokens=tokens)
    return got[tokens], ref


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,T,n_check", [("fp8", 256, 32), ("mx", 256, 32), ("fp8", 4096, 16),
                                           ("mx", 4096, 16), ("mx", 8192, 12)])
def test_config3_moe_layer_48_experts(ctx, fmt, T, n_check):
    got, ref = full_layer_case(ctx, fmt, T, n_check, seed=T + (fmt == "mx"))
    err = rel_err(got, ref)
    record(f"config3_moe_{fmt}_T{T}", out=err)
    assert err <= (5e-3 if fmt == "fp8" else 1e-2), err
