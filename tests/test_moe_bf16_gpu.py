"""16-bit MoE FFN path (grouped bf16 expert GEMMs on tcgen05 kind::f16) vs the
CPU oracle (orc_moe_layer_f32 with round_bf16: bf16 inputs/weights, the
SwiGLU intermediate stored bf16, fp32 accumulation, bf16 output).

Stated bar: max|gpu-ref|/max|ref| <= 1e-2 (bf16 output: one ulp at the
largest element is 3.9e-3 of this norm; an intermediate rounding flip from
the fast-exp SiLU moves one bf16 ulp of h).  Routing semantics as the FP8
paths (experts [lo, hi) routed, shared expert over [shared_lo, shared_hi)).
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import record, rel_err

TOL = 1e-2


def make_case(T, H, I, E, k, seed, dev="cuda"):
    import torch

    g = torch.Generator(device=dev).manual_seed(seed)
    w13 = (torch.randn(E + 1, 2 * I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E + 1, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)
    x = torch.randn(T, H, generator=g, device=dev).to(torch.bfloat16)
    ids, wts = orc.router_topk(torch.randn(T, E, generator=g, device=dev).cpu().numpy(), k)
    return w13, w2, x, ids, wts


def run_bf16(ctx, T, H, I, E, k, seed, ranges=None):
    import torch

    dev = torch.device("cuda:0")
    w13, w2, x, ids_np, w_np = make_case(T, H, I, E, k, seed)
    ids, wts = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
    if ranges is None:
        out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        ctx.moe_ffn_bf16({"n_experts": E, "w13": w13, "w2": w2}, x, ids, wts, out)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
    else:
        got = np.zeros((T, H), np.float32)
        for (lo, hi), (slo, shi) in ranges:
            sub = {"n_experts": E, "w13": torch.cat([w13[lo:hi], w13[E:]]), "w2": torch.cat([w2[lo:hi], w2[E:]])}
            out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
            ctx.moe_ffn_bf16(sub, x, ids, wts, out, expert_lo=lo, expert_hi=hi, shared=(slo, shi))
            torch.cuda.synchronize()
            got += out.float().cpu().numpy()
    ref = orc.moe_layer_f32(x.float().cpu().numpy(), ids_np, w_np, w13.float().cpu().numpy(),
                            w2.float().cpu().numpy(), round_bf16=True)
    return got, ref


@pytest.mark.gpu
@pytest.mark.parametrize("T,H,I,E,k", [(1, 256, 128, 4, 2), (33, 512, 256, 8, 2), (300, 256, 384, 4, 2),
                                       (700, 512, 256, 4, 2)])
def test_moe_ffn_bf16_small(ctx, T, H, I, E, k):
    """ragged chunks, > 128 rows per expert (several work items), the shared
    expert over all tokens"""
    got, ref = run_bf16(ctx, T, H, I, E, k, seed=T)
    assert np.isfinite(got).all()
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_bf16_step3_dims_reduced_experts(ctx):
    """hidden 7168 / inter 5120 (Step-3 expert shape), 8 routed + shared, top-3."""
    got, ref = run_bf16(ctx, 40, 7168, 5120, 8, 3, seed=2)
    record("moe_bf16_step3_8exp", out=rel_err(got, ref))
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_bf16_expert_parallel_partials(ctx):
    T = 50
    got, ref = run_bf16(ctx, T, 512, 256, 8, 3, seed=4, ranges=[((0, 4), (0, 20)), ((4, 8), (20, T))])
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_bf16_row_scatter_matches_local(ctx):
    import torch

    T, H, I, E, k, rpd = 50, 512, 256, 8, 3, 20
    dev = torch.device("cuda:0")
    w13, w2, x, ids_np, w_np = make_case(T, H, I, E, k, 21)
    ids, wts = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
    w = {"n_experts": E, "w13": w13, "w2": w2}
    local = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    ctx.moe_ffn_bf16(w, x, ids, wts, local)
    bufs = [torch.full((rpd, H), float("nan"), dtype=torch.bfloat16, device=dev) for _ in range(3)]
    dst = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
    ctx.moe_ffn_bf16(w, x, ids, wts, local, scatter=(dst, rpd))
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(bufs)[:T], local)
    assert torch.isnan(torch.cat(bufs)[T:].float()).all()


@pytest.mark.gpu
@pytest.mark.parametrize("T,n_check", [(256, 32), (4096, 16)])
def test_config3_moe_bf16_48_experts(ctx, T, n_check):
    """Config 3 (48 routed + shared, top-3) with 16-bit experts at the bench
    shapes; oracle on a token subset, one expert's weights at a time."""
    import torch

    H, I, E, k = 7168, 5120, 48, 3
    dev = torch.device("cuda:0")
    w13, w2, x, ids_np, w_np = make_case(T, H, I, E, k, seed=T + 7)
    out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    ctx.moe_ffn_bf16({"n_experts": E, "w13": w13, "w2": w2}, x, torch.from_numpy(ids_np).to(dev),
                     torch.from_numpy(w_np).to(dev), out)
    torch.cuda.synchronize()
    xf = x.float().cpu().numpy()
    tokens = np.sort(np.random.default_rng(T).choice(T, size=n_check, replace=False))
    ref = orc.moe_layer_by_expert(
        ids_np, w_np, E,
        lambda e, rows: orc.expert_ffn_f32(xf[rows], w13[e].float().cpu().numpy(), w2[e].float().cpu().numpy(), True),
        tokens=tokens)
    err = rel_err(out.float().cpu().numpy()[tokens], ref)
    record(f"config3_moe_bf16_T{T}", out=err)
    assert err <= TOL, err
