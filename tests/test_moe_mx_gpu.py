"""MXFP8 MoE FFN path (hardware block-scaled tcgen05 MMA) vs the CPU oracle.

Stated bars:
  * MXFP8 quantisation (e4m3 codes and UE8M0 scales): bit-exact vs
    orc_quant_mx on the same bf16 input
  * MoE / dense FFN output vs orc_moe_layer_mx / orc_expert_ffn_mx on the same
    MXFP8 inputs/weights: max|gpu-ref|/max|ref| <= 1e-2 (bf16 output: one ulp at
    the largest element is 3.9e-3 of this norm; a fast-exp SiLU can flip an
    e4m3 rounding of the re-quantised intermediate; measured <= 4.8e-3)
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import rel_err
from tests.test_moe_gpu import rand_e4m3


def make_mx_experts(torch, n_local, H, I, gen, dev):
    w13 = rand_e4m3(torch, (n_local + 1, 2 * I, H), gen, dev)
    w2 = rand_e4m3(torch, (n_local + 1, H, I), gen, dev)
    # scales ~ 1/sqrt(K) so activations stay O(1) through both GEMMs
    b13 = 127 - int(round(np.log2(H) / 2)) - 1
    b2 = 127 - int(round(np.log2(I) / 2)) - 1
    sf13 = torch.randint(b13 - 1, b13 + 2, (n_local + 1, 2 * I, H // 32), generator=gen, dtype=torch.int32)
    sf2 = torch.randint(b2 - 1, b2 + 2, (n_local + 1, H, I // 32), generator=gen, dtype=torch.int32)
    return {"w13": w13, "sf13": sf13.to(torch.uint8).to(dev), "w2": w2, "sf2": sf2.to(torch.uint8).to(dev)}


@pytest.mark.gpu
@pytest.mark.parametrize("T,H", [(1, 7168), (37, 7168), (256, 1024)])
def test_quant_mx_bit_exact(ctx, T, H):
    import torch

    g = torch.Generator().manual_seed(T + H)
    x = torch.randn(T, H, generator=g) * torch.exp2(torch.randint(-20, 20, (T, 1), generator=g).float())
    x[0, :32] = 0.0                   # all-zero block -> sf 0
    x[0, 32:64] = 448.0               # exactly representable at e = 0
    x[0, 64] = 1e30                   # huge block
    x[0, 96:128] = 1e-38              # subnormal-range block
    xb = x.to(torch.bfloat16)
    dev = torch.device("cuda:0")
    q = torch.empty(T, H, dtype=torch.uint8, device=dev)
    sf = torch.empty(T, H // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(xb.to(dev), q, sf)
    torch.cuda.synchronize()
    rq, rs = orc.quant_mx(xb.float().numpy())
    np.testing.assert_array_equal(sf.cpu().numpy(), rs)
    np.testing.assert_array_equal(q.cpu().numpy(), rq)


def run_moe_mx(ctx, T, H, I, E, k, seed, ranges=None):
    import torch

    g = torch.Generator().manual_seed(seed)
    dev = torch.device("cuda:0")
    ex = make_mx_experts(torch, E, H, I, g, dev)
    x = torch.randn(T, H, generator=g)
    xq_np, xsf_np = orc.quant_mx(x.numpy())
    logits = torch.randn(T, E, generator=g).numpy()
    ids_np, w_np = orc.router_topk(logits, k)
    xq, xsf = torch.from_numpy(xq_np).to(dev), torch.from_numpy(xsf_np).to(dev)
    ids, wts = torch.from_numpy(ids_np).to(dev), torch.from_numpy(w_np).to(dev)
    if ranges is None:
        out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        ctx.moe_ffn_mx(dict(n_experts=E, **ex), xq, xsf, ids, wts, out)
        torch.cuda.synchronize()
        got = out.float().cpu().numpy()
    else:
        got = np.zeros((T, H), np.float32)
        for (lo, hi), (slo, shi) in ranges:
            sub = {n: torch.cat([ex[n][lo:hi], ex[n][E:]]) for n in ("w13", "sf13", "w2", "sf2")}
            out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
            ctx.moe_ffn_mx(dict(n_experts=E, **sub), xq, xsf, ids, wts, out, expert_lo=lo, expert_hi=hi,
                           shared=(slo, shi))
            torch.cuda.synchronize()
            got += out.float().cpu().numpy()
    ref = orc.moe_layer_mx(xq_np, xsf_np, ids_np, w_np, *(ex[n].cpu().numpy() for n in ("w13", "sf13", "w2", "sf2")))
    return got, ref


# "0": single-CTA kernels (128-row items), "1": CTA-pair kernels (items of up to 384 rows)
KERNELS = ["0", "1"]


@pytest.fixture(params=KERNELS, ids=["cta", "pair"])
def mx_kernel(request, monkeypatch):
    monkeypatch.setenv("AFDK_MX_PAIR", request.param)
    return request.param


@pytest.mark.gpu
def test_moe_ffn_mx_small(ctx, mx_kernel):
    got, ref = run_moe_mx(ctx, 33, 512, 512, 8, 2, 1)
    assert np.isfinite(got).all()
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_mx_many_rows_per_expert(ctx, mx_kernel):
    """> 256 rows for one expert (several work chunks) and a ragged last chunk."""
    got, ref = run_moe_mx(ctx, 300, 512, 1024, 4, 2, 3)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_mx_two_accumulator_chunks(ctx, mx_kernel):
    """~350 rows per routed expert and 700 shared rows: pair items of 257-384
    rows use the second TMEM accumulator; 700 = 384 + 316 splits the shared expert."""
    got, ref = run_moe_mx(ctx, 700, 512, 1024, 4, 2, 6)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_mx_step3_dims_reduced_experts(ctx, mx_kernel):
    """hidden 7168 / inter 5120 (Step-3 expert shape), 8 routed + shared, top-3."""
    got, ref = run_moe_mx(ctx, 40, 7168, 5120, 8, 3, 2)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_mx_step3_dims_large_batch(ctx, mx_kernel):
    """Step-3 expert shape at ~200 rows per expert (the tensor-bound regime)."""
    got, ref = run_moe_mx(ctx, 400, 7168, 5120, 4, 2, 5)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_moe_ffn_mx_expert_parallel_partials(ctx, mx_kernel):
    T = 50
    got, ref = run_moe_mx(ctx, T, 512, 512, 8, 3, 4, ranges=[((0, 4), (0, 20)), ((4, 8), (20, T))])
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


def run_dense(ctx, T, H, I, n_split, seed):
    import torch

    from paper_2507_19427_b200.afdk import Context

    g = torch.Generator().manual_seed(seed)
    dev = torch.device("cuda:0")
    full = make_mx_experts(torch, 0, H, I, g, torch.device("cpu"))  # one [2I, H] / [H, I] FFN
    w13, sf13, w2, sf2 = (full[n][0] for n in ("w13", "sf13", "w2", "sf2"))
    split = Context.dense_split_layout(w13, sf13, w2, sf2, n_split)
    wd = {k: v.to(dev) for k, v in split.items()}
    x = torch.randn(T, H, generator=g)
    xq, xsf = orc.quant_mx(x.numpy())
    out = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    ctx.dense_ffn_mx(wd, torch.from_numpy(xq).to(dev), torch.from_numpy(xsf).to(dev), out)
    torch.cuda.synchronize()
    ref = orc.expert_ffn_mx(xq, xsf, w13.numpy(), sf13.numpy(), w2.numpy(), sf2.numpy())
    return out.float().cpu().numpy(), ref


@pytest.mark.gpu
@pytest.mark.parametrize("T", [1, 37, 300])
def test_dense_ffn_mx(ctx, mx_kernel, T):
    """Dense FFN as 4 intermediate slices == the unsplit FFN (fp32 slice sums)."""
    got, ref = run_dense(ctx, T, 512, 2048, 4, 10 + T)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)


@pytest.mark.gpu
def test_dense_ffn_mx_step3_dims(ctx):
    """Step-3 dense layer: hidden 7168, inter 18432 as 4 slices of 4608."""
    got, ref = run_dense(ctx, 16, 7168, 18432, 4, 3)
    assert rel_err(got, ref) <= 1e-2, rel_err(got, ref)
