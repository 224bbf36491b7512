"""MTP decode (mtp = 2, M=128 contraction) vs the CPU oracle.

Bar (as the single-token core): bf16 P / output against the oracle's
double-accumulated exact softmax on the same inputs, max|gpu-ref|/max|ref|
<= 1e-2 per token, LSE within 2e-3; rows that see no key give 0 / -inf.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import paged_layout, rel_err

H, D, PAGE = 64, 256, 64


def run_case(ctx, seq_lens, seed=0):
    import torch

    scale = D ** -0.5
    g = torch.Generator(device="cpu").manual_seed(seed)
    B = len(seq_lens)
    bt, num_pages = paged_layout(seq_lens, PAGE, seed=seed)
    q = torch.randn(B, 2, H, D, generator=g).to(torch.bfloat16)
    k = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16)
    v = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16)
    for b, L in enumerate(seq_lens):  # slots past seq_len hold NaN
        if L % PAGE and L > 0:
            pg = bt[b, L // PAGE]
            k[pg, L % PAGE:] = float("nan")
            v[pg, L % PAGE:] = float("nan")
    dev = torch.device("cuda:0")
    out = torch.empty(B, 2, H, D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, 2, H, dtype=torch.float32, device=dev)
    ctx.mfa_decode_attention_mtp(q.to(dev), k.to(dev), v.to(dev), torch.from_numpy(bt).to(dev),
                                 torch.tensor(seq_lens, dtype=torch.int32, device=dev), out, scale, lse=lse)
    torch.cuda.synchronize()
    ref, ref_lse = orc.mfa_decode_attention_mtp(q.float().numpy(), k.float().numpy(), v.float().numpy(), bt,
                                                np.array(seq_lens, np.int32), scale)
    return out.float().cpu().numpy(), lse.cpu().numpy(), ref, ref_lse


@pytest.mark.gpu
@pytest.mark.parametrize("seq_lens", [
    [2, 64, 65, 66],              # causal edge inside / across a page boundary
    [4096, 4096, 4096, 4096],     # config-2 context, split over many CTAs
    [1, 300, 0, 129],             # L = 1: token 0 sees no key; empty request
])
def test_mfa_decode_mtp_parity(ctx, seq_lens):
    got, lse, ref, ref_lse = run_case(ctx, seq_lens)
    assert np.isfinite(got).all()
    for j in range(2):
        assert rel_err(got[:, j], ref[:, j]) <= 1e-2, (j, rel_err(got[:, j], ref[:, j]))
    for b, L in enumerate(seq_lens):
        for j in range(2):
            if L - 1 + j <= 0:  # no visible key
                assert np.all(got[b, j] == 0) and np.all(np.isneginf(lse[b, j]))
            else:
                np.testing.assert_allclose(lse[b, j], ref_lse[b, j], rtol=2e-3, atol=2e-3)


@pytest.mark.gpu
def test_mfa_decode_mtp_long_context_split(ctx):
    got, lse, ref, ref_lse = run_case(ctx, [32768, 20000], seed=3)
    for j in range(2):
        assert rel_err(got[:, j], ref[:, j]) <= 1e-2
    np.testing.assert_allclose(lse, ref_lse, rtol=2e-3, atol=2e-3)


@pytest.mark.gpu
def test_mfa_decode_mtp1_is_the_single_token_core(ctx):
    import torch

    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(5)
    bt, num_pages = paged_layout([100, 64], PAGE, seed=5)
    q = torch.randn(2, 1, H, D, generator=g).to(torch.bfloat16).to(dev)
    k = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16).to(dev)
    v = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16).to(dev)
    btd, sl = torch.from_numpy(bt).to(dev), torch.tensor([100, 64], dtype=torch.int32, device=dev)
    o1 = torch.empty(2, 1, H, D, dtype=torch.bfloat16, device=dev)
    o2 = torch.empty(2, H, D, dtype=torch.bfloat16, device=dev)
    ctx.mfa_decode_attention_mtp(q, k, v, btd, sl, o1, 0.0625)
    ctx.mfa_decode_attention(q[:, 0].contiguous(), k, v, btd, sl, o2, 0.0625)
    torch.cuda.synchronize()
    assert torch.equal(o1[:, 0], o2)
