"""K2/K3 parity: B200 MFA decode attention vs the CPU oracle.

Tolerance (stated): bf16 inputs, bf16 P operand and bf16 output against the
oracle's double-accumulated softmax on the same bf16-representable inputs:
max|gpu-ref| / max|ref| <= 1e-2.
"""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import paged_layout, rel_err

TOL = 1e-2
H, D, PAGE = 64, 256, 64


def run_case(ctx, seq_lens, seed=0, poison=True, scale=None):
    import torch

    scale = D ** -0.5 if scale is None else scale
    g = torch.Generator(device="cpu").manual_seed(seed)
    B = len(seq_lens)
    bt, num_pages = paged_layout(seq_lens, PAGE, seed=seed)
    q = torch.randn(B, H, D, generator=g).to(torch.bfloat16)
    k = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16)
    v = torch.randn(num_pages, PAGE, D, generator=g).to(torch.bfloat16)
    if poison:  # slots past seq_len hold NaN: the kernel must never mix them in
        for b, L in enumerate(seq_lens):
            if L % PAGE and L > 0:
                pg = bt[b, L // PAGE]
                k[pg, L % PAGE:] = float("nan")
                v[pg, L % PAGE:] = float("nan")
    dev = torch.device("cuda:0")
    qd, kd, vd = q.to(dev), k.to(dev), v.to(dev)
    btd = torch.from_numpy(bt).to(dev)
    sld = torch.tensor(seq_lens, dtype=torch.int32, device=dev)
    out = torch.empty(B, H, D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, H, dtype=torch.float32, device=dev)
    ctx.mfa_decode_attention(qd, kd, vd, btd, sld, out, scale, lse=lse)
    torch.cuda.synchronize()
    ref, ref_lse = orc.mfa_decode_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                            bt, np.array(seq_lens, np.int32), scale)
    return out.float().cpu().numpy(), lse.cpu().numpy(), ref, ref_lse


@pytest.mark.gpu
@pytest.mark.parametrize("seq_lens", [
    [64],                      # one full page, one CTA range
    [1, 63, 64, 65],           # ragged tails inside a page
    [4096, 4096, 4096, 4096],  # config-2 context, split over many CTAs
    [300, 1, 2000, 0, 129],    # includes an empty request
])
def test_mfa_decode_parity(ctx, seq_lens):
    got, lse, ref, ref_lse = run_case(ctx, seq_lens)
    assert np.isfinite(got).all()
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)
    for b, L in enumerate(seq_lens):
        if L == 0:
            assert np.all(got[b] == 0)
            assert np.all(np.isneginf(lse[b]))
        else:
            np.testing.assert_allclose(lse[b], ref_lse[b], rtol=2e-3, atol=2e-3)


@pytest.mark.gpu
def test_mfa_decode_long_context_split(ctx):
    """Config 4 shape class (32K context) at reduced batch: split-KV combine."""
    got, lse, ref, ref_lse = run_case(ctx, [32768, 20000], seed=3, poison=False)
    assert rel_err(got, ref) <= TOL
    np.testing.assert_allclose(lse, ref_lse, rtol=2e-3, atol=2e-3)


@pytest.mark.gpu
def test_mfa_decode_many_short_requests(ctx):
    """More requests than SMs: CTA ranges span several whole requests."""
    rng = np.random.default_rng(7)
    seq_lens = rng.integers(1, 200, size=300).tolist()
    got, lse, ref, ref_lse = run_case(ctx, seq_lens, seed=7)
    assert rel_err(got, ref) <= TOL


@pytest.mark.gpu
def test_mfa_decode_peaked_scores_rescale(ctx):
    """Large scale -> the running max grows across pages (lazy O rescale path)."""
    got, lse, ref, ref_lse = run_case(ctx, [1000, 3000], seed=5, scale=0.5)
    assert rel_err(got, ref) <= TOL
