"""FP8-KV MFA decode (e4m3 K/V pages + per-tensor scales) vs the CPU oracle.

Oracle semantics (oracle.mfa_decode_attention_fp8): exact softmax attention on
the dequantised K/V and on Q quantised per (request, head) exactly like the
kernel does.  The kernel additionally rounds P to e4m3 for the P.V MMA
(3 mantissa bits on the probabilities), so the stated bar is
max|gpu-ref| / max|ref| <= 3e-2 on O and |lse - ref| <= 2e-2.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import paged_layout, rel_err

TOL = 3e-2
H, D, PAGE = 64, 256, 64


def to_e4m3(torch, x, scale):
    return (x / scale).to(torch.float8_e4m3fn).view(torch.uint8)


def run_case(ctx, seq_lens, seed=0, poison=True):
    import torch

    scale = D ** -0.5
    g = torch.Generator(device="cpu").manual_seed(seed)
    B = len(seq_lens)
    bt, num_pages = paged_layout(seq_lens, PAGE, seed=seed)
    q = torch.randn(B, H, D, generator=g).to(torch.bfloat16)
    k = torch.randn(num_pages, PAGE, D, generator=g) * 1.5
    v = torch.randn(num_pages, PAGE, D, generator=g)
    k_scale = float(k.abs().max()) / 448.0
    v_scale = float(v.abs().max()) / 448.0
    kq, vq = to_e4m3(torch, k, k_scale), to_e4m3(torch, v, v_scale)
    if poison:  # slots past seq_len hold e4m3 NaN (0x7f): never mixed in
        for b, L in enumerate(seq_lens):
            if L % PAGE and L > 0:
                pg = bt[b, L // PAGE]
                kq[pg, L % PAGE:] = 0x7F
                vq[pg, L % PAGE:] = 0x7F
    dev = torch.device("cuda:0")
    out = torch.empty(B, H, D, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, H, dtype=torch.float32, device=dev)
    ctx.mfa_decode_attention_fp8(q.to(dev), kq.to(dev), vq.to(dev), torch.from_numpy(bt).to(dev),
                                 torch.tensor(seq_lens, dtype=torch.int32, device=dev), out, scale,
                                 k_scale, v_scale, lse=lse)
    torch.cuda.synchronize()
    ref, ref_lse = orc.mfa_decode_attention_fp8(q.float().numpy(), kq.numpy(), vq.numpy(), k_scale, v_scale,
                                                bt, np.array(seq_lens, np.int32), scale)
    return out.float().cpu().numpy(), lse.cpu().numpy(), ref, ref_lse


@pytest.mark.gpu
@pytest.mark.parametrize("seq_lens", [
    [64],
    [1, 63, 64, 65],
    [4096, 4096, 4096, 4096],
    [300, 1, 2000, 0, 129],
])
def test_mfa_decode_fp8_parity(ctx, seq_lens):
    got, lse, ref, ref_lse = run_case(ctx, seq_lens)
    assert np.isfinite(got).all()
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)
    for b, L in enumerate(seq_lens):
        if L == 0:
            assert np.all(got[b] == 0)
            assert np.all(np.isneginf(lse[b]))
        else:
            np.testing.assert_allclose(lse[b], ref_lse[b], rtol=0, atol=2e-2)


@pytest.mark.gpu
def test_mfa_decode_fp8_long_context_split(ctx):
    got, lse, ref, ref_lse = run_case(ctx, [32768, 20000], seed=3, poison=False)
    from tests.helpers import record
    record("mfa_fp8_long_context_split", out=rel_err(got, ref), lse=float(np.abs(lse - ref_lse).max()))
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)
    np.testing.assert_allclose(lse, ref_lse, rtol=0, atol=2e-2)


@pytest.mark.gpu
def test_mfa_decode_fp8_many_short_requests(ctx):
    rng = np.random.default_rng(7)
    seq_lens = rng.integers(1, 200, size=300).tolist()
    got, lse, ref, ref_lse = run_case(ctx, seq_lens, seed=7)
    assert rel_err(got, ref) <= TOL, rel_err(got, ref)


@pytest.mark.gpu
def test_mfa_decode_fp8_rejects_bad_scale(ctx):
    import torch

    from paper_2507_19427_b200.afdk import AfdkError

    dev = torch.device("cuda:0")
    q = torch.zeros(1, H, D, dtype=torch.bfloat16, device=dev)
    kv = torch.zeros(1, PAGE, D, dtype=torch.uint8, device=dev)
    bt = torch.zeros(1, 1, dtype=torch.int32, device=dev)
    sl = torch.ones(1, dtype=torch.int32, device=dev)
    out = torch.empty(1, H, D, dtype=torch.bfloat16, device=dev)
    with pytest.raises(AfdkError):
        ctx.mfa_decode_attention_fp8(q, kv, kv, bt, sl, out, 0.0625, 0.0, 1.0)
