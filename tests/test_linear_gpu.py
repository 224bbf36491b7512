"""K1/K4 weight-streaming GEMM vs a plain PyTorch fp32 reference of the same op.

Tolerance (stated): fp32 output rel (max-abs normalised) <= 1e-3 (fp32
accumulation order only); bf16 output <= 8e-3 (one bf16 rounding)."""
import pytest

from tests.helpers import rel_err


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [
    (64, 2560, 7168),   # [q_down|k|v] at config 2
    (64, 16384, 2048),  # q_up
    (64, 7168, 16384),  # o_proj
    (1, 48, 7168),      # router gate, one token, n < 128 (TMA zero-filled rows)
    (5, 1000, 512),     # ragged everything
    (200, 384, 1024),   # n_mma 208
    (256, 256, 64),     # single k-block, max tokens
    (256, 7168, 16384), # o_proj at the AFD micro-batch: 256-row tiles, single-buffered accumulators
    (128, 16384, 2048), # q_up at 128 rows: 256-row tiles, double-buffered (N = 128)
    (100, 2560, 7168),  # qkv, ragged N (112) on 256-row tiles
    (96, 2176, 512),    # n_out not a multiple of 256: the last tile's second panel is TMA zero-filled
    (384, 7168, 16384), # o_proj at a 384-request AFD micro-batch: two N=192 MMAs per weight k-block
    (512, 16384, 2048), # q_up at the 512-row limit (two N=256 MMAs, single-buffered accumulator)
    (272, 2560, 7168),  # just above 256: n_mma rounded to 288, second box half zero-filled
    (300, 1000, 512),   # ragged everything above 256
])
def test_linear_vs_torch(ctx, m, n, k):
    import torch

    g = torch.Generator().manual_seed(m * 7 + n)
    x = torch.randn(m, k, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(n, k, generator=g) / k ** 0.5).to(torch.bfloat16).cuda()
    ref = (x.float() @ w.float().T).cpu().numpy()
    out32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    ctx.linear(x, w, out32)
    out16 = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    ctx.linear(x, w, out16)
    torch.cuda.synchronize()
    assert rel_err(out32.cpu().numpy(), ref) <= 1e-3
    assert rel_err(out16.float().cpu().numpy(), ref) <= 8e-3


@pytest.mark.gpu
def test_linear_deterministic(ctx):
    import torch

    x = torch.randn(64, 7168).to(torch.bfloat16).cuda()
    w = torch.randn(2560, 7168).to(torch.bfloat16).cuda()
    a = torch.empty(64, 2560, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    ctx.linear(x, w, a)
    ctx.linear(x, w, b)
    assert torch.equal(a, b)  # fixed-order partial reduction, no atomics
