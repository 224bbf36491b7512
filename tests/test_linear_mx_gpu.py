"""MXFP8 projection (afdk_linear_mx) vs a PyTorch fp32 reference of the same op.

Reference: the dequantised operands (e4m3 code x 2^(UE8M0 - 127) per 32
elements along K) multiplied in fp32.  The tensor core multiplies the same
exact products and accumulates in fp32, so only the summation order differs:
stated bar max|gpu - ref| / max|ref| <= 1e-4 (fp32 output), 8e-3 (bf16 output).
Operands come from afdk_quant_mx on random bf16 data, so the codes and
scales are what the layer would feed the GEMM."""
import pytest

from tests.helpers import rel_err


def dequant_mx(q, sf):
    import torch

    vals = q.view(torch.float8_e4m3fn).float()
    scale = torch.exp2(sf.float() - 127.0)
    return (vals.view(q.shape[0], -1, 32) * scale.view(q.shape[0], -1, 1)).view(q.shape)


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [
    (64, 2560, 7168),   # [q_down|k|v] at config 2
    (64, 16384, 2048),  # q_up
    (64, 7168, 16384),  # o_proj
    (5, 1000, 512),     # ragged rows and features
    (200, 384, 1024),   # single-buffered accumulator (N = 208)
    (256, 7168, 2048),  # the N = 256 limit
    (1, 48, 7168),      # router-like: one token, n < 128
    (320, 7168, 16384), # o_proj at an AFD micro-batch: two N=160 MMAs per k-block
    (384, 2560, 7168),  # the 384-token limit
    (300, 1000, 512),   # ragged above 256 (N rounded to 320)
])
def test_linear_mx_vs_torch(ctx, m, n, k):
    import torch

    g = torch.Generator().manual_seed(m * 13 + n)
    dev = torch.device("cuda")
    x = torch.randn(m, k, generator=g).to(torch.bfloat16).to(dev)
    w = (torch.randn(n, k, generator=g) * (0.02 + torch.rand(n, 1, generator=g))).to(torch.bfloat16).to(dev)
    xq = torch.empty(m, k, dtype=torch.uint8, device=dev)
    xsf = torch.empty(m, k // 32, dtype=torch.uint8, device=dev)
    wq = torch.empty(n, k, dtype=torch.uint8, device=dev)
    wsf = torch.empty(n, k // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(x, xq, xsf)
    ctx.quant_mx(w, wq, wsf)
    ref = (dequant_mx(xq, xsf) @ dequant_mx(wq, wsf).T).cpu().numpy()
    out32 = torch.empty(m, n, dtype=torch.float32, device=dev)
    ctx.linear_mx(xq, xsf, wq, wsf, out32)
    out16 = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    ctx.linear_mx(xq, xsf, wq, wsf, out16)
    torch.cuda.synchronize()
    e32 = rel_err(out32.cpu().numpy(), ref)
    e16 = rel_err(out16.float().cpu().numpy(), ref)
    try:
        from tests.helpers import record
        record(f"linear_mx_{m}x{n}x{k}", out_fp32=e32, out_bf16=e16)
    except Exception:  # noqa: BLE001
        pass
    assert e32 <= 1e-4, e32
    assert e16 <= 8e-3, e16


@pytest.mark.gpu
def test_linear_mx_rejects_bad_shapes(ctx):
    import torch

    from paper_2507_19427_b200.afdk import AfdkError

    dev = torch.device("cuda")
    xq = torch.zeros(400, 256, dtype=torch.uint8, device=dev)
    xsf = torch.full((400, 8), 127, dtype=torch.uint8, device=dev)
    wq = torch.zeros(128, 256, dtype=torch.uint8, device=dev)
    wsf = torch.full((128, 8), 127, dtype=torch.uint8, device=dev)
    out = torch.empty(400, 128, device=dev)
    with pytest.raises(AfdkError):
        ctx.linear_mx(xq, xsf, wq, wsf, out)  # m > 384
    with pytest.raises(AfdkError):  # k % 512 != 0: the 8-byte scale rows cannot be TMA-loaded
        ctx.linear_mx(xq[:64], xsf[:64], wq, wsf, out[:64])
