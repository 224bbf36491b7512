"""One process driving two B200s through two contexts: kernel attributes
(dynamic shared-memory limits) must be set per device.  Skipped on one GPU."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import paged_layout, rel_err


@pytest.mark.gpu
def test_two_devices_one_process():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2507_19427_b200 import Context

    H, D, P = 64, 256, 64
    seq_lens = [200, 64]
    bt, npg = paged_layout(seq_lens, P, seed=2)
    g = torch.Generator().manual_seed(2)
    q = torch.randn(2, H, D, generator=g).to(torch.bfloat16)
    k = torch.randn(npg, P, D, generator=g).to(torch.bfloat16)
    v = torch.randn(npg, P, D, generator=g).to(torch.bfloat16)
    ref, _ = orc.mfa_decode_attention(q.float().numpy(), k.float().numpy(), v.float().numpy(), bt,
                                      np.array(seq_lens, np.int32), D ** -0.5)
    for dev_id in (0, 1, 0):
        with torch.cuda.device(dev_id):
            ctx = Context(dev_id)
            dev = torch.device(f"cuda:{dev_id}")
            out = torch.empty(2, H, D, dtype=torch.bfloat16, device=dev)
            ctx.mfa_decode_attention(q.to(dev), k.to(dev), v.to(dev), torch.from_numpy(bt).to(dev),
                                     torch.tensor(seq_lens, dtype=torch.int32, device=dev), out, D ** -0.5)
            torch.cuda.synchronize(dev)
            assert rel_err(out.float().cpu().numpy(), ref) <= 1e-2
            ctx.close()


@pytest.mark.gpu
def test_entry_points_restore_callers_device():
    """Every C-ABI call runs on its context's device and hands the caller's
    current device back (afdk_internal.h DeviceGuard)."""
    import torch

    from paper_2507_19427_b200 import Context

    n = torch.cuda.device_count()
    ctx_dev = n - 1
    H, D, P = 64, 256, 64
    bt, npg = paged_layout([100], P, seed=1)
    dev = torch.device(f"cuda:{ctx_dev}")
    ctx = Context(ctx_dev)
    q = torch.randn(1, H, D, device=dev).to(torch.bfloat16)
    k = torch.randn(npg, P, D, device=dev).to(torch.bfloat16)
    out = torch.empty(1, H, D, dtype=torch.bfloat16, device=dev)
    torch.cuda.set_device(0)
    ctx.mfa_decode_attention(q, k, k, torch.from_numpy(bt).to(dev), torch.tensor([100], dtype=torch.int32, device=dev),
                             out, D ** -0.5)
    assert torch.cuda.current_device() == 0
    torch.cuda.synchronize(dev)
    ctx.close()


@pytest.mark.gpu
def test_batch_over_limit_is_invalid(ctx):
    """Shape limits come back as AFDK_ERR_INVALID (a SpecError), not a CUDA error."""
    import torch

    from paper_2507_19427_b200.afdk import AfdkError

    B, H, D, P = 2049, 64, 256, 64
    dev = torch.device("cuda:0")
    q = torch.zeros(B, H, D, dtype=torch.bfloat16, device=dev)
    k = torch.zeros(1, P, D, dtype=torch.bfloat16, device=dev)
    out = torch.empty_like(q)
    with pytest.raises(AfdkError) as ei:
        ctx.mfa_decode_attention(q, k, k, torch.zeros(B, 1, dtype=torch.int32, device=dev),
                                 torch.ones(B, dtype=torch.int32, device=dev), out, D ** -0.5)
    assert ei.value.status == 1, ei.value  # AFDK_ERR_INVALID
