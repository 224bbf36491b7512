"""Bitwise determinism soak of the MoE FFN kernels at the AFD test dims:
the same call repeated N times must give identical bytes (a race inside a
kernel shows up as a rare mismatch).  python scripts/soak_determinism.py [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_19427_b200 import Context

N = int(sys.argv[1]) if len(sys.argv) > 1 else 300
ctx = Context(0)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(5)
H, I, E, k = 1024, 512, 8, 2
res = {}
for T, lo, hi, sh in [(24, 0, 8, (0, 24)), (24, 0, 4, (0, 12)), (24, 4, 8, (12, 24)), (256, 0, 8, (0, 256)),
                      (48, 0, 8, (0, 48))]:
    n = hi - lo
    x = (torch.randn(T, H, generator=g, device=dev)).to(torch.bfloat16)
    logits = torch.randn(T, E, generator=g, device=dev)
    top = logits.topk(k, dim=1)
    ids = top.indices.to(torch.int32).contiguous()
    wts = top.values.softmax(1).contiguous()
    wb = {"n_experts": E, "w13": (torch.randn(n + 1, 2 * I, H, generator=g, device=dev) / H ** 0.5).to(torch.bfloat16),
          "w2": (torch.randn(n + 1, H, I, generator=g, device=dev) / I ** 0.5).to(torch.bfloat16)}
    out0 = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    out = torch.empty_like(out0)
    ctx.moe_ffn_bf16(wb, x, ids, wts, out0, expert_lo=lo, expert_hi=hi, shared=sh)
    torch.cuda.synchronize()
    bad = 0
    for it in range(N):
        out.fill_(0)
        ctx.moe_ffn_bf16(wb, x, ids, wts, out, expert_lo=lo, expert_hi=hi, shared=sh)
        torch.cuda.synchronize()
        if not torch.equal(out, out0):
            bad += 1
            if bad <= 3:
                d = (out.float() - out0.float()).abs()
                rows = (d.amax(1) > 0).nonzero().flatten().tolist()
                print(f"  bf16 T={T} [{lo},{hi}) sh={sh} it {it}: max diff {d.max().item():.3e} rows {rows[:12]}")
    res[f"bf16 T={T} [{lo},{hi}) sh={sh}"] = bad
    # the MXFP8 path on the same routing
    xq = torch.empty(T, H, dtype=torch.uint8, device=dev)
    xs = torch.empty(T, H // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(x, xq, xs)
    mag = torch.randint(0x18, 0x40, (n + 1, 2 * I, H), generator=g, device=dev, dtype=torch.int32)
    wm = {"n_experts": E, "w13": mag.to(torch.uint8),
          "sf13": torch.full((n + 1, 2 * I, H // 32), 120, dtype=torch.uint8, device=dev),
          "w2": torch.randint(0x18, 0x40, (n + 1, H, I), generator=g, device=dev, dtype=torch.int32).to(torch.uint8),
          "sf2": torch.full((n + 1, H, I // 32), 120, dtype=torch.uint8, device=dev)}
    ctx.moe_ffn_mx(wm, xq, xs, ids, wts, out0, expert_lo=lo, expert_hi=hi, shared=sh)
    torch.cuda.synchronize()
    bad = 0
    for it in range(N):
        out.fill_(0)
        ctx.moe_ffn_mx(wm, xq, xs, ids, wts, out, expert_lo=lo, expert_hi=hi, shared=sh)
        torch.cuda.synchronize()
        if not torch.equal(out, out0):
            bad += 1
    res[f"mx   T={T} [{lo},{hi}) sh={sh}"] = bad
for k_, v in res.items():
    print(f"{k_}: {v} / {N} mismatching runs")
