"""Time K5 router (+ fp8 quant) and the MXFP8 quant: python scripts/prof_router.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_19427_b200 import Context

ctx = Context(0)
dev = torch.device("cuda:0")
H, E, k = 7168, 48, 3
gate = (torch.randn(E, H, device=dev) / H ** 0.5).to(torch.bfloat16)
for T in (64, 256, 1024):
    h = torch.randn(T, H, device=dev).to(torch.bfloat16)
    ids = torch.empty(T, k, dtype=torch.int32, device=dev)
    wts = torch.empty(T, k, device=dev)
    xq = torch.empty(T, H, dtype=torch.uint8, device=dev)
    xs = torch.empty(T, H // 128, device=dev)
    xsf = torch.empty(T, H // 32, dtype=torch.uint8, device=dev)

    def t(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    r1 = t(lambda: ctx.router_topk(h, gate, k, ids, wts))
    r2 = t(lambda: ctx.router_topk(h, gate, k, ids, wts, xq=xq, xs=xs))
    r3 = t(lambda: ctx.quant_mx(h, xq, xsf))
    print(f"T={T}: router {r1:.1f} us, router+fp8 quant {r2:.1f} us, quant_mx {r3:.1f} us")
