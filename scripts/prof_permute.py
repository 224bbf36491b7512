"""Time K6 permute alone: python scripts/prof_permute.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_19427_b200 import Context

ctx = Context(0)
dev = torch.device("cuda:0")
for T in (256, 1024, 4096, 8192):
    ids = torch.stack([torch.randperm(48)[:3] for _ in range(T)]).to(torch.int32).to(dev)
    off = torch.empty(49, dtype=torch.int32, device=dev)
    perm = torch.empty(T * 3, dtype=torch.int32, device=dev)
    inv = torch.empty(T * 3, dtype=torch.int32, device=dev)
    for _ in range(3):
        ctx.moe_permute(ids, 48, off, perm, inv)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        ctx.moe_permute(ids, 48, off, perm, inv)
    b.record()
    torch.cuda.synchronize()
    print(f"permute T={T}: {a.elapsed_time(b) / 50 * 1e3:.1f} us")
