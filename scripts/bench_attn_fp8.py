"""MFA decode core, bf16 vs e4m3 KV cache: python scripts/bench_attn_fp8.py [B ctx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ctx = Context(0)
dev = torch.device("cuda:0")
w = bench.make_workload_attn(torch, dev, B, L)
N_ROT = 4
npages = w["kv"][0][0].shape[0]
kv8 = [(torch.randint(0, 0x7e, (npages, 64, 256), dtype=torch.uint8, device=dev),
        torch.randint(0, 0x7e, (npages, 64, 256), dtype=torch.uint8, device=dev)) for _ in range(N_ROT)]
s = torch.cuda.current_stream()


def run(fp8, steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(3):
        step(fp8, i)
    torch.cuda.synchronize()
    a.record(s)
    for i in range(steps):
        step(fp8, i)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def step(fp8, i):
    if fp8:
        k, v = kv8[i % N_ROT]
        ctx.mfa_decode_attention_fp8(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], 0.0625, 0.01, 0.01,
                                     stream=s.cuda_stream)
    else:
        k, v = w["kv"][i % 2]
        ctx.mfa_decode_attention(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], 0.0625, stream=s.cuda_stream)


peak = bench.peaks()[0]
for fp8 in (False, True):
    ms = run(fp8, 20)
    kv = B * L * 2 * 256 * (1 if fp8 else 2)
    gbs = (kv + 2 * B * 64 * 256 * 2) / (ms * 1e-3) / 1e9
    print(f"{'e4m3' if fp8 else 'bf16'} KV  B={B} ctx={L}: {ms * 1e3:.1f} us  {gbs:.0f} GB/s  {gbs / peak:.3f} of HBM peak")
