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

# MTP (mtp = 2): two query tokens per request over the same bf16 KV
q2 = torch.randn(B, 2, 64, 256, device=dev).to(torch.bfloat16)
o2 = torch.empty(B, 2, 64, 256, device=dev, dtype=torch.bfloat16)


def step_mtp(i):
    k, v = w["kv"][i % 2]
    ctx.mfa_decode_attention_mtp(q2, k, v, w["block_table"], w["seq_lens"], o2, 0.0625, stream=s.cuda_stream)


for i in range(3):
    step_mtp(i)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for i in range(20):
    step_mtp(i)
b.record(s)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
kv = B * L * 2 * 256 * 2
print(f"mtp=2 bf16 KV B={B} ctx={L}: {ms * 1e3:.1f} us  {(kv + 4 * B * 128 * 256) / (ms * 1e-3) / 1e9:.0f} GB/s  "
      f"{2 * B / (ms * 1e-3):.0f} query tokens/s")
