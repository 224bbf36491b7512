"""Where the AFD attention stage's time goes, on one GPU: the e4m3-KV layer at
an AFD micro-batch with the bench's KV codes vs the AFD runtime's data
(normal(0,1) K/V -> e4m3 with amax/448 scales), then plus the router and
dispatch quantisation the ATTN op adds.  python scripts/afd_attn_breakdown.py [T]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

T = int(sys.argv[1]) if len(sys.argv) > 1 else 368
ctx = Context(0)
dev = torch.device("cuda:0")
s = bench.make_workload(torch, dev, T, 4096)
npages = s["kv"][0][0].shape[0]
sp = torch.cuda.current_stream().cuda_stream


def codes():
    sign = torch.randint(0, 2, (npages, 64, 256), dtype=torch.uint8, device=dev) * 0x80
    return torch.randint(0x08, 0x58, (npages, 64, 256), dtype=torch.uint8, device=dev) | sign


kv_codes = [(codes(), codes(), 0.05, 0.05) for _ in range(2)]
kv_afd = []
for k, v in s["kv"][:2]:
    ks, vs = float(k.abs().max()) / 448.0, float(v.abs().max()) / 448.0
    kv_afd.append(((k.float() / ks).to(torch.float8_e4m3fn).view(torch.uint8),
                   (v.float() / vs).to(torch.float8_e4m3fn).view(torch.uint8), ks, vs))
del s["kv"]
gate = (torch.randn(48, 7168, device=dev) / 7168 ** 0.5).to(torch.bfloat16)
ids = torch.empty(T, 3, dtype=torch.int32, device=dev)
wts = torch.empty(T, 3, device=dev)
xq = torch.empty(T, 7168, dtype=torch.uint8, device=dev)
xsf = torch.empty(T, 7168 // 32, dtype=torch.uint8, device=dev)


def timed(fn, steps=20):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3


def layer(kvs, extra):
    def f(i):
        k, v, ks, vs = kvs[i % 2]
        ctx.mfa_layer(s["w"], s["x"], k, v, s["block_table"], s["seq_lens"], s["h_res"], s["h_norm"], stream=sp,
                      kv_scales=(ks, vs))
        if extra:
            ctx.router_topk(s["h_norm"], gate, 3, ids, wts, stream=sp)
            ctx.quant_mx(s["h_norm"], xq, xsf, stream=sp)
    return f


def core(kvs):
    def f(i):
        k, v, ks, vs = kvs[i % 2]
        ctx.mfa_decode_attention_fp8(s["q"], k, v, s["block_table"], s["seq_lens"], s["attn_out"], 0.0625, ks, vs,
                                     stream=sp)
    return f


for r in range(2):
    print(f"T={T} round {r}: layer codes {timed(layer(kv_codes, False)):.1f} us, layer afd-kv {timed(layer(kv_afd, False)):.1f} us, "
          f"+router+quant {timed(layer(kv_afd, True)):.1f} us; core codes {timed(core(kv_codes)):.1f} us, "
          f"core afd-kv {timed(core(kv_afd)):.1f} us")
