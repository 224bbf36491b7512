"""One AFD attention op at a micro-batch (e4m3-KV layer + router + MX dispatch
quantisation), for an ncu launch list: python scripts/prof_afd_attn.py [T] [o_mx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

T = int(sys.argv[1]) if len(sys.argv) > 1 else 384
o_mx = len(sys.argv) > 2 and sys.argv[2] == "1"
ctx = Context(0)
dev = torch.device("cuda:0")
s = bench.make_workload(torch, dev, T, 4096)
k, v = s["kv"][0]
ks, vs = float(k.abs().max()) / 448.0, float(v.abs().max()) / 448.0
k8 = (k.float() / ks).to(torch.float8_e4m3fn).view(torch.uint8)
v8 = (v.float() / vs).to(torch.float8_e4m3fn).view(torch.uint8)
del s["kv"]
w = dict(s["w"])
if o_mx:
    w["o_mx"] = torch.empty(w["o"].shape, dtype=torch.uint8, device=dev)
    w["o_sf"] = torch.empty(w["o"].shape[0], w["o"].shape[1] // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(w["o"], w["o_mx"], w["o_sf"])
gate = (torch.randn(48, 7168, device=dev) / 7168 ** 0.5).to(torch.bfloat16)
ids = torch.empty(T, 3, dtype=torch.int32, device=dev)
wts = torch.empty(T, 3, device=dev)
xq = torch.empty(T, 7168, dtype=torch.uint8, device=dev)
xsf = torch.empty(T, 7168 // 32, dtype=torch.uint8, device=dev)
for _ in range(4):  # warm-up, then the profiled op (the last 13 launches)
    ctx.mfa_layer(w, s["x"], k8, v8, s["block_table"], s["seq_lens"], s["h_res"], s["h_norm"], kv_scales=(ks, vs))
    ctx.router_topk(s["h_norm"], gate, 3, ids, wts)
    ctx.quant_mx(s["h_norm"], xq, xsf)
torch.cuda.synchronize()
print("ok")
