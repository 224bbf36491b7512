"""Inspect the pieces of bench.run_afd_modeled_mx."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

dev = torch.device("cuda:0")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = Context(0)
s = bench.make_workload(torch, dev, 256, 4096, seed=11)
torch.cuda.synchronize()
k, v = s["kv"][0]


def one():
    ctx.mfa_layer(s["w"], s["x"], k, v, s["block_table"], s["seq_lens"], s["h_res"], s["h_norm"], stream=st.cuda_stream)


for n_warm in (2, 10):
    for _ in range(n_warm):
        one()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5):
        one()
    b.record(st)
    torch.cuda.synchronize()
    print("warm", n_warm, "layer B=256 us", a.elapsed_time(b) / 5 * 1e3)
for i in range(3):
    k, v = s["kv"][i]
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(5):
        one()
    b.record(st)
    torch.cuda.synchronize()
    print("kv", i, a.elapsed_time(b) / 5 * 1e3)
