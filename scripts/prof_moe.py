"""Run the config-3 MoE FFN layer a few times (for ncu): python scripts/prof_moe.py [T] [fp8|mx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
fmt = sys.argv[2] if len(sys.argv) > 2 else "fp8"
ctx = Context(0)
r = bench.run_moe_bench(ctx, torch, torch.device("cuda:0"), T, steps=3, warmup=2, fmt=fmt)
print(r["format"], r["T"], r["ms_per_layer"], r["hbm"]["frac"], r["tensor"]["frac"])
