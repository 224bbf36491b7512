"""Dense Step-3 FFN layer (hidden 7168, inter 18432) in MXFP8:
python scripts/prof_dense.py T n_split"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_19427_b200 import Context

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ctx = Context(0)
r = bench.run_dense_bench(ctx, torch, torch.device("cuda:0"), T, ns, steps=10, warmup=3)
print(f"dense T={T} n_split={ns}: {r['ms_per_layer'] * 1e3:.1f} us  HBM {r['hbm']['frac']:.3f}  tensor {r['tensor']['frac']:.3f}")
