"""Time / profile one FFN GPU's MoE shard (config 3 sharded over N GPUs): python scripts/prof_moe_shard.py T N fmt"""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_19427_b200 import Context  # noqa: E402

T, N, fmt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ctx = Context(0)
r = bench.run_moe_bench(ctx, torch, torch.device("cuda:0"), T, 10, 3, fmt=fmt, shard=(0, N, None))
print(json.dumps({"T": T, "shard_of": N, "fmt": fmt, "ms": r["ms_per_layer"], "hbm": r["hbm"]["frac"]}))
