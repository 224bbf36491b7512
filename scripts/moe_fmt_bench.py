"""Time the config-3 MoE layer in given formats/T through bench.run_moe_bench
(same workload as bench.py's moe_ffn lines); prints one JSON per point."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_19427_b200 import Context  # noqa: E402


ctx = Context(0)
pts = [(f, int(T)) for f, T in (a.split(":") for a in sys.argv[1:])] or [("bf16", 256), ("bf16", 4096)]
for f, T in pts:
    r = bench.run_moe_bench(ctx, torch, torch.device("cuda:0"), T, 10, 3, fmt=f)
    print(json.dumps(r), flush=True)
