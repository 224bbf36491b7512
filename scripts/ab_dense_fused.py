"""A/B of the dense decode FFN: fused single-CTA kernel vs CTA-pair GEMMs (run with AFDK_DENSE_FUSED=0/1)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_19427_b200 import Context  # noqa: E402

ctx = Context(0)
for T in (64, 128, 256):
    for ns in (1, 2, 4):
        r = bench.run_dense_bench(ctx, torch, torch.device("cuda:0"), T, ns, 20, 3)
        print(json.dumps({"fused": os.environ.get("AFDK_DENSE_FUSED", "auto"), "T": T, "n_split": ns,
                          "ms": round(r["ms_per_layer"], 4), "hbm": round(r["hbm"]["frac"], 3)}), flush=True)
