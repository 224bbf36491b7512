"""A/B of the dense decode FFN layout: n_split x kernel (AFDK_MX_PAIR) at T=256/4096."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_19427_b200 import Context  # noqa: E402

ctx = Context(0)
for T in (256, 4096):
    for ns in (4, 6, 9, 12):
        r = bench.run_dense_bench(ctx, torch, torch.device("cuda:0"), T, ns, 20, 3)
        print(json.dumps({"pair": os.environ.get("AFDK_MX_PAIR", "auto"), "T": T, "n_split": ns,
                          "ms": round(r["ms_per_layer"], 4), "hbm": round(r["hbm"]["frac"], 3),
                          "tensor": round(r["tensor"]["frac"], 3)}), flush=True)
