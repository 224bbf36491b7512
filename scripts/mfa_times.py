"""Per-CTA timeline of one MFA decode core launch (diagnostic build with
-DAFDK_MFA_TIMES=1): python scripts/mfa_times.py [B ctx]; AFDK_LIB=libafdk_times.so"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2507_19427_b200 import Context

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
ctx = Context(0)
lib = ctypes.CDLL(os.environ["AFDK_LIB"])
dev = torch.device("cuda:0")
w = bench.make_workload_attn(torch, dev, B, L)
s = torch.cuda.current_stream()
for i in range(6):
    k, v = w["kv"][i % 2]
    ctx.mfa_decode_attention(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], 0.0625, stream=s.cuda_stream)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 1024)()  # 4 stamps x 256 CTAs
    lib.afdk_debug_mfa_times(buf)
    t = np.array(buf[:4 * 148], dtype=np.int64).reshape(148, 4)
    t0 = t[:, 0].min()
    t = (t - t0) / 1e3
    if i >= 3:
        q = lambda c: np.percentile(t[:, c], [0, 50, 100]).round(2).tolist()
        print(f"start {q(0)} first-S {q(1)} last-seg-done {q(2)} end {q(3)}  (us; min/median/max over CTAs)")
        ends = np.sort(t[:, 3])
        print("  end deciles:", np.percentile(t[:, 3], [10, 25, 50, 75, 90, 100]).round(2).tolist())
        pages = (w["seq_lens"].cpu().numpy() + 63) // 64
        units = np.where(pages > 0, pages + 3, 0)  # kSegCost = 3 page-less units per request (mfa_common.cuh)
        pre = np.concatenate([[0], np.cumsum(units)])
        T, G = pre[-1], 148
        segs = []
        for c in range(G):
            lo, hi = c * T // G, (c + 1) * T // G
            segs.append(int(((pre[1:] > lo) & (pre[:-1] < hi)).sum()))
        segs = np.array(segs)
        for k in sorted(set(segs.tolist())):
            m = segs == k
            print(f"  {k} segments: {m.sum()} CTAs, end median {np.median(t[m, 3]):.2f} max {t[m, 3].max():.2f}, "
                  f"first-S median {np.median(t[m, 1]):.2f}")
        slow = np.argsort(t[:, 3])[-8:]
        print("  slowest CTAs:", slow.tolist(), "SM-order ends:", t[slow, 3].round(1).tolist())
