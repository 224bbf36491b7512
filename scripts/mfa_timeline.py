"""Launch timeline of back-to-back MFA core launches (K2 + K3) in the
diagnostic build (-DAFDK_MFA_TIMES=1):
    AFDK_LIB=paper_2507_19427_b200/libafdk_times.so python scripts/mfa_timeline.py [B ctx fp8]
Per launch n (times in us relative to K2(n)'s first PDL release):
  K2 first entry, last release, last end; K3 first entry, last wait done,
  last exit; and the gap to K2(n+1)'s release."""
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
FP8 = len(sys.argv) > 3 and sys.argv[3] == "fp8"
N = 24
ctx = Context(0)
lib = ctypes.CDLL(os.environ["AFDK_LIB"])
dev = torch.device("cuda:0")
w = bench.make_workload_attn(torch, dev, B, L)
npages = w["kv"][0][0].shape[0]
kv8 = [(torch.randint(0, 0x7e, (npages, 64, 256), dtype=torch.uint8, device=dev),
        torch.randint(0, 0x7e, (npages, 64, 256), dtype=torch.uint8, device=dev)) for _ in range(2)]
s = torch.cuda.current_stream()


def step(i):
    if FP8:
        k, v = kv8[i % 2]
        ctx.mfa_decode_attention_fp8(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], 0.0625, 0.01, 0.01,
                                     stream=s.cuda_stream)
    else:
        k, v = w["kv"][i % 2]
        ctx.mfa_decode_attention(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], 0.0625,
                                 stream=s.cuda_stream)


for i in range(4):
    step(i)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 8))()
lib.afdk_debug_mfa_tl(buf, 1)
if FP8:
    lib.afdk_debug_mfa8_tl(buf, 1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for i in range(N):
    step(i)
b.record(s)
torch.cuda.synchronize()
print(f"{'fp8' if FP8 else 'bf16'} B={B} ctx={L}: {a.elapsed_time(b) / N * 1e3:.1f} us per launch (events)")
lib.afdk_debug_mfa_tl(buf, 0)
t3 = np.array(buf[:], dtype=np.float64).reshape(64, 8)
if FP8:
    lib.afdk_debug_mfa8_tl(buf, 0)
    t2 = np.array(buf[:], dtype=np.float64).reshape(64, 8)
    t = np.concatenate([t2[:, :4], t3[:, 4:]], axis=1)
else:
    t = t3
rows = []
for n in range(N - 1):
    r0 = t[n, 1]
    rel = (t[n] - r0) / 1e3
    nxt = (t[n + 1, 1] - r0) / 1e3
    nxt_entry = (t[n + 1, 0] - r0) / 1e3
    rows.append([rel[0], rel[2], rel[3], rel[4], rel[5], rel[6], nxt_entry, nxt])
rows = np.array(rows)
hdr = ["K2 entry", "K2 last rel", "K2 end", "K3 entry", "K3 wait done", "K3 exit", "K2' entry", "K2' release"]
print("   ".join(f"{h:>12s}" for h in hdr))
for r in rows[-6:]:
    print("   ".join(f"{x:12.2f}" for x in r))
print("median:", "   ".join(f"{x:.2f}" for x in np.median(rows[2:], axis=0)))
