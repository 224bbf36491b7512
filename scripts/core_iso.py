"""MFA core (K2+K3) at config 2: isolated launches (synchronised, events around
each) vs back-to-back (events around 20 launches)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2507_19427_b200 import Context  # noqa: E402

ctx = Context(0)
dev = torch.device("cuda:0")
s = bench.make_workload(torch, dev, 64, 4096)
st = torch.cuda.current_stream()
sp = st.cuda_stream


def core(i):
    k, v = s["kv"][i % bench.N_ROT]
    ctx.mfa_decode_attention(s["q"], k, v, s["block_table"], s["seq_lens"], s["attn_out"], 0.0625, stream=sp)


for i in range(5):
    core(i)
torch.cuda.synchronize()
iso = []
for i in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    core(i)
    b.record(st)
    torch.cuda.synchronize()
    iso.append(a.elapsed_time(b) * 1e3)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for i in range(20):
    core(i)
b.record(st)
torch.cuda.synchronize()
iso.sort()
print(f"isolated us: min {iso[0]:.1f} median {iso[10]:.1f}; back-to-back {a.elapsed_time(b) * 1e3 / 20:.1f} us/launch")
