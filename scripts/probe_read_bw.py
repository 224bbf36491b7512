"""Read-only HBM bandwidth probe (torch reduction over 2 GiB, best of 10): the
practical ceiling of a pure read stream, next to the copy peak in MEASURED_PEAKS.json."""
import torch

x = torch.ones(2**30, dtype=torch.bfloat16, device="cuda")
best = 1e9
for _ in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); x.sum(dtype=torch.float32); b.record(); b.synchronize()
    best = min(best, a.elapsed_time(b))
print(f"read-only sum over 2 GiB: {2**31 / (best * 1e-3) / 1e9:.0f} GB/s")
