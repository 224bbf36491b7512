"""bf16 vs MXFP8 projections at the attention shapes (GEMM + the fixed-order store kernel), CUDA events:
python scripts/bench_linear_mx.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_19427_b200 import Context

ctx = Context(0)
dev = torch.device("cuda:0")
s = torch.cuda.current_stream()
for m, n, k in [(64, 2560, 7168), (64, 16384, 2048), (64, 7168, 16384), (256, 2560, 7168), (256, 16384, 2048),
                (256, 7168, 16384)]:
    ws = [(torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16) for _ in range(3)]  # rotate: > L2
    x = torch.randn(m, k, device=dev).to(torch.bfloat16)
    wq = [torch.empty(n, k, dtype=torch.uint8, device=dev) for _ in range(3)]
    wsf = [torch.empty(n, k // 32, dtype=torch.uint8, device=dev) for _ in range(3)]
    for i in range(3):
        ctx.quant_mx(ws[i], wq[i], wsf[i])
    xq = torch.empty(m, k, dtype=torch.uint8, device=dev)
    xsf = torch.empty(m, k // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(x, xq, xsf)
    out = torch.empty(m, n, dtype=torch.bfloat16, device=dev)

    def run(f, iters=30):
        for i in range(5):
            f(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for i in range(iters):
            f(i)
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters * 1e3

    t16 = run(lambda i: ctx.linear(x, ws[i % 3], out, stream=s.cuda_stream))
    t8 = run(lambda i: ctx.linear_mx(xq, xsf, wq[i % 3], wsf[i % 3], out, stream=s.cuda_stream))
    wb16, wb8 = n * k * 2, n * k * (1 + 1 / 32)
    print(f"m={m} n={n} k={k}: bf16 {t16:.1f} us ({wb16 / t16 / 1e3:.0f} GB/s)  mxfp8 {t8:.1f} us "
          f"({wb8 / t8 / 1e3:.0f} GB/s)  speed-up {t16 / t8:.2f}x", flush=True)
