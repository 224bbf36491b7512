"""Measure the fp8 tensor-core denominators on this B200 with the library
(cuBLASLt through torch._scaled_mm), the way MEASURED_PEAKS.json measures bf16:

  * e4m3 x e4m3, per-tensor scales, 8192^3: best of 10 (burst) and back to
    back for 4 s (sustained, clocks under power draw);
  * MXFP8 (e4m3 + UE8M0 per 32 along K), 8192^3: same two figures;
  * the library doing our MoE layer's GEMM work: one MXFP8 _scaled_mm per
    routed expert (48 experts, T=4096 top-3 uniform routing, + the shared
    expert over all T) for W13 [10240 x 7168] and W2 [7168 x 5120], captured
    in a CUDA graph so launch gaps do not count.

Prints one JSON object; scripts/gpu_fp8_peaks.sh copies it to profiles/.
"""
import json
import sys
import time

import torch

E4 = torch.float8_e4m3fn
E8 = torch.float8_e8m0fnu


def rup(a, b):
    return (a + b - 1) // b * b


def mx_scales(rows, k):
    n = rup(rows, 128) * rup(k // 32, 4)
    return torch.full((n,), 127, dtype=torch.uint8, device="cuda").view(E8)


def operands(m, n, k, mx):
    a = (torch.randn(m, k, device="cuda") * 0.5).to(E4)
    b = (torch.randn(n, k, device="cuda") * 0.5).to(E4).t()   # column-major [k, n]
    if mx:
        sa, sb = mx_scales(m, k), mx_scales(n, k)
    else:
        sa = torch.ones((), device="cuda")
        sb = torch.ones((), device="cuda")
    return a, b, sa, sb


def mm(a, b, sa, sb):
    return torch._scaled_mm(a, b, sa, sb, out_dtype=torch.bfloat16)


def time_best(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def time_sustained(fn, seconds=4.0):
    fn(); torch.cuda.synchronize()
    n = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    s.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        if n % 200 == 0:
            torch.cuda.synchronize()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n


def peak(mx, size=8192):
    a, b, sa, sb = operands(size, size, size, mx)
    fl = 2.0 * size ** 3
    burst = time_best(lambda: mm(a, b, sa, sb))
    sust = time_sustained(lambda: mm(a, b, sa, sb))
    return {"burst_tflops": fl / burst / 1e9, "sustained_tflops": fl / sust / 1e9,
            "shape": [size, size, size]}


def expert_loop(T=4096, E=48, topk=3, hidden=7168, inter=5120, seed=0):
    g = torch.Generator().manual_seed(seed)
    ids = torch.stack([torch.randperm(E, generator=g)[:topk] for _ in range(T)])
    counts = torch.bincount(ids.flatten(), minlength=E).tolist() + [T]
    w13 = [(torch.randn(2 * inter, hidden, device="cuda") * 0.05).to(E4) for _ in range(E + 1)]
    w2 = [(torch.randn(hidden, inter, device="cuda") * 0.05).to(E4) for _ in range(E + 1)]
    s13 = [mx_scales(2 * inter, hidden) for _ in range(E + 1)]
    s2 = [mx_scales(hidden, inter) for _ in range(E + 1)]
    # cuBLASLt wants N % 16 == 0: each expert's token count is padded up
    # (the padding's flops are not credited below)
    pc = [rup(max(c, 1), 16) for c in counts]
    xs = [(torch.randn(c, hidden, device="cuda")).to(E4) for c in pc]
    hs = [(torch.randn(c, inter, device="cuda")).to(E4) for c in pc]
    sx = [mx_scales(c, hidden) for c in pc]
    sh = [mx_scales(c, inter) for c in pc]
    # weights as the M operand (swap-AB, as our kernels do): out^T = W x^T

    def run13():
        for i in range(E + 1):
            torch._scaled_mm(w13[i], xs[i].t(), s13[i], sx[i], out_dtype=torch.bfloat16)

    def run2():
        for i in range(E + 1):
            torch._scaled_mm(w2[i], hs[i].t(), s2[i], sh[i], out_dtype=torch.bfloat16)

    res = {}
    for name, fn, m, k in (("w13", run13, 2 * inter, hidden), ("w2", run2, hidden, inter)):
        fn(); torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            fn()
        ms = time_best(graph.replay, reps=20)
        fl = sum(2.0 * m * k * c for c in counts)
        res[name] = {"ms": ms, "tflops": fl / ms / 1e9}
    a, b, sa, sb = operands(2 * inter, 256, hidden, True)
    ms = time_best(lambda: mm(a, b, sa, sb), reps=20)
    res["one_expert_w13_N256"] = {"ms": ms, "tflops": 2.0 * 2 * inter * 256 * hidden / ms / 1e9}
    res["counts_routed_mean"] = sum(counts[:E]) / E
    res["T"] = T
    return res


def main():
    out = {"gpu": torch.cuda.get_device_name(), "torch": torch.__version__,
           "how": "torch._scaled_mm (cuBLASLt) out bf16; burst = best of 10, "
                  "sustained = back to back for 4 s"}
    for key, mx in (("fp8_tensorwise", False), ("mxfp8", True)):
        try:
            out[key] = peak(mx)
        except Exception as exc:   # report, keep measuring the rest
            out[key] = {"error": str(exc).splitlines()[0][:200]}
    for T in (4096, 8192):
        try:
            out[f"library_expert_loop_T{T}"] = expert_loop(T=T)
        except Exception as exc:
            out[f"library_expert_loop_T{T}"] = {"error": str(exc).splitlines()[0][:200]}
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
