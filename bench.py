"""bench.py — Step-3 decode hot path on B200 (driver contract).

N=1 workload (BASELINE.json configs[1]): Step-3 MFA decode attention, full
dims (64 q-heads x 256, one shared K/V head, q_lora 2048), bf16, batch 64,
4K context.  One step = one attention-side decode layer for the whole batch
through the C-ABI (include/afdk.h).  Metric: decode tokens/sec (per Step-3
layer) — whole-job aggregate over ranks; N>1 runs N independent replicas
(DP attention, "replicas only": attention has no cross-GPU exchange).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/sec/GPU per Step-3 layer at 4K ctx; MFA attn HBM GB/s vs peak"
H, D, PAGE = 64, 256, 64
BATCH, CTX = 64, 4096
N_ROT = 3  # rotating KV-cache layers so the 268 MB/step working set never hits L2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--batch", type=int, default=BATCH)
    p.add_argument("--ctx", type=int, default=CTX)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(sm)}


# --------------------------------------------------------------- workload
def make_workload(torch, dev, batch, ctx_len, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    pages_per_req = (ctx_len + PAGE - 1) // PAGE
    num_pages = batch * pages_per_req
    w = {}
    w["q"] = torch.randn(batch, H, D, generator=g).to(torch.bfloat16).to(dev)
    # page ids shuffled so requests are not contiguous in HBM (a real paged cache)
    perm = torch.randperm(num_pages, generator=g).to(torch.int32)
    w["block_table"] = perm.view(batch, pages_per_req).contiguous().to(dev)
    w["seq_lens"] = torch.full((batch,), ctx_len, dtype=torch.int32, device=dev)
    w["kv"] = []
    for _ in range(N_ROT):
        k = torch.empty(num_pages, PAGE, D, dtype=torch.bfloat16, device=dev).normal_()
        v = torch.empty(num_pages, PAGE, D, dtype=torch.bfloat16, device=dev).normal_()
        w["kv"].append((k, v))
    w["out"] = torch.empty(batch, H, D, dtype=torch.bfloat16, device=dev)
    w["num_pages"] = num_pages
    return w


def kv_bytes(batch, ctx_len):
    return batch * ctx_len * 2 * D * 2  # K + V rows, bf16 (== 2 x kv_state_bytes/61 x batch)


# ------------------------------------------------------------- reference arm
def cpu_attention_sample(batch_sample, ctx_len, seed=0):
    """Times the CPU oracle port (all host threads) on `batch_sample` requests."""
    import numpy as np

    from oracle import oracle as orc

    rng = np.random.default_rng(seed)
    pages = (ctx_len + PAGE - 1) // PAGE
    q = rng.standard_normal((batch_sample, H, D)).astype(np.float32)
    k = rng.standard_normal((batch_sample * pages, PAGE, D)).astype(np.float32)
    v = rng.standard_normal((batch_sample * pages, PAGE, D)).astype(np.float32)
    bt = np.arange(batch_sample * pages, dtype=np.int32).reshape(batch_sample, pages)
    sl = np.full(batch_sample, ctx_len, np.int32)
    t0 = time.perf_counter()
    orc.mfa_decode_attention(q, k, v, bt, sl, D ** -0.5)
    dt = time.perf_counter() - t0
    return batch_sample / dt, dt, orc.num_threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = 4
    for _ in range(args.warmup):
        cpu_attention_sample(1, args.ctx)
    vals, total = [], 0.0
    for s in range(args.steps):
        v, dt, cores = cpu_attention_sample(sample, args.ctx, seed=s)
        vals.append(v)
        total += dt
    value = sum(vals) / len(vals)
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "config2-mfa-decode-attention", "batch": args.batch, "ctx": args.ctx,
                       "sample_requests_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"{sample} requests x {args.ctx} ctx per step (oracle/afd_oracle.c, OpenMP)"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- B200 arm
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")

    from paper_2507_19427_b200 import Context

    ctx = Context(local)
    w = make_workload(torch, dev, args.batch, args.ctx, seed=rank)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    scale = D ** -0.5

    def step(i):
        k, v = w["kv"][i % N_ROT]
        ctx.mfa_decode_attention(w["q"], k, v, w["block_table"], w["seq_lens"], w["out"], scale, stream=sp)

    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()

    # ---- device-timed region (inputs resident in HBM)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * args.batch / (ms * 1e-3)

    # ---- dominant-kernel roofline: per-launch CUDA events on the launch stream
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        evs[i][0].record(stream)
        step(i)
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    op_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    hbm_peak, tf_peak, peak_kind = peaks()
    alg_bytes = kv_bytes(args.batch, args.ctx) + 2 * args.batch * H * D * 2  # KV + q + out
    achieved = alg_bytes / (op_ms * 1e-3) / 1e9

    # ---- end to end through the C-ABI: pinned host q in, host out back, per step
    q_host = w["q"].cpu().pin_memory()
    out_host = torch.empty_like(w["out"], device="cpu").pin_memory()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        w["q"].copy_(q_host, non_blocking=True)
        step(i)
        out_host.copy_(w["out"], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * args.batch / (e2e_ms * 1e-3)

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, dt, cores = cpu_attention_sample(2, args.ctx)
            v2, dt2, _ = cpu_attention_sample(2, args.ctx, seed=1)
            cpu = {"value": (v + v2) / 2, "unit": "tokens/s", "cores": cores, "kind": "port",
                   "sample": f"2 requests x {args.ctx} ctx attention core, twice (oracle/afd_oracle.c, OpenMP)"}
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("mfa_decode_kernel")
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config2-mfa-decode-attention (K2+K3, paged bf16 KV)", "batch": args.batch,
                       "ctx": args.ctx, "n_heads": H, "head_dim": D, "page": PAGE,
                       "parallelism": f"dp{world} (replicas)",
                       "l2": f"inputs > L2: {N_ROT} rotating KV layers of {kv_bytes(args.batch, args.ctx)/1e6:.0f} MB"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "mfa_decode (plan+K2+K3)", "alg_bytes_per_launch": alg_bytes,
                         "launch_ms": op_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s",
                    "h2d_bytes_per_step": q_host.numel() * 2, "d2h_bytes_per_step": out_host.numel() * 2},
            "gpu_launches": 3 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
