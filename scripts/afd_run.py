"""AFD pipeline timing driver: torchrun --nproc-per-node N scripts/afd_run.py --n-attn A

Runs the C++ AFD runtime (through paper_2507_19427_b200.afd) at full Step-3
dims and prints one JSON line (rank 0) with the measured layer period and
throughput.  Correctness: tests/afd_gpu_check.py (pytest tests/test_afd_gpu.py).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-attn", type=int, default=1)
    ap.add_argument("--T-mb", type=int, default=128)
    ap.add_argument("--n-micro", type=int, default=2)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--ctx-len", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--fmt", default="fp8", choices=["fp8", "mx", "bf16"])
    ap.add_argument("--kv", default="bf16", choices=["bf16", "e4m3"])
    ap.add_argument("--f2a", default="push", choices=["push", "pull"])
    ap.add_argument("--attn-chunk", type=int, default=256)
    ap.add_argument("--layer", default="moe", choices=["moe", "dense"])
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2507_19427_b200 import Context
    from paper_2507_19427_b200.afd import AfdConfig, AfdRank, wire_bytes

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # AFDK_OVERSUB=1: more ranks than GPUs: ranks share GPUs round-robin and the
    # rendezvous runs on gloo (NCCL refuses two ranks on one device)
    oversub = os.environ.get("AFDK_OVERSUB") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cfg = AfdConfig(n_attn=a.n_attn, n_ffn=world - a.n_attn, T_mb=a.T_mb, n_micro=a.n_micro, layers=a.layers,
                    ctx_len=a.ctx_len, ffn_format=a.fmt, f2a=a.f2a, attn_chunk=a.attn_chunk, layer_kind=a.layer,
                    kv=a.kv)
    ctxs = [Context(local) for _ in range(cfg.n_micro)]
    r = AfdRank(ctxs, cfg, rank, torch, dist, dev)
    r.setup()

    def run(n):
        dist.barrier()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        start.record(torch.cuda.current_stream())
        for s in r.streams_all():
            s.wait_event(start)
        for _ in range(n):
            r.step()
        cur = torch.cuda.current_stream()
        for s in r.streams_all():
            ev = torch.cuda.Event()
            ev.record(s)
            cur.wait_event(ev)
        end = torch.cuda.Event(enable_timing=True)
        end.record(cur)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end)
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(a.warmup):
        r.reset_inputs()
        run(1)
    ms = run(a.steps)
    period_ms = ms / (a.steps * cfg.layers)
    tokens = cfg.n_attn * cfg.n_micro * cfg.T_mb
    wb = wire_bytes(cfg)
    if rank == 0:
        print(json.dumps({"afd": f"{cfg.n_attn}A{cfg.n_ffn}F", "fmt": cfg.ffn_format, "f2a": cfg.f2a, "world": world, "T_mb": cfg.T_mb,
                          "n_micro": cfg.n_micro, "layers": cfg.layers, "ctx": cfg.ctx_len,
                          "layer_period_ms": period_ms, "tokens_per_layer_period": tokens,
                          "tokens_per_s": tokens / (period_ms * 1e-3),
                          "tokens_per_s_per_gpu": tokens / (period_ms * 1e-3) / world,
                          "wire_bytes_per_layer": {k: v * cfg.n_micro for k, v in wb.items()}}), flush=True)
    dist.barrier()
    r.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
