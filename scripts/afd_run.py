"""AFD pipeline driver: torchrun --nproc-per-node N scripts/afd_run.py --n-attn A [--check]

--check: small dims, one layer; attention rank 0 recomputes the whole layer
(attention + router + all experts) on its own GPU and compares.
Prints one JSON line (rank 0) with the measured layer period and throughput.
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
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--fmt", default="fp8", choices=["fp8", "mx"])
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
    # AFDK_OVERSUB=1: more ranks than GPUs (e.g. the 8-rank protocol on a 4-GPU
    # box for --check): ranks share GPUs round-robin and the rendezvous runs on
    # gloo (NCCL refuses two ranks on one device)
    oversub = os.environ.get("AFDK_OVERSUB") == "1"
    if oversub:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if oversub:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    if a.check:
        cfg = AfdConfig(n_attn=a.n_attn, n_ffn=world - a.n_attn, T_mb=24, n_micro=2, layers=1, hidden=1024,
                        q_lora=256, ctx_len=300, n_experts=8 if (world - a.n_attn) in (1, 2, 4, 8) else 24, top_k=2, inter=512, seed=3, ffn_format=a.fmt, f2a=a.f2a,
                        attn_chunk=min(a.attn_chunk, 256), layer_kind=a.layer, dense_inter=2048 * 6)
    else:
        cfg = AfdConfig(n_attn=a.n_attn, n_ffn=world - a.n_attn, T_mb=a.T_mb, n_micro=a.n_micro, layers=a.layers,
                        ctx_len=a.ctx_len, ffn_format=a.fmt, f2a=a.f2a, attn_chunk=a.attn_chunk,
                        layer_kind=a.layer)
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

    if a.check:
        run(1)
        ok = True
        if rank == 0:
            from tests.helpers import rel_err
            c = cfg
            wall = r.expert_weights(0, c.n_experts)
            errs = []
            for mb in range(c.n_micro):
                k, v, bt = r.kv[0][mb]
                h_res = torch.empty_like(r.x0[mb])
                h_norm = torch.empty_like(r.x0[mb])
                ctxs[0].mfa_layer(r.w, r.x0[mb], k, v, bt, r.seq_lens, h_res, h_norm)
                ids = torch.empty(c.T_mb, c.top_k, dtype=torch.int32, device=dev)
                wts = torch.empty(c.T_mb, c.top_k, device=dev)
                xq = torch.empty(c.T_mb, c.hidden, dtype=torch.uint8, device=dev)
                part = torch.empty_like(h_res)
                if c.layer_kind == "dense":
                    xs = torch.empty(c.T_mb, c.hidden // 32, dtype=torch.uint8, device=dev)
                    ctxs[0].quant_mx(h_norm, xq, xs)
                    ctxs[0].dense_ffn_mx(r.dense_weights(0, c.dense_slices_total), xq, xs, part)
                elif c.ffn_format == "mx":
                    xs = torch.empty(c.T_mb, c.hidden // 32, dtype=torch.uint8, device=dev)
                    ctxs[0].router_topk(h_norm, r.w["gate"], c.top_k, ids, wts)
                    ctxs[0].quant_mx(h_norm, xq, xs)
                    ctxs[0].moe_ffn_mx(wall, xq, xs, ids, wts, part)
                else:
                    xs = torch.empty(c.T_mb, c.hidden // 128, device=dev)
                    ctxs[0].router_topk(h_norm, r.w["gate"], c.top_k, ids, wts, xq=xq, xs=xs)
                    ctxs[0].moe_ffn(wall, xq, xs, ids, wts, part)
                torch.cuda.synchronize()
                ref = (h_res.float() + part.float())
                errs.append(rel_err(r.x[mb].float().cpu().numpy(), ref.cpu().numpy()))
                L = r.lay
                sb = r.send[mb]
                sent_xq = sb[L.off["xq"]:L.off["xq"] + L.size("xq")].view(c.T_mb, c.hidden)
                sent_ids = sb[L.off["ids"]:L.off["ids"] + L.size("ids")].view(torch.int32).view(c.T_mb, c.top_k)
                print("mb", mb, "x err", errs[-1], "h_res err", rel_err(r.h_res[mb].float().cpu().numpy(), h_res.float().cpu().numpy()),
                      "part err", rel_err(r.recv_part[mb][0].float().cpu().numpy(), part.float().cpu().numpy()),
                      "xq eq", bool(torch.equal(sent_xq, xq)), "ids eq", bool(torch.equal(sent_ids, ids)), flush=True)
            ok = max(errs) <= 2e-2
            print(json.dumps({"afd_check": "ok" if ok else "FAIL", "layer": c.layer_kind, "fmt": c.ffn_format, "f2a": c.f2a, "rel_err": errs, "world": world,
                              "n_attn": cfg.n_attn}), flush=True)
        dist.barrier()
        r.close()
        dist.destroy_process_group()
        sys.exit(0 if ok else 1)

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
