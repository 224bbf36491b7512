"""Multi-process check of the C++ AFD runtime on the GPU (TEST HARNESS).

    torchrun --nproc-per-node N tests/afd_gpu_check.py --n-attn A [--fmt fp8|mx|bf16] [--f2a push|pull]
             [--kv bf16|e4m3] [--layer moe|dense] [--attn-chunk C] [--out result.json]

Runs the real runtime (afdk_afd_create / attn_layer / ffn_layer, IPC-mapped
buffers, flags, copy-engine pulls, fused F->A scatter) for STEPS steps x
LAYERS layers x 2 micro-batches at small dims, buffers reused across
sequence numbers.  Every layer's output x is snapshotted on the runtime's
own micro-batch stream (a stream-ordered copy between the layer's REDUCE and
the next layer's ATTN).  After every step, EVERY attention rank recomputes
each layer on its own GPU from the runtime's input to that layer (the
step's input, then the previous layer's snapshot) — attention layer,
router / dispatch quantisation and the whole MoE (all experts, no expert
parallelism) through the single-GPU C-ABI calls — and compares the layer's
output (rel = max|afd - ref| / max|ref|; bar 2e-2: the runtime sums
bf16-rounded EP partials where the recompute rounds the whole layer once).
Per-layer inputs matter: recomputing several layers from the step's input
lets those one-ulp differences reach the next layer's router, where a
near-tie top-k flips a token to another expert (seen as sporadic 3-7e-2
errors with bf16 experts in round 2's 12-step soaks).

Ranks beyond the visible GPU count share GPUs round-robin (IPC between
processes on one device works), with a gloo rendezvous.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LAYERS = 2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-attn", type=int, default=1)
    ap.add_argument("--fmt", default="fp8", choices=["fp8", "mx", "bf16"])
    ap.add_argument("--f2a", default="push", choices=["push", "pull", "nvls"])
    ap.add_argument("--kv", default="bf16", choices=["bf16", "e4m3"])
    ap.add_argument("--layer", default="moe", choices=["moe", "dense"])
    ap.add_argument("--attn-chunk", type=int, default=256)
    ap.add_argument("--T-mb", type=int, default=24)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--o-mx", type=int, default=0,
                    help="1: o_proj, 2: o_proj and q_up as MXFP8 GEMMs on the attention ranks")
    ap.add_argument("--full", type=int, default=0,
                    help="Step-3 dims (hidden 7168, q_lora 2048, 48 experts top-3, inter 5120, 4K context): the "
                         "benchmarked AFD configuration")
    a = ap.parse_args()
    STEPS = a.steps
    import torch
    import torch.distributed as dist

    from paper_2507_19427_b200 import Context
    from paper_2507_19427_b200.afd import AfdConfig, AfdRank

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    shared_gpu = world > torch.cuda.device_count()
    dist.init_process_group("gloo" if shared_gpu else "nccl", **({} if shared_gpu else {"device_id": dev}))
    nf = world - a.n_attn
    dims = dict(hidden=7168, q_lora=2048, ctx_len=4096, n_experts=48, top_k=3, inter=5120, dense_inter=18432) \
        if a.full else dict(hidden=1024, q_lora=512 if a.o_mx >= 2 else 256, ctx_len=300, n_experts=8 if nf in (1, 2, 4, 8) else 24,
                            top_k=2, inter=512, dense_inter=2048 * 6)
    cfg = AfdConfig(n_attn=a.n_attn, n_ffn=nf, T_mb=a.T_mb, n_micro=2, layers=a.layers, seed=3,
                    ffn_format=a.fmt, f2a=a.f2a, kv=a.kv, layer_kind=a.layer, attn_chunk=a.attn_chunk,
                    attn_o_mx=a.o_mx >= 1, attn_qup_mx=a.o_mx >= 2, **dims)
    ctxs = [Context(local) for _ in range(cfg.n_micro)]
    r = AfdRank(ctxs, cfg, rank, torch, dist, dev)
    r.setup()
    errs = []
    if r.role == "attn":
        wall = r.dense_weights(0, cfg.dense_slices_total) if cfg.layer_kind == "dense" else \
            r.expert_weights(0, cfg.n_experts)
    c0 = ctxs[0]
    snaps = None
    if r.role == "attn":
        snaps = [[torch.empty_like(r.x[mb]) for mb in range(cfg.n_micro)] for _ in range(cfg.layers)]
        streams = r.streams_all()

    def snapshot(layer):  # stream-ordered copy of every micro-batch's layer output
        if r.role == "attn":
            for mb in range(cfg.n_micro):
                with torch.cuda.stream(streams[mb]):
                    snaps[layer][mb].copy_(r.x[mb])

    for step in range(STEPS):
        x_in = [x.clone() for x in r.x] if r.role == "attn" else None
        torch.cuda.synchronize()
        r.step(after_layer=snapshot)
        r.sync()
        dist.barrier()
        if r.role != "attn":
            continue
        for mb in range(cfg.n_micro):
            for layer in range(cfg.layers):
                x = x_in[mb] if layer == 0 else snaps[layer - 1][mb]
                k, v, bt, ks, vs = r.kv[layer][mb]
                h_res, h_norm = torch.empty_like(x), torch.empty_like(x)
                for s0 in range(0, cfg.T_mb, cfg.attn_chunk):
                    s1 = min(cfg.T_mb, s0 + cfg.attn_chunk)
                    c0.mfa_layer(r.w, x[s0:s1], k, v, bt[s0:s1], r.seq_lens[s0:s1], h_res[s0:s1], h_norm[s0:s1],
                                 **({"kv_scales": (ks, vs)} if cfg.kv == "e4m3" else {}))
                T = cfg.T_mb
                ids = torch.empty(T, cfg.top_k, dtype=torch.int32, device=dev)
                wts = torch.empty(T, cfg.top_k, device=dev)
                part = torch.empty_like(h_res)
                if cfg.layer_kind == "dense":
                    xq = torch.empty(T, cfg.hidden, dtype=torch.uint8, device=dev)
                    xs = torch.empty(T, cfg.hidden // 32, dtype=torch.uint8, device=dev)
                    c0.quant_mx(h_norm, xq, xs)
                    c0.dense_ffn_mx(wall, xq, xs, part)
                elif cfg.ffn_format == "mx":
                    xq = torch.empty(T, cfg.hidden, dtype=torch.uint8, device=dev)
                    xs = torch.empty(T, cfg.hidden // 32, dtype=torch.uint8, device=dev)
                    c0.router_topk(h_norm, r.w["gate"], cfg.top_k, ids, wts)
                    c0.quant_mx(h_norm, xq, xs)
                    c0.moe_ffn_mx(wall, xq, xs, ids, wts, part)
                elif cfg.ffn_format == "bf16":
                    c0.router_topk(h_norm, r.w["gate"], cfg.top_k, ids, wts)
                    c0.moe_ffn_bf16(wall, h_norm, ids, wts, part)
                else:
                    xq = torch.empty(T, cfg.hidden, dtype=torch.uint8, device=dev)
                    xs = torch.empty(T, cfg.hidden // 128, device=dev)
                    c0.router_topk(h_norm, r.w["gate"], cfg.top_k, ids, wts, xq=xq, xs=xs)
                    c0.moe_ffn(wall, xq, xs, ids, wts, part)
                x = (h_res.float() + part.float()).to(torch.bfloat16)
                torch.cuda.synchronize()
                ref, got = x.float(), snaps[layer][mb].float()
                errs.append(float((got - ref).abs().max() / ref.abs().max().clamp_min(1e-12)))
            assert torch.equal(snaps[-1][mb], r.x[mb])  # the last snapshot is the step's output
    # measured trace of one more step (afdk_afd_trace_start / _trace_csv)
    r.trace_start()
    r.step()
    csv = r.trace_csv()
    rows = [ln.split(",") for ln in csv.strip().splitlines()]
    want = {"attention"} if r.role == "attn" else {"ffn", "fwd_link"}
    if r.role == "attn" and cfg.f2a == "pull":
        want.add("bwd_link")
    got_res = {row[1] for row in rows[1:]}
    trace_ok = (rows[0] == ["time_s", "resource", "layer", "micro_batch", "stage", "duration_s"] and
                want <= got_res and {int(row[2]) for row in rows[1:]} == set(range(cfg.layers)) and
                all(float(row[5]) >= 0 for row in rows[1:]))
    if not trace_ok:
        print("bad trace on rank", rank, csv[:2000], flush=True)
        errs.append(1.0)
    allerr = [None] * world
    dist.all_gather_object(allerr, errs)
    flat = [e for es in allerr for e in es]
    ok = len(flat) == cfg.n_attn * cfg.n_micro * STEPS * cfg.layers and max(flat) <= 2e-2  # a bad trace adds one
    if rank == 0:
        res = {"afd_check": "ok" if ok else "FAIL", "world": world, "n_attn": cfg.n_attn, "fmt": cfg.ffn_format,
               "f2a": cfg.f2a, "kv": cfg.kv, "layer": cfg.layer_kind, "T_mb": cfg.T_mb, "attn_chunk": cfg.attn_chunk,
               "steps": STEPS, "layers": cfg.layers, "seq": STEPS * cfg.layers, "max_rel_err": max(flat), "rel_err": flat,
               "full_dims": bool(a.full),
               "shared_gpu": shared_gpu}
        print(json.dumps(res), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(res, f)
    dist.barrier()
    r.close()
    for c in ctxs:
        c.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
