"""CPU coverage of the AFD host logic (paper_2507_19427_b200/afd.py).

* shard arithmetic: routed experts and shared-expert tokens are covered
  exactly once by the FFN GPUs for every tier size;
* wire accounting agrees with the reference's ffn_net_bytes
  (moeplan.cpp:17-20) for a single FFN GPU;
* a real multi-process run of the A->F / F->A protocol over torch.distributed
  gloo (world size 3: 1 attention + 2 FFN ranks, 127.0.0.1): the attention
  rank packs the dispatch payload, FFN ranks compute their EP partials on
  their expert shard + shared-token shard, the attention rank reduces the
  partials; the result must equal the single-process MoE layer.  Compute is
  done with the CPU oracle here (test double for the GPU kernels).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2507_19427_b200.afd import AfdConfig, PayloadLayout, expert_shard, shared_token_shard, wire_bytes


@pytest.mark.parametrize("n_ffn", [1, 2, 3, 4, 5, 6, 7, 8])
def test_expert_and_token_shards_partition(n_ffn):
    cfg = AfdConfig(n_attn=2, n_ffn=n_ffn, T_mb=37)
    experts = [e for f in range(n_ffn) for e in range(*expert_shard(f, cfg))]
    assert experts == list(range(48))
    toks = [t for f in range(n_ffn) for t in range(*shared_token_shard(f, cfg))]
    assert toks == list(range(cfg.T_ffn))


def test_payload_layout_aligned_and_complete():
    lay = PayloadLayout(T=100, H=7168, k=3)
    offs = sorted(lay.off.values())
    assert all(o % 256 == 0 for o in offs)
    assert lay.nbytes >= sum(lay.size(n) for n in ("xq", "xs", "ids", "wts"))
    assert lay.size("xq") == 100 * 7168 and lay.size("xs") == 100 * 56 * 4


@pytest.mark.parametrize("T_mb", [1, 128, 256])
def test_wire_bytes_match_reference_accounting(T_mb):
    cfg = AfdConfig(n_attn=1, n_ffn=1, T_mb=T_mb)
    wb = wire_bytes(cfg)
    assert wb["payload_a2f"] + wb["payload_f2a"] == orc.ref_ffn_net_bytes(T_mb)


# ------------------------------------------------------- gloo protocol run
H, I, E, K, T = 256, 128, 6, 2, 10


def _experts(seed=5):
    rng = np.random.default_rng(seed)
    w13 = np.zeros((E + 1, 2 * I, H), np.uint8)
    s13 = np.zeros((E + 1, 2 * I // 128, H // 128), np.float32)
    w2 = np.zeros((E + 1, H, I), np.uint8)
    s2 = np.zeros((E + 1, H // 128, I // 128), np.float32)
    for e in range(E + 1):
        w13[e], s13[e] = orc.quant_fp8_tile(rng.standard_normal((2 * I, H)).astype(np.float32) / 16)
        w2[e], s2[e] = orc.quant_fp8_tile(rng.standard_normal((H, I)).astype(np.float32) / 11)
    return w13, s13, w2, s2


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = AfdConfig(n_attn=1, n_ffn=world - 1, T_mb=T, hidden=H, inter=I, n_experts=E, top_k=K)
    w13, s13, w2, s2 = _experts()
    lay = PayloadLayout(T, H, K)
    if rank == 0:  # attention GPU: router + FP8 dispatch payload, broadcast to every FFN rank
        rng = np.random.default_rng(1)
        h = orc.bf16_round(rng.standard_normal((T, H)).astype(np.float32))
        ids, wts = orc.router_topk(rng.standard_normal((T, E)).astype(np.float32), K)
        xq, xs = orc.quant_fp8_rowblock(h)
        payload = np.zeros(lay.nbytes, np.uint8)
        for name, arr in (("xq", xq), ("xs", xs), ("ids", ids), ("wts", wts)):
            b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
            payload[lay.off[name]:lay.off[name] + b.size] = b
        for f in range(1, world):
            dist.send(torch.from_numpy(payload), dst=f)
        total = np.zeros((T, H), np.float32)
        for f in range(1, world):
            part = torch.empty(T, H, dtype=torch.float32)
            dist.recv(part, src=f)
            total += part.numpy()
        ref = orc.moe_layer_fp8(xq, xs, ids, wts, w13, s13, w2, s2, round_bf16=False)
        q.put(float(np.max(np.abs(total - ref)) / np.max(np.abs(ref))))
    else:  # FFN GPU f: its expert shard + its share of the shared expert's tokens
        f = rank - 1
        buf = torch.empty(lay.nbytes, dtype=torch.uint8)
        dist.recv(buf, src=0)
        raw = buf.numpy()
        get = lambda n, dt, shape: raw[lay.off[n]:lay.off[n] + lay.size(n)].view(dt).reshape(shape)
        xq, xs = get("xq", np.uint8, (T, H)), get("xs", np.float32, (T, H // 128))
        ids, wts = get("ids", np.int32, (T, K)), get("wts", np.float32, (T, K))
        lo, hi = expert_shard(f, cfg)
        slo, shi = shared_token_shard(f, cfg)
        part = np.zeros((T, H), np.float64)
        for t in range(T):
            for j in range(K):
                e = int(ids[t, j])
                if lo <= e < hi:
                    part[t] += wts[t, j] * orc.expert_ffn_fp8(xq[t:t + 1], xs[t:t + 1], w13[e], s13[e], w2[e], s2[e])[0]
            if slo <= t < shi:
                part[t] += orc.expert_ffn_fp8(xq[t:t + 1], xs[t:t + 1], w13[E], s13[E], w2[E], s2[E])[0]
        dist.send(torch.from_numpy(part.astype(np.float32)), dst=0)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_afd_protocol_gloo(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) <= 1e-5


def test_afd_config_validation():
    import pytest

    from paper_2507_19427_b200.afd import AfdConfig

    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=8192)
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, attn_chunk=512)
    AfdConfig(n_attn=1, n_ffn=1, T_mb=768)
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, ffn_format="bf16")
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, ffn_format="mx", inter=256)
    AfdConfig(n_attn=2, n_ffn=6, T_mb=256, ffn_format="mx")
