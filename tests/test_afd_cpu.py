"""CPU coverage of the AFD host logic (paper_2507_19427_b200/afd.py).

* shard arithmetic: routed experts and shared-expert tokens are covered
  exactly once by the FFN GPUs for every tier size;
* wire accounting agrees with the reference's ffn_net_bytes
  (moeplan.cpp:17-20) for a single FFN GPU;
* the C++ runtime's own op list (afdk_afd_plan — what afdk_afd_attn_layer /
  afdk_afd_ffn_layer execute on the GPU) run by one process per rank over
  torch.distributed gloo (127.0.0.1) with the runtime's payload layout, for
  several steps/layers/micro-batches in fp8 / MXFP8 / bf16, push and pull
  (tests/afd_emulator.py: oracle compute doubles, flag-release memory
  model); every attention rank's activations must equal a single-process
  recompute bit for bit;
* op-list invariants (matched SIGNAL/WAIT slots, PULL ranges in bounds).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2507_19427_b200.afd import (OP_NAMES, AfdConfig, PayloadLayout, expert_shard, plan, shared_token_shard,
                                       wire_bytes)


@pytest.mark.parametrize("n_ffn", [1, 2, 3, 4, 5, 6, 7, 8])
def test_expert_and_token_shards_partition(n_ffn):
    cfg = AfdConfig(n_attn=2, n_ffn=n_ffn, T_mb=37)
    experts = [e for f in range(n_ffn) for e in range(*expert_shard(f, cfg))]
    assert experts == list(range(48))
    toks = [t for f in range(n_ffn) for t in range(*shared_token_shard(f, cfg))]
    assert toks == list(range(cfg.T_ffn))


def test_payload_layout_aligned_and_complete():
    lay = PayloadLayout(AfdConfig(n_attn=1, n_ffn=1, T_mb=100))
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
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # (n_attn, n_ffn, ffn_format, f2a)
    "1A2F-fp8-push": (1, 2, "fp8", "push"),
    "2A1F-mx-pull": (2, 1, "mx", "pull"),
    "1A1F-bf16-push": (1, 1, "bf16", "push"),
    "1A2F-mx-nvls": (1, 2, "mx", "nvls"),
}
STEPS, LAYERS = 3, 2


def _cfg(case):
    na, nf, fmt, f2a = CASES[case]
    return AfdConfig(n_attn=na, n_ffn=nf, T_mb=12, n_micro=2, layers=LAYERS, hidden=512, inter=512, n_experts=6,
                     top_k=2, ffn_format=fmt, f2a=f2a)


def _x0(cfg):
    rng = np.random.default_rng(11)
    return [[orc.bf16_round(rng.standard_normal((cfg.T_mb, cfg.hidden)).astype(np.float32))
             for _ in range(cfg.n_micro)] for _ in range(cfg.n_attn)]


def _worker(case, rank, world, port, q):
    import torch
    import torch.distributed as dist

    from tests import afd_emulator as emu

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg(case)
    m = emu.model(cfg)
    x0 = _x0(cfg)
    r = emu.Rank(cfg, rank, dist, torch, m, x0[rank] if rank < cfg.n_attn else None)
    seq = 0
    for _ in range(STEPS):
        for _ in range(LAYERS):
            seq += 1
            r.run_layer(seq)
    r.finish()
    if r.attn:
        q.put((rank, [v.copy() for v in r.x], r.log[:12]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_afd_runtime_plan_over_gloo(case):
    """Every rank executes the C++ runtime's own op list (afdk_afd_plan, the
    list afdk_afd_attn_layer / afdk_afd_ffn_layer run on the GPU) for 3 steps
    x 2 layers x 2 micro-batches over gloo, buffers reused across sequence
    numbers; every attention rank's activations must equal the single-process
    recompute bit for bit."""
    import torch.multiprocessing as mp

    from tests import afd_emulator as emu

    cfg = _cfg(case)
    world = cfg.world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(case, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(cfg.n_attn):
        rank, x, log = q.get(timeout=240)
        got[rank] = x
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ref = emu.reference_layers(cfg, emu.model(cfg), _x0(cfg), STEPS * LAYERS)
    for a in range(cfg.n_attn):
        for mb in range(cfg.n_micro):
            np.testing.assert_array_equal(got[a][mb], ref[a][mb])


def test_plan_structure_and_flag_slots():
    """Op-list invariants of the runtime's schedule (host only): every SIGNAL
    has exactly one matching WAIT on the peer (same slot and value); PULL
    ranges lie inside the runtime's buffers; FFN ranks join their copy
    stream before computing."""
    cfg = AfdConfig(n_attn=2, n_ffn=3, T_mb=40, n_experts=48, f2a="pull")
    L = PayloadLayout(cfg)
    sig, wai = [], []
    for r in range(cfg.world):
        ops = plan(cfg, r, 7)
        kinds = [OP_NAMES[o.kind] for o in ops]
        for o in ops:
            assert o.value == 7
            if OP_NAMES[o.kind] == "SIGNAL":
                sig.append((r, o.peer, o.slot))
            if OP_NAMES[o.kind] == "WAIT":
                wai.append((o.peer, r, o.slot))
            if OP_NAMES[o.kind] == "PULL":
                lim = L.rx_total if r >= cfg.n_attn else cfg.n_ffn * L.part_bytes
                assert o.dst_off + o.bytes <= lim
        if r >= cfg.n_attn:
            assert kinds.index("JOIN") < kinds.index("FFN")
    assert sorted(sig) == sorted(wai)


def test_afd_config_validation():
    import pytest

    from paper_2507_19427_b200.afd import AfdConfig

    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=8192)
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, attn_chunk=513)
    AfdConfig(n_attn=1, n_ffn=1, T_mb=768)
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, ffn_format="int4")
    AfdConfig(n_attn=1, n_ffn=1, T_mb=64, ffn_format="bf16")
    with pytest.raises(ValueError):
        AfdConfig(n_attn=1, n_ffn=1, T_mb=64, ffn_format="mx", inter=256)
    AfdConfig(n_attn=2, n_ffn=6, T_mb=256, ffn_format="mx")
