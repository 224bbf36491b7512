"""Attention-FFN Disaggregation inside one B200 box (config 5): Python binding
of the C++ AFD runtime (csrc/afd_runtime.cu, include/afdk.h afdk_afd_*).

nA attention GPUs each own their decode requests (DP attention)
and run the attention-side layer + router; nF FFN GPUs each hold 48/nF routed
experts (expert parallel) and a share of the shared expert's tokens.  The
per-layer schedule (pipesim.cpp:155-237 models it) — op
list, flags, transfers, streams and peer mappings — lives in the C++ runtime
(afdk_afd_plan / afdk_afd_attn_layer / afdk_afd_ffn_layer).  This module
holds only:

  * AfdConfig: the validated configuration (mirrored into afdk_afd_cfg);
  * the shard arithmetic and wire accounting the bench and tests report;
  * AfdRank: synthetic weights / KV caches for one rank (caller-owned data
    in the C-ABI's ownership model) and the rendezvous callback that hands
    the runtime's 72-byte IPC handles to torch.distributed.

One process per GPU; torch.distributed only exchanges handles, runs
barriers and reduces timings.
"""
from __future__ import annotations

import ctypes
from ctypes import c_int, c_void_p
from dataclasses import dataclass

from . import afdk as _k

FFN_FORMATS = {"fp8": 0, "mx": 1, "bf16": 2}
LAYER_KINDS = {"moe": 0, "dense": 1}
F2A = {"push": 0, "pull": 1, "nvls": 2}
OP_NAMES = {0: "ATTN", 1: "SIGNAL", 2: "WAIT", 3: "PULL", 4: "REDUCE", 5: "JOIN", 6: "FFN"}
BUF_SEND, BUF_RECV, BUF_RX, BUF_OUT, BUF_H_RES, BUF_H_NORM = 0, 1, 2, 3, 4, 5


@dataclass
class AfdConfig:
    n_attn: int
    n_ffn: int
    T_mb: int                 # decode requests (tokens) per micro-batch per attention GPU
    n_micro: int = 2          # ping-pong
    layers: int = 1           # layers per step (distinct KV caches, shared weights)
    hidden: int = 7168
    q_lora: int = 2048
    n_heads: int = 64
    head_dim: int = 256
    page: int = 64
    ctx_len: int = 4096
    n_experts: int = 48
    top_k: int = 3
    inter: int = 5120
    seed: int = 0
    ffn_format: str = "fp8"   # "fp8": 1x128/128x128 fp32 scales; "mx": MXFP8; "bf16": 16-bit experts
    f2a: str = "push"         # "push": the FFN combine writes into the attention GPUs' receive
                              # buffers over NVLink (fused); "pull": attention DMA-pulls;
                              # "nvls": partials reduced in the NVSwitch (multimem.ld_reduce)
    layer_kind: str = "moe"   # "moe": routed experts (EP over FFN GPUs); "dense": the dense Step-3
                              # FFN (inter dense_inter) as intermediate slices, tensor-parallel
    dense_inter: int = 18432
    attn_chunk: int = 512     # requests per attention-layer call (its GEMM N limit); a larger
                              # T_mb runs the attention side in chunks and ships ONE payload
    kv: str = "bf16"          # attention KV cache: "bf16" or "e4m3" (per-tensor scales)
    attn_o_mx: bool = False   # o_proj as an MXFP8 GEMM (afdk_mfa_weights.w_o_mx / w_o_sf; T_mb <= 384)
    attn_qup_mx: bool = False  # q_up likewise (afdk_mfa_weights.w_q_up_mx / w_q_up_sf; T_mb <= 384)

    def __post_init__(self):
        # validated identically on every rank before any buffer exchange
        if self.ffn_format not in FFN_FORMATS:
            raise ValueError(f"ffn_format={self.ffn_format!r}: expected one of {sorted(FFN_FORMATS)}")
        if self.layer_kind not in LAYER_KINDS:
            raise ValueError(f"layer_kind={self.layer_kind!r}: expected 'moe' or 'dense'")
        if self.f2a not in F2A:
            raise ValueError(f"f2a={self.f2a!r}: expected one of {sorted(F2A)}")
        if self.kv not in ("bf16", "e4m3"):
            raise ValueError(f"kv={self.kv!r}: expected 'bf16' or 'e4m3'")
        if _k.load().afdk_afd_check_cfg(ctypes.byref(self.c_cfg())) != 0:
            raise ValueError(_k.load().afdk_last_error().decode())

    @property
    def dense_slices_per_gpu(self) -> int:
        return max(1, 4 // self.n_ffn)

    @property
    def dense_slices_total(self) -> int:
        return self.n_ffn * self.dense_slices_per_gpu

    @property
    def world(self) -> int:
        return self.n_attn + self.n_ffn

    def role(self, rank: int) -> str:
        return "attn" if rank < self.n_attn else "ffn"

    @property
    def T_ffn(self) -> int:
        """tokens one FFN GPU sees per micro-batch (broadcast from every attention GPU)"""
        return self.n_attn * self.T_mb

    def c_cfg(self) -> "AfdCfg":
        return AfdCfg(self.n_attn, self.n_ffn, self.n_micro, self.T_mb, self.hidden, self.top_k, self.n_experts,
                      self.inter, self.dense_inter, self.dense_slices_per_gpu, FFN_FORMATS[self.ffn_format],
                      LAYER_KINDS[self.layer_kind], F2A[self.f2a], self.attn_chunk)


AfdCfg, AfdOp, AfdLayout, AfdAttnMb, AfdFfnWeights, ALLGATHER = (
    _k.AfdCfg, _k.AfdOp, _k.AfdLayout, _k.AfdAttnMb, _k.AfdFfnWeights, _k.ALLGATHER)


def layout(cfg: AfdConfig) -> AfdLayout:
    """Payload / receive-buffer layout the runtime uses (afdk_afd_get_layout)."""
    L = AfdLayout()
    _k.check(_k.load().afdk_afd_get_layout(ctypes.byref(cfg.c_cfg()), ctypes.byref(L)))
    return L


def plan(cfg: AfdConfig, rank: int, seq: int) -> list[AfdOp]:
    """The op list the runtime executes for one layer on `rank` (host only)."""
    lib, c = _k.load(), cfg.c_cfg()
    n = c_int(0)
    _k.check(lib.afdk_afd_plan(ctypes.byref(c), rank, seq, None, 0, ctypes.byref(n)))
    ops = (AfdOp * n.value)()
    _k.check(lib.afdk_afd_plan(ctypes.byref(c), rank, seq, ctypes.cast(ops, c_void_p), n.value, ctypes.byref(n)))
    return list(ops)


class PayloadLayout:
    """Python view of one A->F message's sections (xq, xs, ids, wts)."""

    NAMES = ("xq", "xs", "ids", "wts")

    def __init__(self, cfg: AfdConfig):
        L = layout(cfg)
        self.off = {n: L.off[i] for i, n in enumerate(self.NAMES)}
        self._size = {n: L.size[i] for i, n in enumerate(self.NAMES)}
        self.rx_off = {n: L.rx_off[i] for i, n in enumerate(self.NAMES)}
        self.nbytes, self.rx_total, self.part_bytes = L.total, L.rx_total, L.part_bytes

    def size(self, name: str) -> int:
        return self._size[name]


def shard(i: int, n: int, total: int) -> tuple[int, int]:
    """Contiguous split of `total` items over `n` owners (owner i's [lo, hi))."""
    return (i * total) // n, ((i + 1) * total) // n


def expert_shard(f: int, cfg: AfdConfig) -> tuple[int, int]:
    return shard(f, cfg.n_ffn, cfg.n_experts)


def shared_token_shard(f: int, cfg: AfdConfig) -> tuple[int, int]:
    return shard(f, cfg.n_ffn, cfg.T_ffn)


def wire_bytes(cfg: AfdConfig) -> dict:
    """Bytes crossing NVLink per layer per micro-batch (the moeplan.cpp:17-20
    accounting (dispatch + combine)*H*T plus the scale/top-k metadata,
    PAPER.md:655; dispatch = 1 byte for the FP8 formats, 2 for bf16)."""
    T = cfg.n_attn * cfg.T_mb
    L = PayloadLayout(cfg)
    a2f = cfg.n_ffn * cfg.n_attn * sum(L.size(n) for n in PayloadLayout.NAMES)
    f2a = cfg.n_ffn * T * cfg.hidden * 2
    disp = 2 if cfg.ffn_format == "bf16" else 1
    return {"a2f": a2f, "f2a": f2a, "payload_a2f": cfg.n_ffn * T * cfg.hidden * disp, "payload_f2a": f2a}


def flag_index(peer: int, mb: int, cfg: AfdConfig) -> int:
    """Slot of the flag that `peer` raises for micro-batch `mb` on the receiving GPU."""
    return peer * cfg.n_micro + mb


# ---------------------------------------------------------------- GPU rank
class AfdRank:
    """One GPU of the AFD group: synthetic caller-owned data + the C++ runtime.
    Call setup() once (collective), then step()."""

    def __init__(self, ctxs, cfg: AfdConfig, rank: int, torch, dist, dev):
        """ctxs: one afdk Context per micro-batch stream (each owns its workspace)."""
        self.ctxs = ctxs
        self.ctx = ctxs[0]
        self.cfg, self.rank, self.torch, self.dist, self.dev = cfg, rank, torch, dist, dev
        self.role = cfg.role(rank)
        self.idx = rank if self.role == "attn" else rank - cfg.n_attn
        self.lay = PayloadLayout(cfg)
        self.handle = None

    # ---------------------------------------------------------------- data
    def _weights_attn(self, g):
        t, c = self.torch, self.cfg
        bf = lambda x: x.to(t.bfloat16).to(self.dev)
        return {"in_norm": bf(1 + 0.1 * t.randn(c.hidden, generator=g)),
                "qkv": bf(t.randn(c.q_lora + 2 * c.head_dim, c.hidden, generator=g) / c.hidden ** 0.5),
                "q_norm": bf(1 + 0.1 * t.randn(c.q_lora, generator=g)),
                "q_up": bf(t.randn(c.n_heads * c.head_dim, c.q_lora, generator=g) / c.q_lora ** 0.5),
                "o": bf(t.randn(c.hidden, c.n_heads * c.head_dim, generator=g) / (c.n_heads * c.head_dim) ** 0.5),
                "post_norm": bf(1 + 0.1 * t.randn(c.hidden, generator=g)),
                "gate": bf(t.randn(c.n_experts, c.hidden, generator=g) / c.hidden ** 0.5)}

    def expert_weights(self, lo, hi, with_shared=True):
        """Deterministic expert weights in cfg.ffn_format: expert e's tensors
        depend only on (seed, e), so every GPU materialises identical shards."""
        t, c = self.torch, self.cfg
        ids = list(range(lo, hi)) + ([c.n_experts] if with_shared else [])
        w13, w2, s13, s2 = [], [], [], []
        for e in ids:
            g = t.Generator(device=self.dev).manual_seed(c.seed * 1000 + e + 1)
            if c.ffn_format == "bf16":
                w13.append((t.randn(2 * c.inter, c.hidden, generator=g, device=self.dev) / c.hidden ** 0.5)
                           .to(t.bfloat16))
                w2.append((t.randn(c.hidden, c.inter, generator=g, device=self.dev) / c.inter ** 0.5).to(t.bfloat16))
                continue

            def e4m3(shape):
                mag = t.randint(0x18, 0x40, shape, generator=g, dtype=t.int32, device=self.dev)
                sgn = t.randint(0, 2, shape, generator=g, dtype=t.int32, device=self.dev) * 0x80
                return (mag | sgn).to(t.uint8)

            w13.append(e4m3((2 * c.inter, c.hidden)))
            w2.append(e4m3((c.hidden, c.inter)))
            if c.ffn_format == "mx":  # UE8M0 2^-7: |w| ~ 2^-6..2^-3 like the 1x128 recipe below
                s13.append(t.full((2 * c.inter, c.hidden // 32), 120, dtype=t.uint8, device=self.dev))
                s2.append(t.full((c.hidden, c.inter // 32), 120, dtype=t.uint8, device=self.dev))
            else:
                s13.append(t.full((2 * c.inter // 128, c.hidden // 128), 0.5 / c.hidden ** 0.5, device=self.dev))
                s2.append(t.full((c.hidden // 128, c.inter // 128), 0.5 / c.inter ** 0.5, device=self.dev))
        w = {"n_experts": c.n_experts, "w13": t.stack(w13), "w2": t.stack(w2)}
        if c.ffn_format == "mx":
            w.update(sf13=t.stack(s13), sf2=t.stack(s2))
        elif c.ffn_format == "fp8":
            w.update(s13=t.stack(s13), s2=t.stack(s2))
        return w

    def dense_weights(self, lo, hi):
        """MXFP8 slices [lo, hi) of the dense FFN (slice layout of afdk_dense_ffn_mx);
        slice j's tensors depend only on (seed, j)."""
        t, c = self.torch, self.cfg
        Is = c.dense_inter // c.dense_slices_total
        w13, w2 = [], []
        for j in range(lo, hi):
            g = t.Generator(device=self.dev).manual_seed(c.seed * 1000 + 500 + j)

            def e4m3(shape):
                mag = t.randint(0x18, 0x40, shape, generator=g, dtype=t.int32, device=self.dev)
                sgn = t.randint(0, 2, shape, generator=g, dtype=t.int32, device=self.dev) * 0x80
                return (mag | sgn).to(t.uint8)

            w13.append(e4m3((2 * Is, c.hidden)))
            w2.append(e4m3((c.hidden, Is)))
        n = hi - lo
        return {"w13": t.stack(w13), "w2": t.stack(w2),
                "sf13": t.full((n, 2 * Is, c.hidden // 32), 120, dtype=t.uint8, device=self.dev),
                "sf2": t.full((n, c.hidden, Is // 32), 120, dtype=t.uint8, device=self.dev)}

    def alloc(self) -> None:
        """Caller-owned data of this rank (weights, KV caches, activations)."""
        t, c, dev = self.torch, self.cfg, self.dev
        g = t.Generator().manual_seed(c.seed)
        if self.role == "attn":
            self.w = self._weights_attn(g)
            pages = (c.ctx_len + c.page - 1) // c.page
            gx = t.Generator().manual_seed(c.seed + 7 + self.idx)
            self.x0 = [t.randn(c.T_mb, c.hidden, generator=gx).to(t.bfloat16).to(dev) for _ in range(c.n_micro)]
            self.x = [x.clone() for x in self.x0]
            self.kv = []
            for _ in range(c.layers):
                per_mb = []
                for _ in range(c.n_micro):
                    n_pages = c.T_mb * pages
                    k = t.empty(n_pages, c.page, c.head_dim, dtype=t.bfloat16, device=dev).normal_()
                    v = t.empty(n_pages, c.page, c.head_dim, dtype=t.bfloat16, device=dev).normal_()
                    if c.kv == "e4m3":  # per-tensor scales (amax / 448)
                        ks, vs = float(k.abs().max()) / 448.0, float(v.abs().max()) / 448.0
                        k = (k.float() / ks).to(t.float8_e4m3fn).view(t.uint8)
                        v = (v.float() / vs).to(t.float8_e4m3fn).view(t.uint8)
                    else:
                        ks = vs = 0.0
                    bt = t.randperm(n_pages, device=dev).to(t.int32).view(c.T_mb, pages).contiguous()
                    per_mb.append((k, v, bt, ks, vs))
                self.kv.append(per_mb)
            self.seq_lens = t.full((c.T_mb,), c.ctx_len, dtype=t.int32, device=dev)
            w = self.w
            if c.attn_o_mx:  # MXFP8 o_proj weights (afdk_quant_mx's format)
                w["o_mx"] = t.empty(w["o"].shape, dtype=t.uint8, device=dev)
                w["o_sf"] = t.empty(w["o"].shape[0], w["o"].shape[1] // 32, dtype=t.uint8, device=dev)
                self.ctx.quant_mx(w["o"], w["o_mx"], w["o_sf"])
            if c.attn_qup_mx:  # MXFP8 q_up weights
                w["q_up_mx"] = t.empty(w["q_up"].shape, dtype=t.uint8, device=dev)
                w["q_up_sf"] = t.empty(w["q_up"].shape[0], w["q_up"].shape[1] // 32, dtype=t.uint8, device=dev)
                self.ctx.quant_mx(w["q_up"], w["q_up_mx"], w["q_up_sf"])
            self.c_w = _k.MfaWeights(c.hidden, c.q_lora, c.n_heads, c.head_dim, _k.ptr(w["in_norm"]), _k.ptr(w["qkv"]),
                                     _k.ptr(w["q_norm"]), _k.ptr(w["q_up"]), _k.ptr(w["o"]), _k.ptr(w["post_norm"]),
                                     1e-5, 5e5, c.head_dim ** -0.5,
                                     _k.ptr(w["o_mx"]) if c.attn_o_mx else None,
                                     _k.ptr(w["o_sf"]) if c.attn_o_mx else None,
                                     _k.ptr(w["q_up_mx"]) if c.attn_qup_mx else None,
                                     _k.ptr(w["q_up_sf"]) if c.attn_qup_mx else None)
            self.c_mbs = []
            for layer in range(c.layers):
                arr = (AfdAttnMb * c.n_micro)()
                for mb in range(c.n_micro):
                    k, v, bt, ks, vs = self.kv[layer][mb]
                    arr[mb] = AfdAttnMb(_k.ptr(self.x[mb]), _k.ptr(k), _k.ptr(v), k.shape[0], c.page, bt.shape[1],
                                        _k.ptr(bt), _k.ptr(self.seq_lens), ks, vs)
                self.c_mbs.append(arr)
        else:
            lo, hi = expert_shard(self.idx, c)
            if c.layer_kind == "dense":
                S = c.dense_slices_per_gpu
                self.moe_w = self.dense_weights(self.idx * S, (self.idx + 1) * S)
            else:
                self.moe_w = self.expert_weights(lo, hi)
            self.expert_lo, self.expert_hi = lo, hi
            self.shared = shared_token_shard(self.idx, c)
            mw = self.moe_w
            s13 = mw.get("sf13", mw.get("s13"))
            s2 = mw.get("sf2", mw.get("s2"))
            self.c_ffn_w = AfdFfnWeights(_k.ptr(mw["w13"]), _k.ptr(s13), _k.ptr(mw["w2"]), _k.ptr(s2))

    def _allgather(self, user, mine, nbytes, out):
        """Rendezvous callback of afdk_afd_create (torch.distributed transport)."""
        try:
            blob = ctypes.string_at(mine, nbytes)
            got = [None] * self.cfg.world
            self.dist.all_gather_object(got, blob)
            for r, b in enumerate(got):
                ctypes.memmove(out + r * nbytes, b, nbytes)
            return 0
        except Exception:  # noqa: BLE001 - reported as the runtime's create failure
            return 1

    def setup(self):
        """alloc() on every rank, agree that all succeeded, then create the
        runtime (which allocates the exchange buffers, agrees again and maps
        the peers).  A failing rank makes EVERY rank raise, before any buffer
        exchange, instead of leaving its peers waiting on a flag."""
        err = None
        try:
            self.alloc()
        except Exception as e:  # noqa: BLE001 - reported on all ranks below
            err = e
        on_gloo = self.dist.get_backend() == "gloo"
        ok = self.torch.tensor([0 if err else 1], dtype=self.torch.int32, device="cpu" if on_gloo else self.dev)
        self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            raise RuntimeError(f"AFD setup failed on some rank (this rank: {err!r})")
        self.torch.cuda.synchronize(self.dev)
        lib = _k.load()
        ctx_arr = (c_void_p * self.cfg.n_micro)(*[c.handle for c in self.ctxs])
        self._cb = ALLGATHER(self._allgather)  # keep alive while the runtime exists
        h = c_void_p()
        _k.check(lib.afdk_afd_create(ctx_arr, ctypes.byref(self.cfg.c_cfg()), self.rank, self._cb, None,
                                     ctypes.byref(h)))
        self.handle = h
        self._streams = [self.torch.cuda.ExternalStream(lib.afdk_afd_stream(h, i), device=self.dev)
                         for i in range(self.cfg.n_micro + 1)]

    # ----------------------------------------------------------------- step
    def step(self, after_layer=None):
        """One decode step over cfg.layers layers for every micro-batch (enqueue only).
        after_layer(layer) runs after each layer is enqueued (e.g. to enqueue a
        snapshot of x on the runtime's micro-batch streams)."""
        lib = _k.load()
        for layer in range(self.cfg.layers):
            if self.role == "attn":
                _k.check(lib.afdk_afd_attn_layer(self.handle, ctypes.byref(self.c_w), _k.ptr(self.w["gate"]),
                                                 self.c_mbs[layer]))
            else:
                _k.check(lib.afdk_afd_ffn_layer(self.handle, ctypes.byref(self.c_ffn_w)))
            if after_layer is not None:
                after_layer(layer)

    def buffer(self, which: int, mb: int) -> int:
        return _k.load().afdk_afd_buffer(self.handle, which, mb) or 0

    def reset_inputs(self):
        if self.role == "attn":
            for mb in range(self.cfg.n_micro):
                self.x[mb].copy_(self.x0[mb])

    def streams_all(self):
        return list(self._streams)

    def trace_start(self):
        """Record CUDA events around every resource-occupying op from now on."""
        _k.check(_k.load().afdk_afd_trace_start(self.handle))

    def trace_csv(self) -> str:
        """This rank's measured trace (trace_csv schema), host-blocking; stops tracing."""
        lib, n = _k.load(), ctypes.c_size_t(0)
        _k.check(lib.afdk_afd_trace_csv(self.handle, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        _k.check(lib.afdk_afd_trace_csv(self.handle, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def sync(self):
        _k.check(_k.load().afdk_afd_sync(self.handle))

    def close(self):
        if self.handle is not None:
            _k.load().afdk_afd_destroy(self.handle)
            self.handle = None
