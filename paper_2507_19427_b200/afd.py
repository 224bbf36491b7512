"""Attention-FFN Disaggregation runtime inside one B200 box (config 5).

nA attention GPUs each own their decode requests (DP attention)
and run the attention-side layer + router; nF FFN GPUs each hold 48/nF routed
experts (expert parallel) and a share of the shared expert's tokens.  Per
layer and micro-batch (pipesim.cpp:155-237 models it):

  A: mfa_layer -> router/quant into its send buffer -> signal every F
  F: wait all A -> DMA-pull payloads (fp8 tokens, scales, top-k) -> moe_ffn(_mx)
     whose combine kernel stores each token's bf16 partial row straight into
     the owning attention GPU's receive buffer over NVLink -> signal every A
     (f2a="pull": local partial, the attention GPU DMA-pulls its rows)
  A: wait all F -> x = h_res + sum partials

n_micro micro-batches per attention GPU run on their own streams (ping-pong),
so the attention of one overlaps the exchange/FFN of the other.  All data
moves with copy-engine DMA over NVLink and stream-ordered flags
(csrc/exchange.cu): no SM is spent on communication and no host round trip
sits on the per-message path.  One process per GPU; torch.distributed is used
only to exchange IPC handles, for barriers and to reduce the timing.

The shard/layout helpers are pure Python and are exercised by the CPU suite
(tests/test_afd_cpu.py, gloo world size 2-3).
"""
from __future__ import annotations

from dataclasses import dataclass, field


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
    ffn_format: str = "fp8"   # "fp8": 1x128/128x128 fp32 scales; "mx": MXFP8 (UE8M0 per 32)
    f2a: str = "push"         # "push": the FFN combine writes into the attention GPUs' receive
                              # buffers over NVLink (fused); "pull": attention DMA-pulls
    layer_kind: str = "moe"   # "moe": routed experts (EP over FFN GPUs); "dense": the dense Step-3
                              # FFN (inter dense_inter) as intermediate slices, tensor-parallel over FFN GPUs
    dense_inter: int = 18432
    attn_chunk: int = 256     # requests per attention-layer call (its GEMM N limit); a larger
                              # T_mb runs the attention side in chunks and ships ONE payload,
                              # so the FFN tier streams its expert weights once per micro-batch

    def __post_init__(self):
        # validated identically on every rank before any buffer exchange: a rank
        # that failed mid-pipeline would leave its peers waiting on a flag
        if not 1 <= self.attn_chunk <= 256:
            raise ValueError(f"attn_chunk={self.attn_chunk}: the attention-side layer takes 1..256 requests per call")
        if not 1 <= self.T_mb <= 4096:
            raise ValueError(f"T_mb={self.T_mb}: expected 1..4096 requests per micro-batch")
        if self.f2a not in ("push", "pull"):
            raise ValueError(f"f2a={self.f2a!r}: expected 'push' or 'pull'")
        if self.ffn_format not in ("fp8", "mx"):
            raise ValueError(f"ffn_format={self.ffn_format!r}: expected 'fp8' or 'mx'")
        if self.ffn_format == "mx" and (self.hidden % 512 or self.inter % 512):
            raise ValueError("ffn_format='mx' needs hidden and inter to be multiples of 512")
        if self.layer_kind not in ("moe", "dense"):
            raise ValueError(f"layer_kind={self.layer_kind!r}: expected 'moe' or 'dense'")
        if self.layer_kind == "dense":
            if self.ffn_format != "mx":
                raise ValueError("layer_kind='dense' runs the MXFP8 dense FFN (ffn_format='mx')")
            if self.dense_inter % (self.dense_slices_total * 512):
                raise ValueError(f"dense_inter={self.dense_inter} is not a multiple of "
                                 f"{self.dense_slices_total} slices x 512")
        if self.n_attn < 1 or self.n_ffn < 1 or self.n_ffn > self.n_experts:
            raise ValueError("need at least one attention and one FFN GPU, n_ffn <= n_experts")

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


def shard(i: int, n: int, total: int) -> tuple[int, int]:
    """Contiguous split of `total` items over `n` owners (owner i's [lo, hi))."""
    return (i * total) // n, ((i + 1) * total) // n


def expert_shard(f: int, cfg: AfdConfig) -> tuple[int, int]:
    return shard(f, cfg.n_ffn, cfg.n_experts)


def shared_token_shard(f: int, cfg: AfdConfig) -> tuple[int, int]:
    return shard(f, cfg.n_ffn, cfg.T_ffn)


@dataclass
class PayloadLayout:
    """A->F message of one micro-batch, one contiguous buffer per attention GPU:
    e4m3 tokens | scales | int32 top-k ids | fp32 top-k weights.  The scale
    section is T*H/32 bytes in both formats (fp32 per 1x128 block, or one
    UE8M0 byte per 32 elements for MXFP8)."""

    T: int
    H: int
    k: int
    off: dict = field(default_factory=dict)
    nbytes: int = 0

    def __post_init__(self):
        o = 0
        for name, n in (("xq", self.T * self.H), ("xs", self.T * (self.H // 128) * 4), ("ids", self.T * self.k * 4),
                        ("wts", self.T * self.k * 4)):
            self.off[name] = o
            o += (n + 255) // 256 * 256
        self.nbytes = o

    def size(self, name: str) -> int:
        return {"xq": self.T * self.H, "xs": self.T * (self.H // 128) * 4, "ids": self.T * self.k * 4,
                "wts": self.T * self.k * 4}[name]


def wire_bytes(cfg: AfdConfig) -> dict:
    """Bytes crossing NVLink per layer per micro-batch (the moeplan.cpp:17-20
    accounting (1+2)*H*T plus the scale/top-k metadata)."""
    T = cfg.n_attn * cfg.T_mb
    lay = PayloadLayout(cfg.T_mb, cfg.hidden, cfg.top_k)
    a2f = cfg.n_ffn * cfg.n_attn * sum(lay.size(n) for n in ("xq", "xs", "ids", "wts"))
    f2a = cfg.n_ffn * T * cfg.hidden * 2
    return {"a2f": a2f, "f2a": f2a, "payload_a2f": cfg.n_ffn * T * cfg.hidden, "payload_f2a": f2a}


def flag_index(peer: int, mb: int, cfg: AfdConfig) -> int:
    """Slot of the flag that `peer` raises for micro-batch `mb` on the receiving GPU."""
    return peer * cfg.n_micro + mb


# ---------------------------------------------------------------- GPU runtime
class AfdRank:
    """One GPU of the AFD group.  Call setup() once (collective), then step()."""

    def __init__(self, ctxs, cfg: AfdConfig, rank: int, torch, dist, dev):
        """ctxs: one afdk Context per micro-batch stream (each owns its workspace)."""
        self.ctxs = ctxs
        self.ctx = ctxs[0]
        self.cfg, self.rank, self.torch, self.dist, self.dev = cfg, rank, torch, dist, dev
        self.role = cfg.role(rank)
        self.idx = rank if self.role == "attn" else rank - cfg.n_attn
        self.lay = PayloadLayout(cfg.T_mb, cfg.hidden, cfg.top_k)
        self.epoch = 0
        self.streams = [torch.cuda.Stream(device=dev) for _ in range(cfg.n_micro)]
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.flags = torch.zeros(256, dtype=torch.int32, device=dev)
        self.peer_flags = {}
        self.peer_bufs = {}
        self.peer_recv = {}

    # ---------------------------------------------------------------- setup
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
        """Deterministic e4m3 expert weights: expert e's tensors depend only on
        (seed, e), so every GPU materialises identical shards."""
        t, c = self.torch, self.cfg
        ids = list(range(lo, hi)) + ([c.n_experts] if with_shared else [])
        mx = c.ffn_format == "mx"
        w13, w2, s13, s2 = [], [], [], []
        for e in ids:
            g = t.Generator(device=self.dev).manual_seed(c.seed * 1000 + e + 1)

            def e4m3(shape):
                mag = t.randint(0x18, 0x40, shape, generator=g, dtype=t.int32, device=self.dev)
                sgn = t.randint(0, 2, shape, generator=g, dtype=t.int32, device=self.dev) * 0x80
                return (mag | sgn).to(t.uint8)

            w13.append(e4m3((2 * c.inter, c.hidden)))
            w2.append(e4m3((c.hidden, c.inter)))
            if mx:  # UE8M0 2^-7: |w| ~ 2^-6..2^-3 like the 1x128 recipe below
                s13.append(t.full((2 * c.inter, c.hidden // 32), 120, dtype=t.uint8, device=self.dev))
                s2.append(t.full((c.hidden, c.inter // 32), 120, dtype=t.uint8, device=self.dev))
            else:
                s13.append(t.full((2 * c.inter // 128, c.hidden // 128), 0.5 / c.hidden ** 0.5, device=self.dev))
                s2.append(t.full((c.hidden // 128, c.inter // 128), 0.5 / c.inter ** 0.5, device=self.dev))
        if mx:
            return {"n_experts": c.n_experts, "w13": t.stack(w13), "w2": t.stack(w2), "sf13": t.stack(s13),
                    "sf2": t.stack(s2)}
        return {"n_experts": c.n_experts, "w13": t.stack(w13), "w2": t.stack(w2), "s13": t.stack(s13),
                "s2": t.stack(s2)}

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

    def setup(self):
        """alloc() on every rank, agree that all succeeded, then connect().
        A rank that failed to allocate makes EVERY rank raise here, before any
        buffer exchange, instead of leaving its peers waiting on a flag."""
        err = None
        try:
            mine = self.alloc()
        except Exception as e:  # noqa: BLE001 - reported on all ranks below
            err, mine = e, None
        on_gloo = self.dist.get_backend() == "gloo"  # CPU rendezvous (tests, oversubscribed checks)
        ok = self.torch.tensor([0 if err else 1], dtype=self.torch.int32, device="cpu" if on_gloo else self.dev)
        self.dist.all_reduce(ok, op=self.dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            raise RuntimeError(f"AFD setup failed on some rank (this rank: {err!r})")
        self.connect(mine)

    def alloc(self) -> dict:
        """Local allocations and IPC handle export (no collectives)."""
        t, c, dev = self.torch, self.cfg, self.dev
        g = t.Generator().manual_seed(c.seed)
        if self.role == "attn":
            self.w = self._weights_attn(g)
            pages = (c.ctx_len + c.page - 1) // c.page
            gx = t.Generator().manual_seed(c.seed + 7 + self.idx)
            self.x0 = [t.randn(c.T_mb, c.hidden, generator=gx).to(t.bfloat16).to(dev) for _ in range(c.n_micro)]
            self.x = [x.clone() for x in self.x0]
            self.h_res = [t.empty_like(x) for x in self.x0]
            self.h_norm = [t.empty_like(x) for x in self.x0]
            self.send = [t.empty(self.lay.nbytes, dtype=t.uint8, device=dev) for _ in range(c.n_micro)]
            self.recv_part = [t.empty(c.n_ffn, c.T_mb, c.hidden, dtype=t.bfloat16, device=dev)
                              for _ in range(c.n_micro)]
            self.part_ptrs = [t.tensor([rp[f].data_ptr() for f in range(c.n_ffn)], dtype=t.int64, device=dev)
                              for rp in self.recv_part]
            self.kv = []
            for _ in range(c.layers):
                per_mb = []
                for _ in range(c.n_micro):
                    n_pages = c.T_mb * pages
                    k = t.empty(n_pages, c.page, c.head_dim, dtype=t.bfloat16, device=dev).normal_()
                    v = t.empty(n_pages, c.page, c.head_dim, dtype=t.bfloat16, device=dev).normal_()
                    bt = t.randperm(n_pages, device=dev).to(t.int32).view(c.T_mb, pages).contiguous()
                    per_mb.append((k, v, bt))
                self.kv.append(per_mb)
            self.seq_lens = t.full((c.T_mb,), c.ctx_len, dtype=t.int32, device=dev)
            mine = {"flags": self.ctx.ipc_handle(self.flags),
                    "send": [self.ctx.ipc_handle(b) for b in self.send],
                    "recv": [self.ctx.ipc_handle(b) for b in self.recv_part]}
        else:
            lo, hi = expert_shard(self.idx, c)
            if c.layer_kind == "dense":
                S = c.dense_slices_per_gpu
                self.moe_w = self.dense_weights(self.idx * S, (self.idx + 1) * S)
            else:
                self.moe_w = self.expert_weights(lo, hi)
            self.expert_lo, self.expert_hi = lo, hi
            self.shared = shared_token_shard(self.idx, c)
            Tf = c.T_ffn
            xs_shape, xs_dtype = ((Tf, c.hidden // 32), t.uint8) if c.ffn_format == "mx" else \
                ((Tf, c.hidden // 128), t.float32)
            self.rx = [{"xq": t.empty(Tf, c.hidden, dtype=t.uint8, device=dev),
                        "xs": t.empty(*xs_shape, dtype=xs_dtype, device=dev),
                        "ids": t.empty(Tf, c.top_k, dtype=t.int32, device=dev),
                        "wts": t.empty(Tf, c.top_k, dtype=t.float32, device=dev)} for _ in range(c.n_micro)]
            self.out = [t.empty(Tf, c.hidden, dtype=t.bfloat16, device=dev) for _ in range(c.n_micro)]
            self.copied = [t.cuda.Event() for _ in range(c.n_micro)]
            mine = {"flags": self.ctx.ipc_handle(self.flags), "out": [self.ctx.ipc_handle(b) for b in self.out]}
        return mine

    def connect(self, mine: dict) -> None:
        """Collective: exchange IPC handles and open the peers' buffers."""
        t, c, dev = self.torch, self.cfg, self.dev
        allh = [None] * c.world
        self.dist.all_gather_object(allh, (self.rank, mine))
        for r, h in allh:
            if r == self.rank:
                continue
            peer_role = c.role(r)
            if peer_role == self.role:
                continue  # attention GPUs never talk to each other, nor FFN GPUs
            self.peer_flags[r] = self.ctx.ipc_open(h["flags"])
            key = "send" if peer_role == "attn" else "out"
            self.peer_bufs[r] = [self.ctx.ipc_open(x) for x in h[key]]
            if peer_role == "attn" and c.f2a == "push":
                self.peer_recv[r] = [self.ctx.ipc_open(x) for x in h["recv"]]
        if self.role == "ffn" and c.f2a == "push":
            # my slot f of every attention GPU's [n_ffn, T_mb, H] receive buffer
            slot = self.idx * c.T_mb * c.hidden * 2
            self.dst = [t.tensor([self.peer_recv[a][mb] + slot for a in range(c.n_attn)], dtype=t.int64,
                                 device=dev) for mb in range(c.n_micro)]
        t.cuda.synchronize()
        self.dist.barrier()

    # ----------------------------------------------------------------- step
    def _attn_layer(self, layer, mb, seq):
        c, ctx, t = self.cfg, self.ctxs[mb], self.torch
        st = self.streams[mb]
        sp = st.cuda_stream
        k, v, bt = self.kv[layer][mb]
        for c0 in range(0, c.T_mb, c.attn_chunk):
            c1 = min(c.T_mb, c0 + c.attn_chunk)
            ctx.mfa_layer(self.w, self.x[mb][c0:c1], k, v, bt[c0:c1], self.seq_lens[c0:c1], self.h_res[mb][c0:c1],
                          self.h_norm[mb][c0:c1], stream=sp)
        buf, L = self.send[mb], self.lay
        view = lambda name, shape, dtype: buf[L.off[name]:L.off[name] + L.size(name)].view(dtype).view(*shape)
        if c.ffn_format == "mx":
            if c.layer_kind == "moe":
                ctx.router_topk(self.h_norm[mb], self.w["gate"], c.top_k, view("ids", (c.T_mb, c.top_k), t.int32),
                                view("wts", (c.T_mb, c.top_k), t.float32), stream=sp)
            ctx.quant_mx(self.h_norm[mb], view("xq", (c.T_mb, c.hidden), t.uint8),
                         view("xs", (c.T_mb, c.hidden // 32), t.uint8), stream=sp)
        else:
            ctx.router_topk(self.h_norm[mb], self.w["gate"], c.top_k, view("ids", (c.T_mb, c.top_k), t.int32),
                            view("wts", (c.T_mb, c.top_k), t.float32), xq=view("xq", (c.T_mb, c.hidden), t.uint8),
                            xs=view("xs", (c.T_mb, c.hidden // 128), t.float32), stream=sp)
        for f in range(c.n_ffn):
            r = c.n_attn + f
            ctx.signal(self.peer_flags[r] + 4 * flag_index(self.idx, mb, c), seq, stream=sp)
        # F -> A: pull this GPU's rows of every FFN partial, then residual + EP reduction
        row_bytes = c.T_mb * c.hidden * 2
        for f in range(c.n_ffn):
            r = c.n_attn + f
            ctx.wait(self.flags.data_ptr() + 4 * flag_index(f, mb, c), seq, stream=sp)
            if c.f2a == "pull":
                ctx.copy(self.recv_part[mb][f].data_ptr(), self.peer_bufs[r][mb] + self.idx * row_bytes, row_bytes,
                         stream=sp)
        ctx.add_partials(self.h_res[mb], self.part_ptrs[mb], c.n_ffn, self.x[mb], stream=sp)

    def _ffn_layer(self, mb, seq):
        c, ctx, t = self.cfg, self.ctx, self.torch
        cs = self.copy_stream.cuda_stream
        rx, L = self.rx[mb], self.lay
        for a in range(c.n_attn):
            ctx.wait(self.flags.data_ptr() + 4 * flag_index(a, mb, c), seq, stream=cs)
            src = self.peer_bufs[a][mb]
            for name in ("xq", "xs", "ids", "wts"):
                n = L.size(name)
                ctx.copy(rx[name].data_ptr() + a * n, src + L.off[name], n, stream=cs)
        self.copied[mb].record(self.copy_stream)
        st = self.streams[0]
        st.wait_event(self.copied[mb])
        scatter = (self.dst[mb], c.T_mb) if c.f2a == "push" else None
        if c.layer_kind == "dense":  # this GPU's slices of the dense FFN: a tensor-parallel partial
            ctx.dense_ffn_mx(self.moe_w, rx["xq"], rx["xs"], self.out[mb], stream=st.cuda_stream, scatter=scatter)
        else:
            ffn = ctx.moe_ffn_mx if c.ffn_format == "mx" else ctx.moe_ffn
            ffn(self.moe_w, rx["xq"], rx["xs"], rx["ids"], rx["wts"], self.out[mb], expert_lo=self.expert_lo,
                expert_hi=self.expert_hi, shared=self.shared, stream=st.cuda_stream, scatter=scatter)
        for a in range(c.n_attn):
            ctx.signal(self.peer_flags[a] + 4 * flag_index(self.idx, mb, c), seq, stream=st.cuda_stream)

    def step(self):
        """One decode step over cfg.layers layers for every micro-batch (enqueue only)."""
        c = self.cfg
        for layer in range(c.layers):
            self.epoch += 1
            for mb in range(c.n_micro):
                if self.role == "attn":
                    self._attn_layer(layer, mb, self.epoch)
                else:
                    self._ffn_layer(mb, self.epoch)

    def reset_inputs(self):
        if self.role == "attn":
            for mb in range(self.cfg.n_micro):
                self.x[mb].copy_(self.x0[mb])

    def streams_all(self):
        return self.streams + [self.copy_stream]

    def close(self):
        for r, bufs in self.peer_recv.items():
            for p in bufs:
                self.ctx.ipc_close(p)
        self.peer_recv = {}
        for r, p in self.peer_flags.items():
            self.ctx.ipc_close(p)
        for r, bufs in self.peer_bufs.items():
            for p in bufs:
                self.ctx.ipc_close(p)
        self.peer_flags, self.peer_bufs = {}, {}
