"""CPU executor of the C++ AFD runtime's op list (TEST INFRASTRUCTURE).

tests/test_afd_cpu.py runs one process per rank over torch.distributed gloo;
every process executes, op by op, the list the product's runtime executes on
the GPU — afdk_afd_plan() from libafdk.so (csrc/afd_runtime.cu), no GPU
needed — with the runtime's own payload layout (afdk_afd_get_layout).  Only
the memory model and the compute are doubles:

  * memory: each rank owns byte buffers shaped like the runtime's (send,
    recv, rx, out).  A SIGNAL carries the sequence number AND a snapshot of
    the buffer the peer may read after waiting on it (release semantics of
    the flag write: the attention payload for A->F; for F->A, the rows this
    FFN rank stores into the peer in push mode or exposes for the peer's
    pull); a WAIT receives messages from its peer until the flag reaches the
    value; a PULL copies from the snapshot.  Message order per peer is the
    GPU's stream order.
  * compute: ATTN / FFN / REDUCE use the CPU oracle (router top-k, FP8 1x128
    / MXFP8 / bf16 dispatch formats and expert FFNs) at tiny dims; the
    attention layer itself is a cheap deterministic stand-in (h_res = x +
    0.5 tanh(x), h_norm = RMSNorm(h_res)), since the protocol, not the
    attention numerics, is under test here.

reference_layers() recomputes the same layers in one process without any
protocol; the distributed result must be bit-identical.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc
from paper_2507_19427_b200 import afd

SEND, RECV, RX, OUT = afd.BUF_SEND, afd.BUF_RECV, afd.BUF_RX, afd.BUF_OUT


# ---------------------------------------------------------- compute doubles
def model(cfg, seed=3):
    rng = np.random.default_rng(seed)
    H, I, E = cfg.hidden, cfg.inter, cfg.n_experts
    m = {"norm": (1 + 0.1 * rng.standard_normal(H)).astype(np.float32),
         "gate": (rng.standard_normal((E, H)) / np.sqrt(H)).astype(np.float32)}
    w13 = (rng.standard_normal((E + 1, 2 * I, H)) / np.sqrt(H)).astype(np.float32)
    w2 = (rng.standard_normal((E + 1, H, I)) / np.sqrt(I)).astype(np.float32)
    if cfg.ffn_format == "fp8":
        m["w"] = [orc.quant_fp8_tile(w13[e]) + orc.quant_fp8_tile(w2[e]) for e in range(E + 1)]
    elif cfg.ffn_format == "mx":
        m["w"] = [orc.quant_mx(w13[e]) + orc.quant_mx(w2[e]) for e in range(E + 1)]
    else:
        m["w"] = [(orc.bf16_round(w13[e]), orc.bf16_round(w2[e])) for e in range(E + 1)]
    return m


def attn_double(m, x):
    h_res = orc.bf16_round(x + 0.5 * np.tanh(x))
    return h_res, orc.rmsnorm(h_res, m["norm"], round_bf16=True)


def dispatch(cfg, m, h_norm):
    """(xq bytes, xs bytes, ids, wts) of the payload in cfg.ffn_format."""
    ids, wts = orc.router_topk(h_norm @ m["gate"].T, cfg.top_k)
    if cfg.ffn_format == "fp8":
        xq, xs = orc.quant_fp8_rowblock(h_norm)
    elif cfg.ffn_format == "mx":
        xq, xs = orc.quant_mx(h_norm)
    else:
        xq, xs = orc.bf16_bits(h_norm), np.zeros(0, np.uint8)
    return xq, xs, ids, wts


def expert(cfg, m, e, xq, xs):
    if cfg.ffn_format == "fp8":
        q13, s13, q2, s2 = m["w"][e]
        return orc.expert_ffn_fp8(xq, xs, q13, s13, q2, s2)
    if cfg.ffn_format == "mx":
        q13, s13, q2, s2 = m["w"][e]
        return orc.expert_ffn_mx(xq, xs, q13, s13, q2, s2)
    w13, w2 = m["w"][e]
    return orc.expert_ffn_f32(orc.bf16_from_bits(xq), w13, w2, round_bf16=True)


def ffn_partial(cfg, m, f, xq, xs, ids, wts):
    """FFN rank f's bf16 partial over all T_ffn tokens: its routed experts +
    its share of the shared expert (afdk_afd_ffn_layer's shard rule)."""
    lo, hi = afd.expert_shard(f, cfg)
    slo, shi = afd.shared_token_shard(f, cfg)
    T = ids.shape[0]
    acc = np.zeros((T, cfg.hidden), np.float64)
    for e in range(lo, hi):
        hit = ids == e
        rows = np.nonzero(hit.any(axis=1))[0]
        if len(rows):
            y = expert(cfg, m, e, xq[rows], xs[rows] if xs.size else xs)
            acc[rows] += wts[rows][hit[rows]][:, None].astype(np.float64) * y
    if shi > slo:
        r = np.arange(slo, shi)
        acc[r] += expert(cfg, m, cfg.n_experts, xq[r], xs[r] if xs.size else xs)
    return orc.bf16_round(acc.astype(np.float32))


def reduce(h_res, parts):
    acc = h_res.astype(np.float32).copy()
    for p in parts:
        acc += p
    return orc.bf16_round(acc)


def reference_layers(cfg, m, x0, n_layers):
    """Single-process recompute: x0[a][mb] -> x after n_layers layers."""
    x = [[v.copy() for v in row] for row in x0]
    for _ in range(n_layers):
        for mb in range(cfg.n_micro):
            outs = [attn_double(m, x[a][mb]) for a in range(cfg.n_attn)]
            pl = [dispatch(cfg, m, hn) for _, hn in outs]
            xq = np.concatenate([p[0] for p in pl])
            xs = np.concatenate([p[1] for p in pl]) if pl[0][1].size else pl[0][1]
            ids = np.concatenate([p[2] for p in pl])
            wts = np.concatenate([p[3] for p in pl])
            parts = [ffn_partial(cfg, m, f, xq, xs, ids, wts) for f in range(cfg.n_ffn)]
            T = cfg.T_mb
            for a in range(cfg.n_attn):
                x[a][mb] = reduce(outs[a][0], [p[a * T:(a + 1) * T] for p in parts])
    return x


# ----------------------------------------------------------------- executor
class Rank:
    def __init__(self, cfg, rank, dist, torch, m, x0=None):
        self.cfg, self.rank, self.dist, self.torch, self.m = cfg, rank, dist, torch, m
        self.attn = rank < cfg.n_attn
        self.idx = rank if self.attn else rank - cfg.n_attn
        self.L = afd.PayloadLayout(cfg)
        n = cfg.n_micro
        T, H = cfg.T_mb, cfg.hidden
        if self.attn:
            self.x = [v.copy() for v in x0]
            self.send = [np.zeros(self.L.nbytes, np.uint8) for _ in range(n)]
            self.recv = [np.zeros(cfg.n_ffn * T * H * 2, np.uint8) for _ in range(n)]
            self.h_res = [None] * n
        else:
            self.rx = [np.zeros(self.L.rx_total, np.uint8) for _ in range(n)]
            self.out = [np.zeros(cfg.n_attn * T * H * 2, np.uint8) for _ in range(n)]
        self.flags = {}
        self.snap = {}
        self.pending = []
        self.log = []

    # transport: (header int64[5], payload uint8[n]) per message
    def _send(self, peer, slot, value, buf, mb, data):
        hdr = self.torch.tensor([slot, value, buf, mb, data.size], dtype=self.torch.int64)
        self.pending.append(self.dist.isend(hdr, dst=peer))
        if data.size:
            t = self.torch.from_numpy(np.ascontiguousarray(data))
            self.pending.append((self.dist.isend(t, dst=peer), t))

    def _recv_one(self, peer):
        hdr = self.torch.empty(5, dtype=self.torch.int64)
        self.dist.recv(hdr, src=peer)
        slot, value, buf, mb, n = (int(v) for v in hdr)
        data = np.zeros(0, np.uint8)
        if n:
            t = self.torch.empty(n, dtype=self.torch.uint8)
            self.dist.recv(t, src=peer)
            data = t.numpy()
        if buf == RECV:  # push: the FFN rank stored its partial rows into my receive buffer
            f = peer - self.cfg.n_attn
            pb = self.L.part_bytes
            self.recv[mb][f * pb:(f + 1) * pb] = data
        elif n:
            self.snap[(peer, buf, mb)] = data
        self.flags[slot] = max(self.flags.get(slot, 0), value)

    def _sect(self, buf, name, shape, dt):
        off, n = self.L.off[name], self.L.size(name)
        return buf[off:off + n].view(dt).reshape(shape)

    def run_layer(self, seq):
        cfg, T, H = self.cfg, self.cfg.T_mb, self.cfg.hidden
        for o in afd.plan(cfg, self.rank, seq):
            k = afd.OP_NAMES[o.kind]
            self.log.append((k, o.mb, o.peer, o.slot, o.value))
            if k == "ATTN":
                h_res, h_norm = attn_double(self.m, self.x[o.mb])
                self.h_res[o.mb] = h_res
                xq, xs, ids, wts = dispatch(cfg, self.m, h_norm)
                buf = self.send[o.mb]
                buf[:] = 0
                for name, arr in zip(afd.PayloadLayout.NAMES, (xq, xs, ids, wts)):
                    b = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
                    assert b.size == self.L.size(name), (name, b.size, self.L.size(name))
                    buf[self.L.off[name]:self.L.off[name] + b.size] = b
            elif k == "SIGNAL":
                if self.attn:  # release my payload to the FFN rank
                    self._send(o.peer, o.slot, o.value, SEND, o.mb, self.send[o.mb])
                elif cfg.f2a in ("push", "nvls"):  # the rows my combine stored for attention rank a
                    a, pb = o.peer, self.L.part_bytes
                    self._send(o.peer, o.slot, o.value, RECV, o.mb, self.out[o.mb][a * pb:(a + 1) * pb])
                else:  # pull: expose my whole partial buffer
                    self._send(o.peer, o.slot, o.value, OUT, o.mb, self.out[o.mb])
            elif k == "WAIT":
                while self.flags.get(o.slot, 0) < o.value:
                    self._recv_one(o.peer)
            elif k == "PULL":
                src = self.snap[(o.peer, OUT if self.attn else SEND, o.mb)]
                dst = self.recv[o.mb] if self.attn else self.rx[o.mb]
                assert o.src_off + o.bytes <= src.size and o.dst_off + o.bytes <= dst.size
                dst[o.dst_off:o.dst_off + o.bytes] = src[o.src_off:o.src_off + o.bytes]
            elif k == "JOIN":
                pass
            elif k == "FFN":
                rx, Tf = self.rx[o.mb], cfg.T_ffn
                get = lambda name, shape, dt: rx[self.L.rx_off[name]:self.L.rx_off[name] + self.L.size(name) *
                                                 cfg.n_attn].view(dt).reshape(shape)
                if cfg.ffn_format == "bf16":
                    xq, xs = get("xq", (Tf, H), np.uint16), np.zeros(0, np.uint8)
                elif cfg.ffn_format == "mx":
                    xq, xs = get("xq", (Tf, H), np.uint8), get("xs", (Tf, H // 32), np.uint8)
                else:
                    xq, xs = get("xq", (Tf, H), np.uint8), get("xs", (Tf, H // 128), np.float32)
                ids, wts = get("ids", (Tf, cfg.top_k), np.int32), get("wts", (Tf, cfg.top_k), np.float32)
                part = ffn_partial(cfg, self.m, self.idx, xq, xs, ids, wts)
                self.out[o.mb][:] = orc.bf16_bits(part).view(np.uint8).reshape(-1)
            elif k == "REDUCE":
                pb = self.L.part_bytes
                parts = [orc.bf16_from_bits(self.recv[o.mb][f * pb:(f + 1) * pb].view(np.uint16)).reshape(T, H)
                         for f in range(cfg.n_ffn)]
                self.x[o.mb] = reduce(self.h_res[o.mb], parts)
            else:
                raise AssertionError(k)

    def finish(self):
        for p in self.pending:
            (p[0] if isinstance(p, tuple) else p).wait()
        self.pending = []
