// afd_runtime.cu — the AFD pipeline runtime (host C++ behind include/afdk.h).
//
// The reference models this pipeline analytically: pipesim.cpp:155-237
// schedules attention -> fwd link -> FFN -> bwd link per layer and
// micro-batch.  This file runs it: a per-rank op list (afdk_afd_plan,
// pure host logic, the same list the CPU protocol test executes over gloo)
// and an executor that maps each op onto the rank's streams with the
// library's own kernels and zero-SM transport (csrc/exchange.cu: copy-engine
// DMA over NVLink, stream-ordered sequence flags).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/afdk.h"
#include "afdk_internal.h"

namespace afdk {
namespace {

constexpr int kHandle = 72;  // afdk_ipc_handle bytes
constexpr int kMaxFlags = 256;

size_t a256(size_t b) { return (b + 255) / 256 * 256; }

int dispatch_bytes(const afdk_afd_cfg& c) { return c.ffn_format == AFDK_FFN_BF16 ? 2 : 1; }
size_t scale_bytes_per_token(const afdk_afd_cfg& c) {
  if (c.ffn_format == AFDK_FFN_FP8) return (size_t)(c.hidden / 128) * 4;  // fp32 per 1x128 block
  if (c.ffn_format == AFDK_FFN_MX) return (size_t)(c.hidden / 32);        // UE8M0 per 32
  return 0;                                                               // bf16 rows carry no scales
}

std::string check_cfg(const afdk_afd_cfg* c) {
  if (!c) return "NULL cfg";
  if (c->n_attn < 1 || c->n_ffn < 1) return "need at least one attention and one FFN rank";
  if (c->n_micro < 1 || c->n_micro > AFDK_AFD_MAX_MICRO) return "n_micro must be in [1, 4]";
  if ((c->n_attn + c->n_ffn) * c->n_micro > kMaxFlags) return "too many ranks x micro-batches for the flag table";
  if (c->T_mb < 1 || c->T_mb > 4096) return "T_mb must be in [1, 4096]";
  if (c->attn_chunk < 1 || c->attn_chunk > 512) return "attn_chunk must be in [1, 512]";
  if (c->hidden < 512 || c->hidden % 512) return "hidden must be a positive multiple of 512";
  if (c->ffn_format < AFDK_FFN_FP8 || c->ffn_format > AFDK_FFN_BF16) return "unknown ffn_format";
  if (c->f2a != AFDK_F2A_PUSH && c->f2a != AFDK_F2A_PULL && c->f2a != AFDK_F2A_NVLS) return "unknown f2a";
  if (c->layer_kind == AFDK_LAYER_MOE) {
    if (c->n_experts < 1 || c->n_experts > 64 || c->n_ffn > c->n_experts) return "need 1 <= n_ffn <= n_experts <= 64";
    if (c->top_k < 1 || c->top_k > 8) return "top_k must be in [1, 8]";
    if (c->inter < 128 || c->inter % 128) return "inter must be a positive multiple of 128";
    if (c->ffn_format == AFDK_FFN_MX && c->inter % 512) return "ffn_format MX needs inter % 512 == 0";
  } else if (c->layer_kind == AFDK_LAYER_DENSE) {
    if (c->ffn_format != AFDK_FFN_MX) return "dense layers run the MXFP8 dense FFN (ffn_format MX)";
    if (c->dense_slices < 1) return "dense_slices must be >= 1";
    const long total = (long)c->n_ffn * c->dense_slices;
    if (c->dense_inter < 512 || c->dense_inter % (total * 512)) return "dense_inter must be a multiple of slices x 512";
  } else {
    return "unknown layer_kind";
  }
  return "";
}

void layout(const afdk_afd_cfg& c, afdk_afd_layout* L) {
  std::memset(L, 0, sizeof(*L));
  const size_t T = c.T_mb;
  const size_t sz[4] = {T * c.hidden * dispatch_bytes(c), T * scale_bytes_per_token(c), T * c.top_k * 4,
                        T * c.top_k * 4};
  size_t o = 0, ro = 0;
  for (int i = 0; i < 4; ++i) {
    L->off[i] = o;
    L->size[i] = sz[i];
    o += a256(sz[i]);
    L->rx_off[i] = ro;
    ro += a256(sz[i] * c.n_attn);
  }
  L->total = o;
  L->rx_total = ro;
  L->part_bytes = T * c.hidden * 2;
}

int flag_slot(const afdk_afd_cfg& c, int peer_idx, int mb) { return peer_idx * c.n_micro + mb; }

// The op list of one layer on one rank (see afdk.h for the schedule).
std::vector<afdk_afd_op> plan(const afdk_afd_cfg& c, int rank, uint32_t seq) {
  afdk_afd_layout L;
  layout(c, &L);
  std::vector<afdk_afd_op> ops;
  auto op = [&](int kind, int stream, int mb) {
    afdk_afd_op o{};
    o.kind = kind;
    o.stream = stream;
    o.mb = mb;
    o.peer = -1;
    o.slot = -1;
    o.value = seq;
    ops.push_back(o);
    return &ops.back();
  };
  if (rank < c.n_attn) {
    const int a = rank;
    for (int m = 0; m < c.n_micro; ++m) {
      op(AFDK_OP_ATTN, m, m);
      for (int f = 0; f < c.n_ffn; ++f) {
        afdk_afd_op* o = op(AFDK_OP_SIGNAL, m, m);
        o->peer = c.n_attn + f;
        o->slot = flag_slot(c, a, m);
      }
      for (int f = 0; f < c.n_ffn; ++f) {
        afdk_afd_op* w = op(AFDK_OP_WAIT, m, m);
        w->peer = c.n_attn + f;
        w->slot = flag_slot(c, f, m);
        if (c.f2a == AFDK_F2A_PULL) {  // my rows of FFN f's partial
          afdk_afd_op* p = op(AFDK_OP_PULL, m, m);
          p->peer = c.n_attn + f;
          p->src_buf = AFDK_BUF_OUT;
          p->dst_buf = AFDK_BUF_RECV;
          p->src_off = (size_t)a * L.part_bytes;
          p->dst_off = (size_t)f * L.part_bytes;
          p->bytes = L.part_bytes;
        }
      }
      op(AFDK_OP_REDUCE, m, m);
    }
  } else {
    const int f = rank - c.n_attn;
    const int cs = c.n_micro;  // copy stream
    for (int m = 0; m < c.n_micro; ++m) {
      for (int a = 0; a < c.n_attn; ++a) {
        afdk_afd_op* w = op(AFDK_OP_WAIT, cs, m);
        w->peer = a;
        w->slot = flag_slot(c, a, m);
        if (c.n_attn == 1) {  // rx layout == payload layout: the whole message as one DMA
          afdk_afd_op* p = op(AFDK_OP_PULL, cs, m);
          p->peer = a;
          p->src_buf = AFDK_BUF_SEND;
          p->dst_buf = AFDK_BUF_RX;
          p->src_off = 0;
          p->dst_off = 0;
          p->bytes = L.total;
          continue;
        }
        for (int s = 0; s < 4; ++s) {
          if (L.size[s] == 0) continue;
          afdk_afd_op* p = op(AFDK_OP_PULL, cs, m);
          p->peer = a;
          p->src_buf = AFDK_BUF_SEND;
          p->dst_buf = AFDK_BUF_RX;
          p->src_off = L.off[s];
          p->dst_off = L.rx_off[s] + (size_t)a * L.size[s];
          p->bytes = L.size[s];
        }
      }
      op(AFDK_OP_JOIN, 0, m);
      op(AFDK_OP_FFN, 0, m);
      for (int a = 0; a < c.n_attn; ++a) {
        afdk_afd_op* o = op(AFDK_OP_SIGNAL, 0, m);
        o->peer = a;
        o->slot = flag_slot(c, f, m);
      }
    }
  }
  return ops;
}

}  // namespace
}  // namespace afdk

// ------------------------------------------------------------- the runtime
struct afdk_afd {
  afdk_afd_cfg cfg{};
  afdk_afd_layout lay{};
  int rank = 0, world = 0, device = 0;
  bool attn = false;
  int idx = 0;  // attention index or FFN index
  std::vector<afdk_ctx*> ctxs;
  std::vector<cudaStream_t> streams;  // n_micro + copy
  std::vector<cudaEvent_t> joins;
  // attention rank, serialised attention compute (default; AFDK_AFD_ATTN_SERIAL=0
  // restores per-micro-batch streams): the ATTN ops of all micro-batches run in
  // order on one stream instead of overlapping as persistent full-GPU kernels.
  // 1A3F MXFP8 e4m3 NVLS, layer period serial / overlapped: T_mb 256 0.767-0.770
  // / 0.775-0.777 ms, 320 0.806-0.809 / 0.830-0.834, 384 0.865-0.868 / 0.892-0.898
  bool attn_serial = false;
  cudaStream_t cstream = nullptr;
  std::vector<cudaEvent_t> ser_in, ser_out;
  uint32_t* flags = nullptr;
  std::vector<void*> own;  // every runtime allocation (freed at destroy)
  // attention rank
  std::vector<uint8_t*> send, recv, h_res, h_norm;
  std::vector<void**> part_ptrs;  // device arrays of n_ffn pointers
  // FFN rank
  std::vector<uint8_t*> rx, out;
  std::vector<uint64_t*> dst;     // device arrays of n_attn peer row-block pointers (push)
  // peers (by rank): opened mappings
  std::vector<uint32_t*> peer_flags;
  std::vector<std::vector<uint8_t*>> peer_bufs;  // attn peer: send[mb]; FFN peer: out[mb]
  std::vector<std::vector<uint8_t*>> peer_recv;  // attn peer: recv[mb] (push)
  std::vector<void*> opened;
  // NVLS return (f2a = AFDK_F2A_NVLS): groups [n_attn][n_micro] (an attention
  // rank holds only its own row a), unicast / multicast views
  std::vector<afdk_nvls*> nvls;
  std::vector<uint8_t*> nv_uc, nv_mc;  // index a * n_micro + mb
  uint32_t seq = 0;
  // measured trace (afdk_afd_trace_start / afdk_afd_trace_csv)
  struct Rec {
    cudaEvent_t a, b;
    int kind, seq, mb;
  };
  bool tracing = false;
  uint32_t trace_seq0 = 0;
  cudaEvent_t t0 = nullptr;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
};

namespace {

using afdk::set_error;

afdk_status cuda_err(const char* what, cudaError_t e) {
  set_error(std::string("afd runtime: ") + what + ": " + cudaGetErrorString(e));
  return AFDK_ERR_CUDA;
}

void* dmalloc(afdk_afd* r, size_t bytes, cudaError_t* e) {
  void* p = nullptr;
  *e = cudaMalloc(&p, bytes < 256 ? 256 : bytes);
  if (*e != cudaSuccess) return nullptr;
  r->own.push_back(p);
  return p;
}

// Local allocations of this rank (no collectives).
afdk_status alloc_local(afdk_afd* r) {
  const afdk_afd_cfg& c = r->cfg;
  cudaError_t e = cudaSuccess;
  for (int i = 0; i <= c.n_micro; ++i) {
    cudaStream_t s;
    if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return cuda_err("stream", e);
    r->streams.push_back(s);
  }
  for (int i = 0; i < c.n_micro; ++i) {
    cudaEvent_t ev;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_err("event", e);
    r->joins.push_back(ev);
  }
  if (r->attn) {
    const char* env = std::getenv("AFDK_AFD_ATTN_SERIAL");
    r->attn_serial = !(env && env[0] == '0');
  }
  if (r->attn_serial) {
    if ((e = cudaStreamCreateWithFlags(&r->cstream, cudaStreamNonBlocking)) != cudaSuccess) return cuda_err("stream", e);
    for (int i = 0; i < 2 * c.n_micro; ++i) {
      cudaEvent_t ev;
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return cuda_err("event", e);
      (i < c.n_micro ? r->ser_in : r->ser_out).push_back(ev);
    }
  }
  r->flags = static_cast<uint32_t*>(dmalloc(r, afdk::kMaxFlags * 4, &e));
  if (!r->flags || (e = cudaMemset(r->flags, 0, afdk::kMaxFlags * 4)) != cudaSuccess) return cuda_err("flags", e);
  const size_t row = (size_t)c.T_mb * c.hidden * 2;
  for (int m = 0; m < c.n_micro; ++m) {
    if (r->attn) {
      auto* s = static_cast<uint8_t*>(dmalloc(r, r->lay.total, &e));
      auto* rc = static_cast<uint8_t*>(dmalloc(r, (size_t)c.n_ffn * row, &e));
      auto* hr = static_cast<uint8_t*>(dmalloc(r, row, &e));
      auto* hn = static_cast<uint8_t*>(dmalloc(r, row, &e));
      auto* pp = static_cast<void**>(dmalloc(r, (size_t)c.n_ffn * sizeof(void*), &e));
      if (!s || !rc || !hr || !hn || !pp) return cuda_err("attention buffers", e);
      std::vector<void*> hp(c.n_ffn);
      for (int f = 0; f < c.n_ffn; ++f) hp[f] = rc + (size_t)f * row;
      if ((e = cudaMemcpy(pp, hp.data(), hp.size() * sizeof(void*), cudaMemcpyHostToDevice)) != cudaSuccess)
        return cuda_err("partial pointers", e);
      r->send.push_back(s);
      r->recv.push_back(rc);
      r->h_res.push_back(hr);
      r->h_norm.push_back(hn);
      r->part_ptrs.push_back(pp);
    } else {
      auto* x = static_cast<uint8_t*>(dmalloc(r, r->lay.rx_total, &e));
      auto* o = static_cast<uint8_t*>(dmalloc(r, (size_t)c.n_attn * row, &e));
      auto* d = static_cast<uint64_t*>(dmalloc(r, (size_t)c.n_attn * 8, &e));
      if (!x || !o || !d) return cuda_err("FFN buffers", e);
      r->rx.push_back(x);
      r->out.push_back(o);
      r->dst.push_back(d);
    }
  }
  return AFDK_OK;
}

// Fixed-size per-rank blob: status, then flags + per-mb handles.
struct Blob {
  int32_t ok;
  int32_t rank;
  int32_t pid;                            // NVLS: the group creator's process ...
  int32_t nvls_fd[AFDK_AFD_MAX_MICRO];    // ... and its exported descriptors (attention ranks)
  uint8_t flags[afdk::kHandle];
  uint8_t bufs[AFDK_AFD_MAX_MICRO][afdk::kHandle];  // attn: send; FFN: out
  uint8_t recv[AFDK_AFD_MAX_MICRO][afdk::kHandle];  // attn: recv
};

afdk_status export_handles(afdk_afd* r, Blob* b) {
  afdk_ctx* ctx = r->ctxs[0];
  afdk_status s;
  const afdk_afd_cfg& c = r->cfg;
  if (c.f2a == AFDK_F2A_NVLS) {
    r->nvls.assign((size_t)c.n_attn * c.n_micro, nullptr);
    r->nv_uc.assign(r->nvls.size(), nullptr);
    r->nv_mc.assign(r->nvls.size(), nullptr);
    b->pid = (int32_t)getpid();
    if (r->attn)  // this attention rank creates its groups: members = itself + every FFN rank
      for (int m = 0; m < c.n_micro; ++m) {
        int fd = -1;
        if ((s = afdk_nvls_create(ctx, 1 + c.n_ffn, r->lay.part_bytes, 0, -1, &r->nvls[(size_t)r->idx * c.n_micro + m],
                                  &fd)) != AFDK_OK)
          return s;
        b->nvls_fd[m] = fd;
      }
  }
  if ((s = afdk_ipc_handle(ctx, r->flags, b->flags)) != AFDK_OK) return s;
  for (int m = 0; m < r->cfg.n_micro; ++m) {
    if ((s = afdk_ipc_handle(ctx, r->attn ? r->send[m] : r->out[m], b->bufs[m])) != AFDK_OK) return s;
    if (r->attn && (s = afdk_ipc_handle(ctx, r->recv[m], b->recv[m])) != AFDK_OK) return s;
  }
  return AFDK_OK;
}

afdk_status connect(afdk_afd* r, const std::vector<Blob>& all) {
  const afdk_afd_cfg& c = r->cfg;
  afdk_ctx* ctx = r->ctxs[0];
  r->peer_flags.assign(r->world, nullptr);
  r->peer_bufs.assign(r->world, {});
  r->peer_recv.assign(r->world, {});
  auto open = [&](const uint8_t* h, uint8_t** p) {
    void* v = nullptr;
    const afdk_status s = afdk_ipc_open(ctx, h, &v);
    if (s == AFDK_OK) { r->opened.push_back(v); *p = static_cast<uint8_t*>(v); }
    return s;
  };
  for (int q = 0; q < r->world; ++q) {
    const bool q_attn = q < c.n_attn;
    if (q == r->rank || q_attn == r->attn) continue;  // A talks to F only
    uint8_t* fp = nullptr;
    afdk_status s;
    if ((s = open(all[q].flags, &fp)) != AFDK_OK) return s;
    r->peer_flags[q] = reinterpret_cast<uint32_t*>(fp);
    for (int m = 0; m < c.n_micro; ++m) {
      uint8_t* p = nullptr;
      if ((s = open(all[q].bufs[m], &p)) != AFDK_OK) return s;
      r->peer_bufs[q].push_back(p);
      if (q_attn && c.f2a == AFDK_F2A_PUSH) {
        uint8_t* rp = nullptr;
        if ((s = open(all[q].recv[m], &rp)) != AFDK_OK) return s;
        r->peer_recv[q].push_back(rp);
      }
    }
  }
  if (c.f2a == AFDK_F2A_NVLS) {
    afdk_status s;
    if (!r->attn)  // join every attention rank's groups (all joins before any bind)
      for (int a = 0; a < c.n_attn; ++a)
        for (int m = 0; m < c.n_micro; ++m)
          if ((s = afdk_nvls_create(ctx, 1 + c.n_ffn, r->lay.part_bytes, all[a].pid, all[a].nvls_fd[m],
                                    &r->nvls[(size_t)a * c.n_micro + m], nullptr)) != AFDK_OK)
            return s;
    for (size_t i = 0; i < r->nvls.size(); ++i) {
      if (!r->nvls[i]) continue;
      void *uc = nullptr, *mc = nullptr;
      if ((s = afdk_nvls_bind(r->nvls[i], &uc, &mc)) != AFDK_OK) return s;
      r->nv_uc[i] = static_cast<uint8_t*>(uc);
      r->nv_mc[i] = static_cast<uint8_t*>(mc);
    }
    if (r->attn) {  // h_res IS this rank's member buffer: x = ld_reduce(h_res + partials)
      for (int m = 0; m < c.n_micro; ++m) r->h_res[m] = r->nv_uc[(size_t)r->idx * c.n_micro + m];
    } else {  // the combine writes token rows of attention rank a into my member buffer of group (a, mb)
      for (int m = 0; m < c.n_micro; ++m) {
        std::vector<uint64_t> d(c.n_attn);
        for (int a = 0; a < c.n_attn; ++a) d[a] = reinterpret_cast<uint64_t>(r->nv_uc[(size_t)a * c.n_micro + m]);
        const cudaError_t e = cudaMemcpy(r->dst[m], d.data(), d.size() * 8, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return cuda_err("nvls scatter pointers", e);
      }
    }
  }
  if (!r->attn && c.f2a == AFDK_F2A_PUSH) {
    // my slot idx of every attention rank's [n_ffn, T_mb, hidden] receive buffer
    const size_t slot = (size_t)r->idx * r->lay.part_bytes;
    for (int m = 0; m < c.n_micro; ++m) {
      std::vector<uint64_t> d(c.n_attn);
      for (int a = 0; a < c.n_attn; ++a) d[a] = reinterpret_cast<uint64_t>(r->peer_recv[a][m] + slot);
      const cudaError_t e = cudaMemcpy(r->dst[m], d.data(), d.size() * 8, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_err("scatter pointers", e);
    }
  }
  return AFDK_OK;
}

void release(afdk_afd* r) {
  if (!r) return;
  afdk::DeviceGuard g(r->device);
  for (cudaStream_t s : r->streams) cudaStreamSynchronize(s);
  if (r->cstream) cudaStreamSynchronize(r->cstream);
  if (!r->ctxs.empty())
    for (void* p : r->opened) afdk_ipc_close(r->ctxs[0], p);
  for (afdk_nvls* g : r->nvls) afdk_nvls_destroy(g);
  for (cudaEvent_t e : r->joins) cudaEventDestroy(e);
  for (cudaEvent_t e : r->ser_in) cudaEventDestroy(e);
  for (cudaEvent_t e : r->ser_out) cudaEventDestroy(e);
  if (r->cstream) cudaStreamDestroy(r->cstream);
  for (cudaEvent_t e : r->ev_pool) cudaEventDestroy(e);
  if (r->t0) cudaEventDestroy(r->t0);
  for (cudaStream_t s : r->streams) cudaStreamDestroy(s);
  for (void* p : r->own) cudaFree(p);
  delete r;
}

inline uint8_t* sect(uint8_t* base, const afdk_afd_layout& L, int s) { return base + L.off[s]; }

// Executes the shared ops (SIGNAL / WAIT / PULL / JOIN); ATTN / REDUCE / FFN
// are role callbacks.
afdk_status trace_event(afdk_afd* r, cudaEvent_t* ev) {
  if (r->ev_used == r->ev_pool.size()) {
    cudaEvent_t e;
    const cudaError_t err = cudaEventCreate(&e);
    if (err != cudaSuccess) return cuda_err("trace event", err);
    r->ev_pool.push_back(e);
  }
  *ev = r->ev_pool[r->ev_used++];
  return AFDK_OK;
}

template <typename Compute>
afdk_status run_plan(afdk_afd* r, Compute&& compute) {
  const uint32_t seq = ++r->seq;
  const std::vector<afdk_afd_op> ops = afdk::plan(r->cfg, r->rank, seq);
  afdk_ctx* ctx0 = r->ctxs[0];
  for (const afdk_afd_op& o : ops) {
    cudaStream_t s = r->streams[o.stream];
    afdk_status st = AFDK_OK;
    // serialised attention: ATTN(m) moves to the compute stream, ordered after
    // its micro-batch stream's earlier work and before its later work
    const bool serial = r->attn_serial && o.kind == AFDK_OP_ATTN;
    if (serial) {
      cudaError_t e = cudaEventRecord(r->ser_in[o.mb], s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(r->cstream, r->ser_in[o.mb], 0);
      if (e != cudaSuccess) return cuda_err("attn serial", e);
      s = r->cstream;
    }
    // measured trace: an event pair around every op that occupies a resource
    const bool traced = r->tracing && (o.kind == AFDK_OP_ATTN || o.kind == AFDK_OP_REDUCE ||
                                       o.kind == AFDK_OP_FFN || o.kind == AFDK_OP_PULL);
    afdk_afd::Rec rec{};
    if (traced) {
      if ((st = trace_event(r, &rec.a)) != AFDK_OK || (st = trace_event(r, &rec.b)) != AFDK_OK) return st;
      rec.kind = o.kind;
      rec.seq = (int)seq;
      rec.mb = o.mb;
      cudaEventRecord(rec.a, s);
    }
    switch (o.kind) {
      case AFDK_OP_SIGNAL:
        st = afdk_signal(ctx0, r->peer_flags[o.peer] + o.slot, o.value, s);
        break;
      case AFDK_OP_WAIT:
        st = afdk_wait(ctx0, r->flags + o.slot, o.value, s);
        break;
      case AFDK_OP_PULL: {
        uint8_t* src = r->peer_bufs[o.peer][o.mb] + o.src_off;
        uint8_t* dst = (o.dst_buf == AFDK_BUF_RX ? r->rx[o.mb] : r->recv[o.mb]) + o.dst_off;
        st = afdk_copy(ctx0, dst, src, o.bytes, s);
        break;
      }
      case AFDK_OP_JOIN: {
        cudaError_t e = cudaEventRecord(r->joins[o.mb], r->streams[r->cfg.n_micro]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, r->joins[o.mb], 0);
        if (e != cudaSuccess) st = cuda_err("join", e);
        break;
      }
      default:
        st = compute(o, s);
    }
    if (st != AFDK_OK) return st;
    if (traced) {
      cudaEventRecord(rec.b, s);
      r->recs.push_back(rec);
    }
    if (serial) {
      cudaError_t e = cudaEventRecord(r->ser_out[o.mb], s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(r->streams[o.stream], r->ser_out[o.mb], 0);
      if (e != cudaSuccess) return cuda_err("attn serial", e);
    }
  }
  return AFDK_OK;
}

}  // namespace

extern "C" {

afdk_status afdk_afd_check_cfg(const afdk_afd_cfg* cfg) {
  const std::string m = afdk::check_cfg(cfg);
  if (!m.empty()) { set_error("afdk_afd: " + m); return AFDK_ERR_INVALID; }
  return AFDK_OK;
}

afdk_status afdk_afd_get_layout(const afdk_afd_cfg* cfg, afdk_afd_layout* out) {
  if (afdk_afd_check_cfg(cfg) != AFDK_OK) return AFDK_ERR_INVALID;
  if (!out) { set_error("afdk_afd_get_layout: NULL out"); return AFDK_ERR_INVALID; }
  afdk::layout(*cfg, out);
  return AFDK_OK;
}

afdk_status afdk_afd_plan(const afdk_afd_cfg* cfg, int rank, uint32_t seq, afdk_afd_op* ops, int cap, int* n_ops) {
  if (afdk_afd_check_cfg(cfg) != AFDK_OK) return AFDK_ERR_INVALID;
  if (rank < 0 || rank >= cfg->n_attn + cfg->n_ffn || !n_ops) {
    set_error("afdk_afd_plan: rank out of range / NULL n_ops");
    return AFDK_ERR_INVALID;
  }
  const std::vector<afdk_afd_op> p = afdk::plan(*cfg, rank, seq);
  *n_ops = (int)p.size();
  if (!ops) return AFDK_OK;  // size query
  if (cap < (int)p.size()) { set_error("afdk_afd_plan: op buffer too small"); return AFDK_ERR_INVALID; }
  std::memcpy(ops, p.data(), p.size() * sizeof(afdk_afd_op));
  return AFDK_OK;
}

afdk_status afdk_afd_create(afdk_ctx* const* ctxs, const afdk_afd_cfg* cfg, int rank, afdk_allgather_fn allgather,
                            void* user, afdk_afd** out) {
  if (!out || !ctxs || !allgather) { set_error("afdk_afd_create: NULL argument"); return AFDK_ERR_INVALID; }
  *out = nullptr;
  if (afdk_afd_check_cfg(cfg) != AFDK_OK) return AFDK_ERR_INVALID;
  const int world = cfg->n_attn + cfg->n_ffn;
  if (rank < 0 || rank >= world) { set_error("afdk_afd_create: rank out of range"); return AFDK_ERR_INVALID; }
  auto* r = new afdk_afd();
  r->cfg = *cfg;
  r->rank = rank;
  r->world = world;
  r->attn = rank < cfg->n_attn;
  r->idx = r->attn ? rank : rank - cfg->n_attn;
  afdk::layout(*cfg, &r->lay);
  for (int m = 0; m < cfg->n_micro; ++m) {
    if (!ctxs[m]) { delete r; set_error("afdk_afd_create: NULL context"); return AFDK_ERR_INVALID; }
    r->ctxs.push_back(ctxs[m]);
  }
  r->device = afdk_ctx_device(ctxs[0]);  // run on the contexts' device
  afdk::DeviceGuard g(r->device);

  // 1) local allocation + handle export; 2) agree on success; 3) map peers
  Blob mine{};
  mine.rank = rank;
  afdk_status st = alloc_local(r);
  if (st == AFDK_OK) st = export_handles(r, &mine);
  const std::string local_err = st == AFDK_OK ? "" : afdk_last_error();
  mine.ok = st == AFDK_OK ? 1 : 0;
  std::vector<Blob> all(world);
  if (allgather(user, &mine, sizeof(Blob), all.data()) != 0) {
    release(r);
    set_error("afdk_afd_create: allgather callback failed");
    return AFDK_ERR_INVALID;
  }
  for (int q = 0; q < world; ++q) {
    if (!all[q].ok || all[q].rank != q) {
      release(r);
      set_error("afdk_afd_create: rank " + std::to_string(q) + " failed to set up" +
                (local_err.empty() ? "" : " (this rank: " + local_err + ")"));
      return st != AFDK_OK ? st : AFDK_ERR_CUDA;
    }
  }
  st = connect(r, all);
  int32_t ok = st == AFDK_OK ? 1 : 0;
  std::vector<int32_t> oks(world);
  cudaDeviceSynchronize();
  if (allgather(user, &ok, sizeof(ok), oks.data()) != 0) st = AFDK_ERR_INVALID;
  for (int q = 0; q < world && st == AFDK_OK; ++q)
    if (!oks[q]) { set_error("afdk_afd_create: rank " + std::to_string(q) + " failed to map its peers"); st = AFDK_ERR_CUDA; }
  if (st != AFDK_OK) { release(r); return st; }
  *out = r;
  return AFDK_OK;
}

void afdk_afd_destroy(afdk_afd* afd) { release(afd); }

afdk_stream afdk_afd_stream(afdk_afd* afd, int i) {
  return (afd && i >= 0 && i < (int)afd->streams.size()) ? afd->streams[i] : nullptr;
}

void* afdk_afd_buffer(afdk_afd* afd, int which, int mb) {
  if (!afd || mb < 0 || mb >= afd->cfg.n_micro) return nullptr;
  if (afd->attn) {
    switch (which) {
      case AFDK_BUF_SEND: return afd->send[mb];
      case AFDK_BUF_RECV: return afd->recv[mb];
      case 4: return afd->h_res[mb];
      case 5: return afd->h_norm[mb];
      default: return nullptr;
    }
  }
  return which == AFDK_BUF_RX ? afd->rx[mb] : which == AFDK_BUF_OUT ? afd->out[mb] : nullptr;
}

uint32_t afdk_afd_seq(const afdk_afd* afd) { return afd ? afd->seq : 0; }

afdk_status afdk_afd_trace_start(afdk_afd* afd) {
  if (!afd) { set_error("afdk_afd_trace_start: NULL"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(afd->device);
  cudaError_t e = cudaSuccess;
  if (!afd->t0 && (e = cudaEventCreate(&afd->t0)) != cudaSuccess) return cuda_err("trace t0", e);
  afd->recs.clear();
  afd->ev_used = 0;
  afd->trace_seq0 = afd->seq;
  afd->tracing = true;
  // t0 on stream 0; every other stream starts after it
  if ((e = cudaEventRecord(afd->t0, afd->streams[0])) != cudaSuccess) return cuda_err("trace t0", e);
  for (size_t i = 1; i < afd->streams.size(); ++i)
    if ((e = cudaStreamWaitEvent(afd->streams[i], afd->t0, 0)) != cudaSuccess) return cuda_err("trace t0", e);
  if (afd->cstream && (e = cudaStreamWaitEvent(afd->cstream, afd->t0, 0)) != cudaSuccess) return cuda_err("trace t0", e);
  return AFDK_OK;
}

afdk_status afdk_afd_trace_csv(afdk_afd* afd, char* buf, size_t cap, size_t* len) {
  if (!afd || !len) { set_error("afdk_afd_trace_csv: NULL argument"); return AFDK_ERR_INVALID; }
  if (!afd->t0) { set_error("afdk_afd_trace_csv: tracing never started"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(afd->device);
  afd->tracing = false;
  struct Row {
    double t, d;
    const char* res;
    const char* stage;
    int layer, mb;
  };
  std::vector<Row> rows;
  for (const auto& rc : afd->recs) {
    float ms_a = 0.f, ms_b = 0.f;
    cudaError_t e = cudaEventSynchronize(rc.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms_a, afd->t0, rc.a);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms_b, afd->t0, rc.b);
    if (e != cudaSuccess) return cuda_err("trace timing", e);
    const char* res = "attention";
    const char* stage = "attention";
    if (rc.kind == AFDK_OP_FFN) res = stage = "ffn";
    if (rc.kind == AFDK_OP_PULL) { res = afd->attn ? "bwd_link" : "fwd_link"; stage = "comm"; }
    rows.push_back({ms_a * 1e-3, (ms_b - ms_a) * 1e-3, res, stage, rc.seq - (int)afd->trace_seq0 - 1, rc.mb});
  }
  // the pulls of one (layer, micro-batch) form one link interval
  std::vector<Row> merged;
  for (const Row& r : rows) {
    bool folded = false;
    if (std::strcmp(r.stage, "comm") == 0)
      for (Row& m : merged)
        if (m.res == r.res && m.layer == r.layer && m.mb == r.mb) {
          const double end = std::max(m.t + m.d, r.t + r.d);
          m.t = std::min(m.t, r.t);
          m.d = end - m.t;
          folded = true;
          break;
        }
    if (!folded) merged.push_back(r);
  }
  std::stable_sort(merged.begin(), merged.end(), [](const Row& a, const Row& b) { return a.t < b.t; });
  std::string csv = "time_s,resource,layer,micro_batch,stage,duration_s\n";
  char line[256];
  for (const Row& r : merged) {
    std::snprintf(line, sizeof(line), "%.9f,%s,%d,%d,%s,%.9f\n", r.t, r.res, r.layer, r.mb, r.stage, r.d);
    csv += line;
  }
  *len = csv.size();
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, csv.size());
    std::memcpy(buf, csv.data(), n);
    buf[n] = '\0';
  }
  return AFDK_OK;
}

afdk_status afdk_afd_sync(afdk_afd* afd) {
  if (!afd) { set_error("afdk_afd_sync: NULL"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(afd->device);
  if (afd->cstream) {
    const cudaError_t e = cudaStreamSynchronize(afd->cstream);
    if (e != cudaSuccess) return cuda_err("sync", e);
  }
  for (cudaStream_t s : afd->streams) {
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_err("sync", e);
  }
  return AFDK_OK;
}

afdk_status afdk_afd_attn_layer(afdk_afd* afd, const afdk_mfa_weights* w, const void* gate_w,
                                const afdk_afd_attn_mb* mbs) {
  if (!afd || !w || !mbs) { set_error("afdk_afd_attn_layer: NULL argument"); return AFDK_ERR_INVALID; }
  if (!afd->attn) { set_error("afdk_afd_attn_layer: this rank is an FFN rank"); return AFDK_ERR_INVALID; }
  const afdk_afd_cfg& c = afd->cfg;
  if (c.layer_kind == AFDK_LAYER_MOE && !gate_w) { set_error("afdk_afd_attn_layer: MoE layers need gate_w"); return AFDK_ERR_INVALID; }
  afdk::DeviceGuard g(afd->device);
  const afdk_afd_layout& L = afd->lay;
  const size_t row = (size_t)c.hidden * 2;
  return run_plan(afd, [&](const afdk_afd_op& o, cudaStream_t s) -> afdk_status {
    const int m = o.mb;
    const afdk_afd_attn_mb& in = mbs[m];
    afdk_ctx* ctx = afd->ctxs[m];
    afdk_status st = AFDK_OK;
    if (o.kind == AFDK_OP_REDUCE) {
      if (c.f2a == AFDK_F2A_NVLS)  // x = h_res + sum of the FFN partials, summed in the switch
        return afdk_nvls_reduce_bf16(ctx, afd->nv_mc[(size_t)afd->idx * c.n_micro + m], in.x,
                                     (size_t)c.T_mb * c.hidden, s);
      return afdk_add_partials(ctx, afd->h_res[m], const_cast<const void* const*>(afd->part_ptrs[m]), c.n_ffn,
                               (size_t)c.T_mb * c.hidden, in.x, s);
    }
    if (o.kind != AFDK_OP_ATTN) { set_error("afd runtime: unexpected op on an attention rank"); return AFDK_ERR_INVALID; }
    // the attention-side layer in attn_chunk pieces (its GEMM N limit); one payload
    for (int c0 = 0; c0 < c.T_mb && st == AFDK_OK; c0 += c.attn_chunk) {
      const int n = (c.T_mb - c0) < c.attn_chunk ? (c.T_mb - c0) : c.attn_chunk;
      afdk_mfa_layer_args a{n, static_cast<const uint8_t*>(in.x) + c0 * row, in.k_cache, in.v_cache, in.num_pages,
                            in.page_size, in.block_table + (size_t)c0 * in.max_pages, in.max_pages,
                            in.seq_lens + c0, afd->h_res[m] + c0 * row, afd->h_norm[m] + c0 * row};
      st = in.k_scale > 0.0f ? afdk_mfa_layer_fp8(ctx, w, &a, in.k_scale, in.v_scale, s) : afdk_mfa_layer(ctx, w, &a, s);
    }
    if (st != AFDK_OK) return st;
    uint8_t* buf = afd->send[m];
    auto* ids = reinterpret_cast<int32_t*>(sect(buf, L, 2));
    auto* wts = reinterpret_cast<float*>(sect(buf, L, 3));
    if (c.ffn_format == AFDK_FFN_FP8) {  // router + 1x128 FP8 dispatch quantisation in one pass
      return afdk_router_topk(ctx, afd->h_norm[m], gate_w, c.T_mb, c.hidden, c.n_experts, c.top_k, 0, nullptr, ids,
                              wts, sect(buf, L, 0), reinterpret_cast<float*>(sect(buf, L, 1)), s);
    }
    if (c.layer_kind == AFDK_LAYER_MOE)
      st = afdk_router_topk(ctx, afd->h_norm[m], gate_w, c.T_mb, c.hidden, c.n_experts, c.top_k, 0, nullptr, ids, wts,
                            nullptr, nullptr, s);
    if (st != AFDK_OK) return st;
    if (c.ffn_format == AFDK_FFN_MX)
      return afdk_quant_mx(ctx, afd->h_norm[m], c.T_mb, c.hidden, sect(buf, L, 0), sect(buf, L, 1), s);
    return afdk_copy(ctx, sect(buf, L, 0), afd->h_norm[m], (size_t)c.T_mb * row, s);  // bf16 rows
  });
}

afdk_status afdk_afd_ffn_layer(afdk_afd* afd, const afdk_afd_ffn_weights* w) {
  if (!afd || !w) { set_error("afdk_afd_ffn_layer: NULL argument"); return AFDK_ERR_INVALID; }
  if (afd->attn) { set_error("afdk_afd_ffn_layer: this rank is an attention rank"); return AFDK_ERR_INVALID; }
  const afdk_afd_cfg& c = afd->cfg;
  afdk::DeviceGuard g(afd->device);
  const afdk_afd_layout& L = afd->lay;
  const int f = afd->idx;
  const int lo = f * c.n_experts / c.n_ffn, hi = (f + 1) * c.n_experts / c.n_ffn;
  const int Tf = c.n_attn * c.T_mb;
  const int sh_lo = (int)((long)f * Tf / c.n_ffn), sh_hi = (int)((long)(f + 1) * Tf / c.n_ffn);
  return run_plan(afd, [&](const afdk_afd_op& o, cudaStream_t s) -> afdk_status {
    if (o.kind != AFDK_OP_FFN) { set_error("afd runtime: unexpected op on an FFN rank"); return AFDK_ERR_INVALID; }
    const int m = o.mb;
    afdk_ctx* ctx = afd->ctxs[0];
    uint8_t* rx = afd->rx[m];
    const bool push = c.f2a != AFDK_F2A_PULL;  // NVLS: the scatter targets are local member buffers
    afdk_row_scatter sc{c.n_attn, c.T_mb, afd->dst[m]};
    void* out = afd->out[m];
    const auto* ids = reinterpret_cast<const int32_t*>(rx + L.rx_off[2]);
    const auto* wts = reinterpret_cast<const float*>(rx + L.rx_off[3]);
    if (c.layer_kind == AFDK_LAYER_DENSE) {
      const int Is = c.dense_inter / (c.n_ffn * c.dense_slices);
      afdk_dense_mx_weights dw{c.hidden, Is, c.dense_slices, w->w13, static_cast<const uint8_t*>(w->s13), w->w2,
                               static_cast<const uint8_t*>(w->s2)};
      return push ? afdk_dense_ffn_mx_scatter(ctx, &dw, Tf, rx + L.rx_off[0], rx + L.rx_off[1], &sc, s)
                  : afdk_dense_ffn_mx(ctx, &dw, Tf, rx + L.rx_off[0], rx + L.rx_off[1], out, s);
    }
    if (c.ffn_format == AFDK_FFN_FP8) {
      afdk_moe_weights mw{c.hidden, c.inter, c.n_experts, c.top_k, lo, hi, w->w13,
                          static_cast<const float*>(w->s13), w->w2, static_cast<const float*>(w->s2)};
      afdk_moe_args a{Tf, rx + L.rx_off[0], reinterpret_cast<const float*>(rx + L.rx_off[1]), ids, wts, sh_lo, sh_hi,
                      out};
      return push ? afdk_moe_ffn_scatter(ctx, &mw, &a, &sc, s) : afdk_moe_ffn(ctx, &mw, &a, s);
    }
    if (c.ffn_format == AFDK_FFN_MX) {
      afdk_moe_mx_weights mw{c.hidden, c.inter, c.n_experts, c.top_k, lo, hi, w->w13,
                             static_cast<const uint8_t*>(w->s13), w->w2, static_cast<const uint8_t*>(w->s2)};
      afdk_moe_mx_args a{Tf, rx + L.rx_off[0], rx + L.rx_off[1], ids, wts, sh_lo, sh_hi, out};
      return push ? afdk_moe_ffn_mx_scatter(ctx, &mw, &a, &sc, s) : afdk_moe_ffn_mx(ctx, &mw, &a, s);
    }
    afdk_moe_bf16_weights mw{c.hidden, c.inter, c.n_experts, c.top_k, lo, hi, w->w13, w->w2};
    afdk_moe_bf16_args a{Tf, rx + L.rx_off[0], ids, wts, sh_lo, sh_hi, out};
    return push ? afdk_moe_ffn_bf16_scatter(ctx, &mw, &a, &sc, s) : afdk_moe_ffn_bf16(ctx, &mw, &a, s);
  });
}

}  // extern "C"
