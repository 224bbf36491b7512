// afd_cpp_demo.cpp — the disaggregated decode pipeline driven from C++ alone
// (no Python, no torch): what a C++ caller of the reference's interface does
// to run the AFD runtime behind the C-ABI (include/afdk.h, afdk_afd_*).
//
//   usage: afd_cpp_demo <world> <n_attn> <fp8|mx|bf16> <push|pull> [steps]
//
// The parent forks one process per rank (rank r on GPU r % device_count) and
// the ranks rendezvous through files in a private temp directory (the
// allgather callback of afdk_afd_create; any transport works).  Every rank
// builds its caller-owned data on the host from a fixed seed — attention
// weights, KV caches and inputs on attention ranks; its expert shard plus
// the shared expert on FFN ranks, expert e's tensors a function of (seed, e)
// only — and runs `steps` decode steps x 2 layers x 2 micro-batches.  Each
// layer's output is snapshotted by a copy enqueued on the runtime's
// micro-batch stream between that layer and the next.  After each step every
// attention rank recomputes every layer on its own GPU from the runtime's
// input to that layer through the single-GPU calls (afdk_mfa_layer,
// afdk_router_topk / afdk_quant_mx, the MoE over ALL experts,
// afdk_add_partials) and compares (bar 2e-2 of max|ref|, as
// tests/afd_gpu_check.py: the runtime sums bf16-rounded EP partials where the
// recompute rounds the whole MoE once).  Prints one JSON line from rank 0;
// exit status 0 iff every rank passed.
#include <cuda_runtime.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "afdk.h"

namespace {

constexpr int kHidden = 1024, kQLora = 256, kHeads = 64, kHeadDim = 256, kPage = 64;
constexpr int kExperts = 8, kTopK = 2, kInter = 512, kTmb = 24, kCtx = 300, kLayers = 2, kMicro = 2;

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      std::fprintf(stderr, "rank %d: %s:%d %s\n", g_rank, __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(3);                                                                              \
    }                                                                                            \
  } while (0)
#define AK(x)                                                                                    \
  do {                                                                                           \
    afdk_status s_ = (x);                                                                        \
    if (s_ != AFDK_OK) {                                                                         \
      std::fprintf(stderr, "rank %d: %s:%d afdk status %d: %s\n", g_rank, __FILE__, __LINE__, (int)s_, \
                   afdk_last_error());                                                           \
      std::exit(4);                                                                              \
    }                                                                                            \
  } while (0)

int g_rank = -1;

// ------------------------------------------------------------ host data
struct Rng {  // splitmix64 + Box-Muller: deterministic on every rank
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed * 0x9E3779B97F4A7C15ull + 1) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uni() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
  float normal() { return (float)(std::sqrt(-2.0 * std::log(uni())) * std::cos(6.283185307179586 * uni())); }
};

uint16_t bf16(float f) {  // round to nearest even
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

std::vector<uint16_t> randn_bf16(Rng& g, size_t n, float scale, float offset = 0.f) {
  std::vector<uint16_t> v(n);
  for (auto& x : v) x = bf16(offset + scale * g.normal());
  return v;
}

std::vector<uint8_t> rand_e4m3(Rng& g, size_t n) {  // |w| in 2^-6..~2^0 before scaling
  std::vector<uint8_t> v(n);
  for (auto& x : v) x = (uint8_t)((0x18 + g.next() % 0x28) | ((g.next() & 1) << 7));
  return v;
}

template <class T>
void* upload(const std::vector<T>& h) {
  void* d = nullptr;
  CK(cudaMalloc(&d, h.size() * sizeof(T)));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

void* dalloc(size_t bytes) {
  void* d = nullptr;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  return d;
}

float bf16_to_f(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// ------------------------------------------------------- file rendezvous
struct FileGather {
  std::string dir;
  int rank, world, round = 0;
};

int file_allgather(void* user, const void* mine, size_t bytes, void* all) {
  auto* fg = static_cast<FileGather*>(user);
  const int r = fg->round++;
  char path[512], tmp[512];
  std::snprintf(path, sizeof path, "%s/g%d_r%d", fg->dir.c_str(), r, fg->rank);
  std::snprintf(tmp, sizeof tmp, "%s.tmp", path);
  FILE* f = std::fopen(tmp, "wb");
  if (!f || std::fwrite(mine, 1, bytes, f) != bytes) return 1;
  std::fclose(f);
  if (std::rename(tmp, path) != 0) return 1;  // atomic publish
  const auto t0 = std::chrono::steady_clock::now();
  for (int p = 0; p < fg->world; ++p) {
    std::snprintf(path, sizeof path, "%s/g%d_r%d", fg->dir.c_str(), r, p);
    for (;;) {
      FILE* in = std::fopen(path, "rb");
      if (in) {
        const size_t got = std::fread(static_cast<char*>(all) + p * bytes, 1, bytes, in);
        std::fclose(in);
        if (got == bytes) break;
        return 1;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300)) return 1;
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  return 0;
}

// ------------------------------------------------------------ experts
// Expert e (e == kExperts: the shared expert) in the format's layout.
struct ExpertHost {
  std::vector<uint8_t> w13, w2;              // e4m3 codes, or bf16 as bytes
  std::vector<uint8_t> sf13, sf2;            // MX: UE8M0
  std::vector<float> s13, s2;                // FP8: 128x128 fp32
};

ExpertHost make_expert(int fmt, int e) {
  Rng g(1000 + e);
  ExpertHost x;
  const size_t n13 = (size_t)2 * kInter * kHidden, n2 = (size_t)kHidden * kInter;
  if (fmt == AFDK_FFN_BF16) {
    auto a = randn_bf16(g, n13, 1.f / std::sqrt((float)kHidden));
    auto b = randn_bf16(g, n2, 1.f / std::sqrt((float)kInter));
    x.w13.resize(n13 * 2);
    x.w2.resize(n2 * 2);
    std::memcpy(x.w13.data(), a.data(), n13 * 2);
    std::memcpy(x.w2.data(), b.data(), n2 * 2);
    return x;
  }
  x.w13 = rand_e4m3(g, n13);
  x.w2 = rand_e4m3(g, n2);
  if (fmt == AFDK_FFN_MX) {  // 2^-7
    x.sf13.assign(n13 / 32, 120);
    x.sf2.assign(n2 / 32, 120);
  } else {
    x.s13.assign((size_t)(2 * kInter / 128) * (kHidden / 128), 0.5f / std::sqrt((float)kHidden));
    x.s2.assign((size_t)(kHidden / 128) * (kInter / 128), 0.5f / std::sqrt((float)kInter));
  }
  return x;
}

struct ExpertDev {
  void *w13, *w2, *s13, *s2;
};

// experts lo..hi-1 followed by the shared expert, stacked ([(n+1), ...])
ExpertDev upload_experts(int fmt, int lo, int hi) {
  std::vector<uint8_t> w13, w2, sf13, sf2;
  std::vector<float> s13, s2;
  for (int e = lo; e <= hi; ++e) {
    const ExpertHost x = make_expert(fmt, e == hi ? kExperts : e);
    w13.insert(w13.end(), x.w13.begin(), x.w13.end());
    w2.insert(w2.end(), x.w2.begin(), x.w2.end());
    sf13.insert(sf13.end(), x.sf13.begin(), x.sf13.end());
    sf2.insert(sf2.end(), x.sf2.begin(), x.sf2.end());
    s13.insert(s13.end(), x.s13.begin(), x.s13.end());
    s2.insert(s2.end(), x.s2.begin(), x.s2.end());
  }
  ExpertDev d{upload(w13), upload(w2), nullptr, nullptr};
  if (fmt == AFDK_FFN_MX) {
    d.s13 = upload(sf13);
    d.s2 = upload(sf2);
  } else if (fmt == AFDK_FFN_FP8) {
    d.s13 = upload(s13);
    d.s2 = upload(s2);
  }
  return d;
}

// ---------------------------------------------------------- attention side
struct AttnHost {
  void *in_norm, *qkv, *q_norm, *q_up, *o, *post_norm, *gate;
  afdk_mfa_weights w;
};

AttnHost make_attn() {
  Rng g(7);
  AttnHost a;
  a.in_norm = upload(randn_bf16(g, kHidden, 0.1f, 1.f));
  a.qkv = upload(randn_bf16(g, (size_t)(kQLora + 2 * kHeadDim) * kHidden, 1.f / std::sqrt((float)kHidden)));
  a.q_norm = upload(randn_bf16(g, kQLora, 0.1f, 1.f));
  a.q_up = upload(randn_bf16(g, (size_t)kHeads * kHeadDim * kQLora, 1.f / std::sqrt((float)kQLora)));
  a.o = upload(randn_bf16(g, (size_t)kHidden * kHeads * kHeadDim, 1.f / std::sqrt((float)kHeads * kHeadDim)));
  a.post_norm = upload(randn_bf16(g, kHidden, 0.1f, 1.f));
  a.gate = upload(randn_bf16(g, (size_t)kExperts * kHidden, 1.f / std::sqrt((float)kHidden)));
  a.w = afdk_mfa_weights{kHidden, kQLora, kHeads, kHeadDim, a.in_norm, a.qkv, a.q_norm, a.q_up, a.o,
                         a.post_norm, 1e-5f, 5e5f, 1.f / std::sqrt((float)kHeadDim)};
  return a;
}

struct Kv {  // one (layer, micro-batch) cache
  void *k, *v;
  int32_t* bt;
  int num_pages, max_pages;
};

Kv make_kv(Rng& g) {
  const int pages = (kCtx + kPage - 1) / kPage, n = kTmb * pages;
  Kv kv;
  kv.k = upload(randn_bf16(g, (size_t)n * kPage * kHeadDim, 1.f));
  kv.v = upload(randn_bf16(g, (size_t)n * kPage * kHeadDim, 1.f));
  std::vector<int32_t> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int i = n - 1; i > 0; --i) std::swap(perm[i], perm[g.next() % (i + 1)]);  // scattered pages
  kv.bt = static_cast<int32_t*>(upload(perm));
  kv.num_pages = n;
  kv.max_pages = pages;
  return kv;
}

// one layer of one micro-batch on this GPU, without disaggregation
void recompute_layer(afdk_ctx* ctx, const AttnHost& a, const ExpertDev& all, int fmt, const Kv& kv,
                     const int32_t* seq_lens, void* x, void* h_res, void* h_norm, int32_t* ids, float* wts, void* xq,
                     void* xs, void* part, void** parts_dev) {
  afdk_mfa_layer_args la{kTmb, x, kv.k, kv.v, kv.num_pages, kPage, kv.bt, kv.max_pages, seq_lens, h_res, h_norm};
  AK(afdk_mfa_layer(ctx, &a.w, &la, nullptr));
  if (fmt == AFDK_FFN_FP8) {
    AK(afdk_router_topk(ctx, h_norm, a.gate, kTmb, kHidden, kExperts, kTopK, 0, nullptr, ids, wts, xq,
                        static_cast<float*>(xs), nullptr));
    afdk_moe_weights mw{kHidden, kInter, kExperts, kTopK, 0, kExperts, all.w13, static_cast<const float*>(all.s13),
                        all.w2, static_cast<const float*>(all.s2)};
    afdk_moe_args ma{kTmb, xq, static_cast<const float*>(xs), ids, wts, 0, kTmb, part};
    AK(afdk_moe_ffn(ctx, &mw, &ma, nullptr));
  } else if (fmt == AFDK_FFN_MX) {
    AK(afdk_router_topk(ctx, h_norm, a.gate, kTmb, kHidden, kExperts, kTopK, 0, nullptr, ids, wts, nullptr,
                        nullptr, nullptr));
    AK(afdk_quant_mx(ctx, h_norm, kTmb, kHidden, xq, static_cast<uint8_t*>(xs), nullptr));
    afdk_moe_mx_weights mw{kHidden, kInter, kExperts, kTopK, 0, kExperts, all.w13,
                           static_cast<const uint8_t*>(all.s13), all.w2, static_cast<const uint8_t*>(all.s2)};
    afdk_moe_mx_args ma{kTmb, xq, static_cast<const uint8_t*>(xs), ids, wts, 0, kTmb, part};
    AK(afdk_moe_ffn_mx(ctx, &mw, &ma, nullptr));
  } else {
    AK(afdk_router_topk(ctx, h_norm, a.gate, kTmb, kHidden, kExperts, kTopK, 0, nullptr, ids, wts, nullptr,
                        nullptr, nullptr));
    afdk_moe_bf16_weights mw{kHidden, kInter, kExperts, kTopK, 0, kExperts, all.w13, all.w2};
    afdk_moe_bf16_args ma{kTmb, h_norm, ids, wts, 0, kTmb, part};
    AK(afdk_moe_ffn_bf16(ctx, &mw, &ma, nullptr));
  }
  AK(afdk_add_partials(ctx, h_res, const_cast<const void* const*>(parts_dev), 1, (size_t)kTmb * kHidden, x,
                       nullptr));
}

int run_rank(int rank, int world, int n_attn, int fmt, int f2a, int steps, const std::string& dir,
             double* max_err_out) {
  g_rank = rank;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const int dev = rank % ndev;
  CK(cudaSetDevice(dev));
  const int n_ffn = world - n_attn;
  const bool attn = rank < n_attn;

  afdk_cfg cc{dev, 0};
  afdk_ctx* ctxs[kMicro];
  for (auto& c : ctxs) AK(afdk_create(&c, &cc));
  afdk_afd_cfg cfg{n_attn, n_ffn, kMicro, kTmb, kHidden, kTopK, kExperts, kInter, 0, 0, fmt, AFDK_LAYER_MOE, f2a, 256};
  AK(afdk_afd_check_cfg(&cfg));

  // caller-owned data
  AttnHost aw{};
  std::vector<std::vector<Kv>> kv;  // [layer][mb]
  std::vector<void*> x(kMicro);
  int32_t* seq_lens = nullptr;
  ExpertDev shard{}, all{};
  if (attn) {
    aw = make_attn();
    Rng g(100 + rank);
    for (int l = 0; l < kLayers; ++l) {
      kv.emplace_back();
      for (int m = 0; m < kMicro; ++m) kv[l].push_back(make_kv(g));
    }
    for (int m = 0; m < kMicro; ++m) x[m] = upload(randn_bf16(g, (size_t)kTmb * kHidden, 1.f));
    seq_lens = static_cast<int32_t*>(upload(std::vector<int32_t>(kTmb, kCtx)));
    all = upload_experts(fmt, 0, kExperts);  // for the recompute only
  } else {
    const int f = rank - n_attn;
    shard = upload_experts(fmt, f * kExperts / n_ffn, (f + 1) * kExperts / n_ffn);
  }
  CK(cudaDeviceSynchronize());

  FileGather fg{dir, rank, world};
  afdk_afd* afd = nullptr;
  AK(afdk_afd_create(ctxs, &cfg, rank, file_allgather, &fg, &afd));

  // recompute scratch (attention ranks)
  const size_t act = (size_t)kTmb * kHidden * 2;
  void *xr = nullptr, *h_res = nullptr, *h_norm = nullptr, *xq = nullptr, *xs = nullptr, *part = nullptr;
  int32_t* ids = nullptr;
  float* wts = nullptr;
  void** parts_dev = nullptr;
  if (attn) {
    xr = dalloc(act);
    h_res = dalloc(act);
    h_norm = dalloc(act);
    part = dalloc(act);
    xq = dalloc((size_t)kTmb * kHidden);
    xs = dalloc((size_t)kTmb * (kHidden / 32) * 4);
    ids = static_cast<int32_t*>(dalloc((size_t)kTmb * kTopK * 4));
    wts = static_cast<float*>(dalloc((size_t)kTmb * kTopK * 4));
    parts_dev = static_cast<void**>(upload(std::vector<void*>{part}));
  }

  std::vector<std::vector<void*>> snap(kLayers, std::vector<void*>(kMicro, nullptr));  // [layer][mb]
  if (attn)
    for (auto& l : snap)
      for (auto& p : l) p = dalloc(act);
  double max_err = 0.0;
  std::vector<uint16_t> got(kTmb * kHidden), ref(kTmb * kHidden);
  for (int s = 0; s < steps; ++s) {
    std::vector<std::vector<uint16_t>> x_in(kMicro, std::vector<uint16_t>(kTmb * kHidden));
    if (attn)
      for (int m = 0; m < kMicro; ++m) CK(cudaMemcpy(x_in[m].data(), x[m], act, cudaMemcpyDeviceToHost));
    for (int l = 0; l < kLayers; ++l) {
      if (attn) {
        afdk_afd_attn_mb mbs[kMicro];
        for (int m = 0; m < kMicro; ++m)
          mbs[m] = afdk_afd_attn_mb{x[m], kv[l][m].k, kv[l][m].v, kv[l][m].num_pages, kPage, kv[l][m].max_pages,
                                    kv[l][m].bt, seq_lens, 0.f, 0.f};
        AK(afdk_afd_attn_layer(afd, &aw.w, aw.gate, mbs));
        for (int m = 0; m < kMicro; ++m)  // this layer's output, ordered before the next layer's ATTN
          CK(cudaMemcpyAsync(snap[l][m], x[m], act, cudaMemcpyDeviceToDevice,
                             static_cast<cudaStream_t>(afdk_afd_stream(afd, m))));
      } else {
        afdk_afd_ffn_weights fw{shard.w13, shard.s13, shard.w2, shard.s2};
        AK(afdk_afd_ffn_layer(afd, &fw));
      }
    }
    AK(afdk_afd_sync(afd));
    if (!attn) continue;
    for (int m = 0; m < kMicro; ++m)
      for (int l = 0; l < kLayers; ++l) {
        if (l == 0)
          CK(cudaMemcpy(xr, x_in[m].data(), act, cudaMemcpyHostToDevice));
        else
          CK(cudaMemcpy(xr, snap[l - 1][m], act, cudaMemcpyDeviceToDevice));
        recompute_layer(ctxs[0], aw, all, fmt, kv[l][m], seq_lens, xr, h_res, h_norm, ids, wts, xq, xs, part,
                        parts_dev);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(got.data(), snap[l][m], act, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ref.data(), xr, act, cudaMemcpyDeviceToHost));
        double amax = 0.0, dmax = 0.0;
        bool finite = true;
        for (size_t i = 0; i < got.size(); ++i) {
          const double r = bf16_to_f(ref[i]), v = bf16_to_f(got[i]);
          finite = finite && std::isfinite(v) && std::isfinite(r);
          amax = std::max(amax, std::fabs(r));
          dmax = std::max(dmax, std::fabs(v - r));
        }
        const double err = finite ? dmax / std::max(amax, 1e-12) : 1e30;
        max_err = std::max(max_err, err);
      }
  }
  // every rank idle before anyone unmaps: one more rendezvous round
  int token = 0;
  std::vector<int> tokens(world);
  if (file_allgather(&fg, &token, sizeof token, tokens.data()) != 0) return 5;
  afdk_afd_destroy(afd);
  for (auto& c : ctxs) afdk_destroy(c);
  *max_err_out = max_err;
  return max_err <= 2e-2 ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s <world> <n_attn> <fp8|mx|bf16> <push|pull> [steps]\n", argv[0]);
    return 2;
  }
  const int world = std::atoi(argv[1]), n_attn = std::atoi(argv[2]);
  const std::string fs = argv[3], ts = argv[4];
  const int steps = argc > 5 ? std::atoi(argv[5]) : 2;
  const int fmt = fs == "fp8" ? AFDK_FFN_FP8 : fs == "mx" ? AFDK_FFN_MX : fs == "bf16" ? AFDK_FFN_BF16 : -1;
  const int f2a = ts == "push" ? AFDK_F2A_PUSH : ts == "pull" ? AFDK_F2A_PULL : -1;
  if (world < 2 || n_attn < 1 || n_attn >= world || fmt < 0 || f2a < 0 || steps < 1) {
    std::fprintf(stderr, "bad arguments\n");
    return 2;
  }
  char tmpl[] = "/tmp/afd_cpp_demo.XXXXXX";
  if (!mkdtemp(tmpl)) return 2;
  const std::string dir = tmpl;
  char errdir[512];
  std::snprintf(errdir, sizeof errdir, "%s/err", dir.c_str());
  mkdir(errdir, 0700);

  // fork BEFORE any CUDA call: every rank initialises its own CUDA state
  std::vector<pid_t> kids;
  for (int r = 0; r < world; ++r) {
    const pid_t p = fork();
    if (p == 0) {
      double err = -1.0;
      const int rc = run_rank(r, world, n_attn, fmt, f2a, steps, dir, &err);
      char path[600];
      std::snprintf(path, sizeof path, "%s/r%d", errdir, r);
      if (FILE* f = std::fopen(path, "w")) {
        std::fprintf(f, "%d %.6e\n", rc, err);
        std::fclose(f);
      }
      std::_Exit(rc);
    }
    kids.push_back(p);
  }
  bool ok = true;
  for (pid_t p : kids) {
    int st = 0;
    waitpid(p, &st, 0);
    ok = ok && WIFEXITED(st) && WEXITSTATUS(st) == 0;
  }
  double max_err = 0.0;
  std::string errs;
  for (int r = 0; r < n_attn; ++r) {
    char path[600];
    std::snprintf(path, sizeof path, "%s/r%d", errdir, r);
    int rc = -1;
    double e = -1.0;
    if (FILE* f = std::fopen(path, "r")) {
      if (std::fscanf(f, "%d %lf", &rc, &e) != 2) rc = -1;
      std::fclose(f);
    }
    ok = ok && rc == 0;
    max_err = std::max(max_err, e);
    errs += (r ? ", " : "") + std::to_string(e);
  }
  std::printf(
      "{\"afd_cpp_demo\": \"%s\", \"world\": %d, \"n_attn\": %d, \"fmt\": \"%s\", \"f2a\": \"%s\", \"steps\": %d, "
      "\"layers\": %d, \"T_mb\": %d, \"max_rel_err\": %.3e, \"rel_err_per_attn_rank\": [%s]}\n",
      ok ? "ok" : "FAIL", world, n_attn, fs.c_str(), ts.c_str(), steps, kLayers, kTmb, max_err, errs.c_str());
  std::string rm = "rm -rf '" + dir + "'";
  if (std::system(rm.c_str()) != 0) return ok ? 0 : 1;
  return ok ? 0 : 1;
}
