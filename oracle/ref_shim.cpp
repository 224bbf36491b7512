// ref_shim.cpp — extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (the accounting oracle).  oracle/Makefile compiles
// this file together with the reference's own sources, read in place from
// /root/reference/proj/src (never copied), into oracle/_ref/libafdref.so.
// Python tests load it with ctypes to pin:
//   * the oracle's byte/FLOP accounting  (costmodel.cpp:46-79, moeplan.cpp:7-20)
//   * the product's StageTimes/simulate  (pipesim.cpp:59-237)
// Nothing in the product links this library.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "afdsim/catalog.hpp"
#include "afdsim/costmodel.hpp"
#include "afdsim/moeplan.hpp"
#include "afdsim/pipesim.hpp"
#include "afdsim/planner.hpp"
#include "afdsim/sizing.hpp"

namespace {

thread_local std::string g_err;

afd::AcceleratorSpec make_accel(const char* name, double f16, double f8, double bw,
                                double net, int gps, double net_eff) {
  afd::AcceleratorSpec a;
  a.name = name;
  a.flops_16bit = f16;
  if (f8 > 0) a.flops_8bit = f8;
  a.mem_bw = bw;
  a.net_bw_per_server = net;
  a.gpus_per_server = gps;
  a.net_efficiency = net_eff;
  return a;
}

afd::Workload make_workload(long long ctx, double kvq, double mtp) {
  afd::Workload w;
  w.avg_ctx = ctx;
  w.kv_quant_factor = kvq;
  w.mtp_factor = mtp;
  return w;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Step-3 (or any builtin) model card fields the kernels are shaped by.
// out: n_layers, hidden, n_q_heads, qk_dim, v_dim, kv_token_bytes,
//      attn_linear_params, ffn_activated_params, ffn_total_weight_bytes
int ref_model_card(const char* model, long long out[9]) {
  return guarded([&] {
    const auto cat = afd::builtin_catalog();
    const auto& m = cat.model(model);
    const auto& g = m.attention_groups.front();
    long long v[9] = {m.n_layers, m.hidden_dim, g.n_q_heads, g.qk_dim, g.v_dim,
                      (long long)g.kv_token_bytes, (long long)m.attn_linear_params,
                      (long long)m.ffn_activated_params,
                      (long long)m.ffn_total_weight_bytes};
    std::memcpy(out, v, sizeof(v));
  });
}

int ref_cost_breakdown(const char* model, long long ctx, double kvq, double mtp,
                       double out[4]) {
  return guarded([&] {
    const auto cat = afd::builtin_catalog();
    const auto c = afd::cost_breakdown(cat.model(model), make_workload(ctx, kvq, mtp));
    out[0] = c.kv_state_bytes;
    out[1] = c.attn_core_flops;
    out[2] = c.attn_linear_flops;
    out[3] = c.ffn_flops;
  });
}

int ref_ffn_net_bytes(const char* model, long long batch, double* out) {
  return guarded([&] {
    const auto cat = afd::builtin_catalog();
    *out = afd::ffn_net_bytes(cat.model(model), batch);
  });
}

int ref_b_dense_moe(const char* model, double f16, double f8, double bw, long long out[3]) {
  return guarded([&] {
    const auto cat = afd::builtin_catalog();
    const auto a = make_accel("X", f16, f8, bw, 1e11, 8, 1.0);
    out[0] = afd::b_dense(a, afd::ComputeKind::eight_bit);
    out[1] = afd::b_dense(a, afd::ComputeKind::sixteen_bit);
    out[2] = afd::b_moe(a, cat.model(model));
  });
}

int ref_stage_budget(double tpot, int stages, int layers, double* out) {
  return guarded([&] {
    afd::Workload w;
    w.tpot_sla = tpot;
    w.pipeline_stages = stages;
    afd::ModelSpec m = afd::builtin_catalog().model("step3");
    m.n_layers = layers;
    *out = afd::stage_budget(w, m);
  });
}

// derive_stage_times for `model` on one accelerator used for both tiers.
int ref_derive_stage_times(const char* model, const char* hw, double f16, double f8,
                           double bw, double net, int gps, double net_eff,
                           int attn_inst, int ffn_inst, long long micro_batch,
                           int n_micro, long long ctx, double* attn, double* fwd,
                           double* ffn, double* bwd, int L) {
  return guarded([&] {
    auto cat = afd::builtin_catalog();
    cat.accelerators.push_back(make_accel(hw, f16, f8, bw, net, gps, net_eff));
    afd::DeploymentPlan p;
    p.attn_hw = hw;
    p.ffn_hw = hw;
    p.attn_instances = attn_inst;
    p.ffn_instances = ffn_inst;
    p.micro_batch = micro_batch;
    p.n_micro = n_micro;
    p.total_batch = micro_batch * n_micro;
    p.total_gpus = (attn_inst + ffn_inst) * gps;
    afd::Workload w;
    w.avg_ctx = ctx;
    const auto st = afd::derive_stage_times(cat.model(model), p, w, cat);
    if (st.layers() != L) throw afd::Error("layer count mismatch");
    for (int l = 0; l < L; ++l) {
      attn[l] = st.attn[l];
      fwd[l] = st.comm_fwd[l];
      ffn[l] = st.ffn[l];
      bwd[l] = st.comm_bwd[l];
    }
  });
}

int ref_simulate(const double* attn, const double* fwd, const double* ffn,
                 const double* bwd, int L, int n_micro, long long total_batch,
                 int total_gpus, int token_steps, int shared_link, double out[10]) {
  return guarded([&] {
    afd::StageTimes st;
    st.attn.assign(attn, attn + L);
    st.comm_fwd.assign(fwd, fwd + L);
    st.ffn.assign(ffn, ffn + L);
    st.comm_bwd.assign(bwd, bwd + L);
    afd::DeploymentPlan p;
    p.n_micro = n_micro;
    p.total_batch = total_batch;
    p.total_gpus = total_gpus;
    afd::SimOptions o;
    o.token_steps = token_steps;
    o.shared_link = shared_link != 0;
    const auto r = afd::simulate(st, p, o);
    out[0] = r.tpot;
    out[1] = r.tgs;
    for (int i = 0; i < 4; ++i) out[2 + i] = r.utilization[i];
    for (int i = 0; i < 4; ++i) out[6 + i] = r.bubble_fraction[i];
  });
}

int ref_analytic_tpot_bound(const double* attn, const double* fwd, const double* ffn,
                            const double* bwd, int L, int n_micro, double* out) {
  return guarded([&] {
    afd::StageTimes st;
    st.attn.assign(attn, attn + L);
    st.comm_fwd.assign(fwd, fwd + L);
    st.ffn.assign(ffn, ffn + L);
    st.comm_bwd.assign(bwd, bwd + L);
    afd::DeploymentPlan p;
    p.n_micro = n_micro;
    *out = afd::analytic_tpot_bound(st, p);
  });
}

// trace_csv of a simulated run (byte-stable text; caller frees with ref_free)
char* ref_trace_csv(const double* attn, const double* fwd, const double* ffn,
                    const double* bwd, int L, int n_micro, long long total_batch,
                    int total_gpus) {
  char* res = nullptr;
  guarded([&] {
    afd::StageTimes st;
    st.attn.assign(attn, attn + L);
    st.comm_fwd.assign(fwd, fwd + L);
    st.ffn.assign(ffn, ffn + L);
    st.comm_bwd.assign(bwd, bwd + L);
    afd::DeploymentPlan p;
    p.n_micro = n_micro;
    p.total_batch = total_batch;
    p.total_gpus = total_gpus;
    const std::string s = afd::trace_csv(afd::simulate(st, p));
    res = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(res, s.c_str(), s.size() + 1);
  });
  return res;
}

// vet_plan (planner.cpp:111-137) of an AFD plan on one accelerator used for
// both tiers; flags = {sparsity_ok, net_ok, stage_ok}
int ref_vet_plan(const char* model, const char* hw, double f16, double f8, double bw, double net, int gps,
                 double net_eff, int attn_inst, int ffn_inst, long long micro_batch, int n_micro, long long ctx,
                 double tpot, int stages, int flags[3]) {
  return guarded([&] {
    auto cat = afd::builtin_catalog();
    cat.accelerators.push_back(make_accel(hw, f16, f8, bw, net, gps, net_eff));
    afd::DeploymentPlan p;
    p.attn_hw = hw;
    p.ffn_hw = hw;
    p.attn_instances = attn_inst;
    p.ffn_instances = ffn_inst;
    p.micro_batch = micro_batch;
    p.n_micro = n_micro;
    p.total_batch = micro_batch * n_micro;
    p.total_gpus = (attn_inst + ffn_inst) * gps;
    afd::Workload w;
    w.avg_ctx = ctx;
    w.tpot_sla = tpot;
    w.pipeline_stages = stages;
    const auto f = afd::vet_plan(p, cat.model(model), w, cat);
    flags[0] = f.sparsity_ok;
    flags[1] = f.net_ok;
    flags[2] = f.stage_ok;
  });
}

// the builtin catalog in the reference's own TOML schema (dump_catalog)
char* ref_dump_builtin_catalog() {
  char* res = nullptr;
  guarded([&] {
    const std::string t = afd::dump_catalog(afd::builtin_catalog());
    res = static_cast<char*>(std::malloc(t.size() + 1));
    std::memcpy(res, t.c_str(), t.size() + 1);
  });
  return res;
}

// parse a catalog text with the reference's loader (parse_catalog validates
// every entry) and return accelerator `name`'s fields:
// {flops_16bit, flops_8bit (0 if absent), mem_bw, net_bw_per_server, gpus_per_server, net_efficiency}
int ref_catalog_accel(const char* text, const char* name, double out[6]) {
  return guarded([&] {
    const afd::Catalog cat = afd::parse_catalog(text, "b200_catalog");
    const afd::AcceleratorSpec& a = cat.accelerator(name);
    out[0] = a.flops_16bit;
    out[1] = a.flops_8bit.value_or(0.0);
    out[2] = a.mem_bw;
    out[3] = a.net_bw_per_server;
    out[4] = a.gpus_per_server;
    out[5] = a.net_efficiency;
  });
}

void ref_free(void* p) { std::free(p); }

}  // extern "C"
