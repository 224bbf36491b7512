// pipeline_model.cpp — the layer-wise AFD pipeline model evaluated on
// MEASURED stage times.
//
// Semantics are the reference's (pipesim.hpp:44-60, pipesim.cpp:155-237):
// four resources (attention, A->F link, FFN, F->A link; the two links are one
// resource when shared_link), each serving its tasks first-come in
// (token step, layer, micro-batch) order; micro-batch b starts layer l+1 only
// after its layer-l output returned and its next token only after layer L.
// tpot is the completion gap between token steps 1 and 0.  This
// implementation is independent of the reference's loop: every resource owns
// an explicit service queue and a sweep advances whichever queue head has its
// input ready.  tests/test_pipeline_model_cpu.py checks it against the
// reference library (oracle/_ref) bit for bit on random instances.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/afd_b200.hpp"

namespace afd {
namespace b200 {

namespace {

struct Task {
  int stage, s, l, b;
};

}  // namespace

SimResult simulate(const StageTimes& t, const DeploymentPlan& plan, const SimOptions& opts) {
  const int L = t.layers();
  const int n = plan.n_micro;
  const int steps = std::max(2, opts.token_steps);
  if (t.comm_fwd.size() != t.attn.size() || t.comm_bwd.size() != t.attn.size() || t.ffn.size() != t.attn.size())
    throw Error("StageTimes arrays must have equal length");
  for (const auto* v : {&t.attn, &t.comm_fwd, &t.comm_bwd, &t.ffn})
    for (double x : *v)
      if (!(x >= 0.0)) throw Error("StageTimes entries must be >= 0");
  if (L == 0) throw Error("simulate: empty stage times");
  if (n < 1) throw Error("simulate: n_micro must be >= 1");
  if (plan.mode != PlanMode::afd) throw Error("simulate models the disaggregated pipeline only");

  const std::vector<double>* dur[4] = {&t.attn, &t.comm_fwd, &t.ffn, &t.comm_bwd};
  const int res_of_stage[4] = {0, 1, 2, opts.shared_link ? 1 : 3};
  const SimResource name_of_stage[4] = {SimResource::attention, SimResource::fwd_link, SimResource::ffn,
                                        SimResource::bwd_link};
  // service queues
  std::vector<Task> queue[4];
  for (int s = 0; s < steps; ++s)
    for (int l = 0; l < L; ++l)
      for (int st = 0; st < 4; ++st)
        for (int b = 0; b < n; ++b) queue[res_of_stage[st]].push_back({st, s, l, b});
  const size_t per_stage = static_cast<size_t>(steps) * L * n;
  auto key = [&](int st, int s, int l, int b) { return st * per_stage + (static_cast<size_t>(s) * L + l) * n + b; };
  std::vector<double> finish(4 * per_stage, -1.0);
  size_t head[4] = {0, 0, 0, 0};
  double free_at[4] = {0.0, 0.0, 0.0, 0.0};
  const int measured = 1;
  std::vector<TraceEvent> trace;
  std::array<double, 4> busy{};

  auto input_ready = [&](const Task& k, double* when) {
    if (k.stage == 0) {
      if (k.l > 0) *when = finish[key(3, k.s, k.l - 1, k.b)];
      else if (k.s > 0) *when = finish[key(3, k.s - 1, L - 1, k.b)];
      else *when = 0.0;
    } else {
      *when = finish[key(k.stage - 1, k.s, k.l, k.b)];
    }
    return *when >= 0.0;
  };

  size_t done = 0;
  const size_t total = 4 * per_stage;
  while (done < total) {
    bool progressed = false;
    for (int r = 0; r < 4; ++r) {
      while (head[r] < queue[r].size()) {
        const Task& k = queue[r][head[r]];
        double ready;
        if (!input_ready(k, &ready)) break;
        const double d = (*dur[k.stage])[k.l];
        const double start = std::max(ready, free_at[r]);
        const double end = start + d;
        free_at[r] = end;
        finish[key(k.stage, k.s, k.l, k.b)] = end;
        if (k.s == measured) {
          busy[static_cast<int>(name_of_stage[k.stage])] += d;
          trace.push_back({start, name_of_stage[k.stage], k.l, k.b, d});
        }
        ++head[r];
        ++done;
        progressed = true;
      }
    }
    if (!progressed) throw Error("simulate: dependency cycle (internal error)");
  }

  auto completion = [&](int s) {
    double c = 0.0;
    for (int b = 0; b < n; ++b) c = std::max(c, finish[key(3, s, L - 1, b)]);
    return c;
  };
  SimResult res;
  res.tpot = completion(measured) - completion(measured - 1);
  if (plan.total_gpus > 0 && res.tpot > 0.0)
    res.tgs = static_cast<double>(plan.total_batch) / (res.tpot * static_cast<double>(plan.total_gpus));
  for (int r = 0; r < 4; ++r) {
    res.utilization[r] = res.tpot > 0.0 ? busy[r] / res.tpot : 0.0;
    res.bubble_fraction[r] = 1.0 - res.utilization[r];
  }
  std::stable_sort(trace.begin(), trace.end(), [](const TraceEvent& a, const TraceEvent& b) {
    if (a.time != b.time) return a.time < b.time;
    if (a.layer != b.layer) return a.layer < b.layer;
    if (a.micro_batch != b.micro_batch) return a.micro_batch < b.micro_batch;
    return static_cast<int>(a.resource) < static_cast<int>(b.resource);
  });
  res.trace = std::move(trace);
  return res;
}

std::string trace_csv(const SimResult& r) {
  static const char* res_name[4] = {"attention", "fwd_link", "ffn", "bwd_link"};
  static const char* stage_name[4] = {"attention", "comm", "ffn", "comm"};
  std::ostringstream os;
  os << "time_s,resource,layer,micro_batch,stage,duration_s\n";
  char a[64], b[64];
  for (const auto& e : r.trace) {
    const int k = static_cast<int>(e.resource);
    std::snprintf(a, sizeof(a), "%.9f", e.time);
    std::snprintf(b, sizeof(b), "%.9f", e.duration);
    os << a << ',' << res_name[k] << ',' << e.layer << ',' << e.micro_batch << ',' << stage_name[k] << ',' << b
       << '\n';
  }
  return os.str();
}

// vet_plan's stage check (planner.cpp:124-131) on any StageTimes: every
// layer's attention and FFN stage must fit stage_budget = tpot_sla /
// pipeline_stages / n_layers (sizing.cpp:9-11).
StageCheck vet_stages(const StageTimes& t, const Workload& w, const ModelSpec& model) {
  if (model.n_layers < 1 || w.pipeline_stages < 1 || !(w.tpot_sla > 0.0))
    throw SpecError("vet_stages: need n_layers >= 1, pipeline_stages >= 1, tpot_sla > 0");
  StageCheck c;
  c.budget = w.tpot_sla / w.pipeline_stages / model.n_layers;
  c.stage_ok = true;
  for (int l = 0; l < t.layers(); ++l) {
    c.worst_attn = std::max(c.worst_attn, t.attn[l]);
    c.worst_ffn = std::max(c.worst_ffn, t.ffn[l]);
    if ((t.attn[l] > c.budget || t.ffn[l] > c.budget) && c.stage_ok) {
      c.stage_ok = false;
      c.first_bad_layer = l;
    }
  }
  return c;
}

}  // namespace b200
}  // namespace afd

static afd::StageTimes stage_times(const double* attn, const double* fwd, const double* ffn, const double* bwd,
                                   int layers) {
  afd::StageTimes st;
  st.attn.assign(attn, attn + layers);
  st.comm_fwd.assign(fwd, fwd + layers);
  st.ffn.assign(ffn, ffn + layers);
  st.comm_bwd.assign(bwd, bwd + layers);
  return st;
}

extern "C" afdk_status afdk_trace_csv(const double* attn, const double* fwd, const double* ffn, const double* bwd,
                                      int layers, const afdk_sim_plan* p, char* buf, size_t cap, size_t* len) {
  if (!attn || !fwd || !ffn || !bwd || !p || !len || layers < 1) return AFDK_ERR_INVALID;
  try {
    afd::DeploymentPlan plan;
    plan.n_micro = p->n_micro;
    plan.total_batch = p->total_batch;
    plan.total_gpus = p->total_gpus;
    afd::SimOptions o;
    o.token_steps = p->token_steps;
    o.shared_link = p->shared_link != 0;
    const std::string csv = afd::b200::trace_csv(afd::b200::simulate(stage_times(attn, fwd, ffn, bwd, layers), plan, o));
    *len = csv.size();
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, csv.size());
      std::memcpy(buf, csv.data(), n);
      buf[n] = '\0';
    }
    return AFDK_OK;
  } catch (const std::exception&) {
    return AFDK_ERR_INVALID;
  }
}

extern "C" afdk_status afdk_vet_stages(const double* attn, const double* ffn, int layers, double tpot_sla,
                                       int pipeline_stages, int n_model_layers, afdk_stage_check* out) {
  if (!attn || !ffn || !out || layers < 1) return AFDK_ERR_INVALID;
  try {
    afd::StageTimes st;
    st.attn.assign(attn, attn + layers);
    st.ffn.assign(ffn, ffn + layers);
    st.comm_fwd.assign(layers, 0.0);
    st.comm_bwd.assign(layers, 0.0);
    afd::Workload w;
    w.tpot_sla = tpot_sla;
    w.pipeline_stages = pipeline_stages;
    afd::ModelSpec m;
    m.n_layers = n_model_layers;
    const afd::b200::StageCheck c = afd::b200::vet_stages(st, w, m);
    out->stage_ok = c.stage_ok ? 1 : 0;
    out->first_bad_layer = c.first_bad_layer;
    out->budget_s = c.budget;
    out->worst_attn_s = c.worst_attn;
    out->worst_ffn_s = c.worst_ffn;
    return AFDK_OK;
  } catch (const std::exception&) {
    return AFDK_ERR_INVALID;
  }
}

extern "C" afdk_status afdk_simulate(const double* attn, const double* fwd, const double* ffn, const double* bwd,
                                     int layers, const afdk_sim_plan* p, afdk_sim_result* out) {
  if (!attn || !fwd || !ffn || !bwd || !p || !out || layers < 1) return AFDK_ERR_INVALID;
  try {
    afd::StageTimes st;
    st.attn.assign(attn, attn + layers);
    st.comm_fwd.assign(fwd, fwd + layers);
    st.ffn.assign(ffn, ffn + layers);
    st.comm_bwd.assign(bwd, bwd + layers);
    afd::DeploymentPlan plan;
    plan.n_micro = p->n_micro;
    plan.total_batch = p->total_batch;
    plan.total_gpus = p->total_gpus;
    afd::SimOptions o;
    o.token_steps = p->token_steps;
    o.shared_link = p->shared_link != 0;
    const auto r = afd::b200::simulate(st, plan, o);
    out->tpot = r.tpot;
    out->tgs = r.tgs;
    for (int i = 0; i < 4; ++i) {
      out->utilization[i] = r.utilization[i];
      out->bubble_fraction[i] = r.bubble_fraction[i];
    }
    return AFDK_OK;
  } catch (const std::exception&) {
    return AFDK_ERR_INVALID;
  }
}
