// stage_times_demo.cpp — the C++ host path a reference user takes: build the
// Step-3 model card and an nA-mF plan with the reference's value types,
// get MEASURED per-layer stage times from the B200 provider (same signature as
// derive_stage_times, pipesim.hpp:28) and run the pipeline model on them.
//   usage: stage_times_demo <attn_gpus> <ffn_gpus> <micro_batch> <avg_ctx> <n_micro>
// prints one JSON line.
#include <cstdio>
#include <cstdlib>

#include "afd_b200.hpp"

int main(int argc, char** argv) {
  const int na = argc > 1 ? std::atoi(argv[1]) : 2;
  const int nf = argc > 2 ? std::atoi(argv[2]) : 6;
  const long long mb = argc > 3 ? std::atoll(argv[3]) : 256;
  const long long ctx = argc > 4 ? std::atoll(argv[4]) : 4096;
  const int n_micro = argc > 5 ? std::atoi(argv[5]) : 3;

  // Step-3 model card (builtin_catalog.cpp:232-255) and a one-GPU-per-instance B200 entry
  afd::ModelSpec m;
  m.name = "step3";
  m.n_layers = 61;
  m.hidden_dim = 7168;
  afd::AttentionLayerGroup g;
  g.layer_count = 61;
  g.n_q_heads = 64;
  g.qk_dim = 256;
  g.v_dim = 256;
  g.kv_token_bytes = 512;
  m.attention_groups.push_back(g);
  afd::Catalog cat;
  afd::AcceleratorSpec b200;
  b200.name = "B200";
  b200.gpus_per_server = 1;
  cat.accelerators.push_back(b200);
  afd::DeploymentPlan p;
  p.attn_hw = p.ffn_hw = "B200";
  p.attn_instances = na;
  p.ffn_instances = nf;
  p.micro_batch = mb;
  p.n_micro = n_micro;
  p.total_batch = mb * n_micro;
  p.total_gpus = na + nf;
  afd::Workload w;
  w.avg_ctx = ctx;
  try {
    const afd::StageTimes st = afd::measure_stage_times(m, p, w, cat);
    const auto lm = afd::b200::measure_layer(m, p, w, cat);  // cached: no second run
    const afd::SimResult r = afd::b200::simulate(st, p);
    std::printf(
        "{\"plan\": \"%dA%dF\", \"micro_batch\": %lld, \"n_micro\": %d, \"ctx\": %lld, \"attn_us\": %.3f, "
        "\"moe_ffn_us\": %.3f, \"dense_ffn_us\": %.3f, \"comm_fwd_us\": %.3f, \"comm_bwd_us\": %.3f, "
        "\"link_gbs\": %.1f, \"link_source\": \"%s\", \"tpot_ms\": %.4f, \"tgs\": %.1f, "
        "\"util\": [%.3f, %.3f, %.3f, %.3f]}\n",
        na, nf, mb, n_micro, ctx, 1e6 * lm.attn_s, 1e6 * lm.moe_ffn_s, 1e6 * lm.dense_ffn_s, 1e6 * lm.comm_fwd_s,
        1e6 * lm.comm_bwd_s, lm.link_gbs, lm.link_source.c_str(), 1e3 * r.tpot, r.tgs, r.utilization[0],
        r.utilization[1], r.utilization[2], r.utilization[3]);
  } catch (const afd::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
