// stage_times_ref_demo.cpp — the drop-in proof: compiled against the
// REFERENCE's own headers (-DAFD_B200_USE_REFERENCE_HEADERS
// -I/root/reference/proj/include) and linked against the reference's own
// library (oracle/_ref/libafdref.so, built from proj/src in place) plus
// libafdk.so.  A reference user's code path:
//   model = afd::builtin_catalog().model("step3")   (reference catalog)
//   st    = afd::measure_stage_times(model, plan, w, cat)   (B200, measured)
//   afd::simulate(st, plan)  / afd::analytic_tpot_bound(st, plan)  (REFERENCE)
// and, beside it, the reference's analytic derive_stage_times on the same
// plan.  Prints one JSON line; the GPU test checks the reference's simulate
// and the product's pipeline model agree bit for bit on the measured times.
//   usage: stage_times_ref_demo <attn_gpus> <ffn_gpus> <micro_batch> <avg_ctx> <n_micro>
#include <cstdio>
#include <cstdlib>

#include "afd_b200.hpp"
#include "afdsim/catalog.hpp"

int main(int argc, char** argv) {
  const int na = argc > 1 ? std::atoi(argv[1]) : 2;
  const int nf = argc > 2 ? std::atoi(argv[2]) : 6;
  const long long mb = argc > 3 ? std::atoll(argv[3]) : 256;
  const long long ctx = argc > 4 ? std::atoll(argv[4]) : 4096;
  const int n_micro = argc > 5 ? std::atoi(argv[5]) : 3;
  try {
    afd::Catalog cat = afd::builtin_catalog();
    const afd::ModelSpec& m = cat.model("step3");
    afd::AcceleratorSpec b200;  // one GPU per instance; datasheet rates for the analytic side
    b200.name = "B200";
    b200.flops_16bit = 2.25e15;
    b200.flops_8bit = 4.5e15;
    b200.mem_bw = 8e12;
    b200.net_bw_per_server = 9e11;
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
    const afd::StageTimes measured = afd::measure_stage_times(m, p, w, cat);  // B200 provider
    const afd::SimResult ref_sim = afd::simulate(measured, p);                // reference pipesim.cpp
    const double ref_bound = afd::analytic_tpot_bound(measured, p);          // reference pipesim.cpp
    const afd::SimResult our_sim = afd::b200::simulate(measured, p);         // product pipeline model
    const afd::StageTimes analytic = afd::derive_stage_times(m, p, w, cat);  // reference roofline model
    const afd::SimResult ana_sim = afd::simulate(analytic, p);
    std::printf(
        "{\"plan\": \"%dA%dF\", \"model\": \"%s\", \"layers\": %d, \"micro_batch\": %lld, \"n_micro\": %d, "
        "\"attn_us\": %.3f, \"ffn_moe_us\": %.3f, \"ffn_dense_us\": %.3f, \"comm_fwd_us\": %.3f, \"comm_bwd_us\": %.3f, "
        "\"ref_simulate_tpot_ms\": %.9f, \"ref_simulate_tgs\": %.6f, \"ref_tpot_bound_ms\": %.9f, "
        "\"product_simulate_tpot_ms\": %.9f, \"product_simulate_tgs\": %.6f, "
        "\"analytic_tpot_ms\": %.9f, \"analytic_attn_us\": %.3f, \"analytic_ffn_us\": %.3f}\n",
        na, nf, m.name.c_str(), measured.layers(), mb, n_micro, 1e6 * measured.attn[10], 1e6 * measured.ffn[10],
        1e6 * measured.ffn[0], 1e6 * measured.comm_fwd[10], 1e6 * measured.comm_bwd[10], 1e3 * ref_sim.tpot,
        ref_sim.tgs, 1e3 * ref_bound, 1e3 * our_sim.tpot, our_sim.tgs, 1e3 * ana_sim.tpot, 1e6 * analytic.attn[10],
        1e6 * analytic.ffn[10]);
  } catch (const afd::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
