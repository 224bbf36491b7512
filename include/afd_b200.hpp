// afd_b200.hpp — C++ host API of the B200 Step-3 decode hot path.
//
// Drop-in for the reference's operator API (proj/include/afdsim): the
// reference maps the path onto per-layer times ANALYTICALLY with
//   StageTimes derive_stage_times(const ModelSpec&, const DeploymentPlan&,
//                                 const Workload&, const Catalog&);
// (pipesim.hpp:28-29, pipesim.cpp:59-127).  measure_stage_times below has the
// identical parameter list and fills the same StageTimes by RUNNING the
// layer on B200: the attention tier's layer (afdk_mfa_layer + router/FP8
// dispatch) at the plan's per-GPU batch and context, the FFN tier's MoE (or
// dense) layer at the plan's expert shard and token count, and the A->F /
// F->A NVLink transfers.  Everything downstream in the reference —
// simulate(), analytic_tpot_bound(), vet_plan() — consumes it unchanged.
//
// Below it sit thin RAII/exception wrappers (afd::ops) over the C-ABI
// include/afdk.h, mapping AFDK_ERR_INVALID to afd::SpecError and every other
// failure to afd::Error like the reference's error convention (types.hpp:12-25).
#pragma once

#ifdef AFD_B200_USE_REFERENCE_HEADERS
#include "afdsim/pipesim.hpp"
#include "afdsim/plan.hpp"
#include "afdsim/types.hpp"
#else
#include "afd_compat.hpp"
#endif

#include <cstdint>
#include <string>

#include "afdk.h"

namespace afd {

// Measured provider, same signature as derive_stage_times (pipesim.hpp:28).
// Results are cached per (shape, workload); the first call for a shape runs
// kernels on the current CUDA device, later calls are pure lookups (safe to
// call from the planner's OpenMP loop once warmed).
// Supports the Step-3 geometry (MFA 64x256, hidden from the model card) on
// an sm_100 device; throws SpecError otherwise.  Formats follow the model
// card's QuantScheme (types.hpp:34-40): weight_bytes 1 -> MXFP8 experts,
// 2 -> bf16 experts; kv_store_bytes 1 -> e4m3 KV cache, 2 -> bf16.
StageTimes measure_stage_times(const ModelSpec& model, const DeploymentPlan& plan, const Workload& w,
                               const Catalog& catalog);

namespace b200 {

struct LayerMeasurement {
  double attn_s = 0, moe_ffn_s = 0, dense_ffn_s = 0, comm_fwd_s = 0, comm_bwd_s = 0;
  std::int64_t attn_batch = 0;   // requests per attention GPU per micro-batch
  std::int64_t ffn_tokens = 0;   // tokens per FFN GPU per micro-batch
  int local_experts = 0;
  double link_gbs = 0;           // per-direction NVLink bandwidth used for comm
  std::string link_source;       // "measured peer DMA of the payload" or the pool figure
};

// The measurement behind measure_stage_times (exposed for reporting).
LayerMeasurement measure_layer(const ModelSpec& model, const DeploymentPlan& plan, const Workload& w,
                               const Catalog& catalog);
void clear_measurement_cache();

// vet_plan's stage_ok (planner.cpp:124-131) evaluated on any StageTimes —
// measured ones in particular: every layer's attention and FFN time within
// stage_budget(w, model) = tpot_sla / pipeline_stages / n_layers
// (sizing.cpp:9-11).
struct StageCheck {
  bool stage_ok = true;
  int first_bad_layer = -1;
  double budget = 0, worst_attn = 0, worst_ffn = 0;
};
StageCheck vet_stages(const StageTimes& times, const Workload& w, const ModelSpec& model);

// Pipeline model on measured times (semantics of pipesim.cpp:155-237).
SimResult simulate(const StageTimes& times, const DeploymentPlan& plan, const SimOptions& opts = {});
std::string trace_csv(const SimResult& result);

}  // namespace b200

namespace ops {

inline void check(afdk_status s) {
  if (s == AFDK_OK) return;
  if (s == AFDK_ERR_INVALID) throw SpecError(afdk_last_error());
  throw Error(afdk_last_error());
}

class Context {
 public:
  explicit Context(int device = 0, int num_sms = 0) {
    afdk_cfg cfg{device, num_sms};
    check(afdk_create(&ctx_, &cfg));
  }
  ~Context() { afdk_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  afdk_ctx* get() const { return ctx_; }

 private:
  afdk_ctx* ctx_ = nullptr;
};

inline void mfa_decode(Context& c, const afdk_mfa_decode_args& a, void* stream = nullptr) {
  check(afdk_mfa_decode_attention(c.get(), &a, stream));
}
inline void mfa_layer(Context& c, const afdk_mfa_weights& w, const afdk_mfa_layer_args& a, void* stream = nullptr) {
  check(afdk_mfa_layer(c.get(), &w, &a, stream));
}
inline void moe_ffn(Context& c, const afdk_moe_weights& w, const afdk_moe_args& a, void* stream = nullptr) {
  check(afdk_moe_ffn(c.get(), &w, &a, stream));
}

}  // namespace ops
}  // namespace afd
