// afd_compat.hpp — stand-alone declarations of the afd:: value types the B200
// provider exchanges with the reference planner.
//
// In an integrated build the reference's own headers
// proj/include/afdsim/{types,plan,pipesim}.hpp are used instead and this file
// is not included (define AFD_B200_USE_REFERENCE_HEADERS).  For the
// stand-alone library and its tests it restates, member for member and in the
// same order, the subset the provider touches so objects are layout
// compatible with the reference's:
//   ModelSpec / AttentionLayerGroup / QuantScheme  types.hpp:34-77
//   AcceleratorSpec / Workload / Catalog           types.hpp:79-115
//   DeploymentPlan / PlanFlags / PlanMode          plan.hpp:10-35
//   StageTimes / TraceEvent / SimResult / SimOptions / SimResource
//                                                  pipesim.hpp:14-53
// Member functions are deliberately absent: the provider reads data members
// only, so it links against either definition.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace afd {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : Error {
  using Error::Error;
};
struct SpecError : Error {
  using Error::Error;
};

enum class ComputeKind { eight_bit, sixteen_bit };
enum class AttentionKind { full, windowed, linear_state };

struct QuantScheme {
  int kv_store_bytes = 1;
  int weight_bytes = 1;
  int dispatch_bytes = 1;
  int combine_bytes = 2;
  ComputeKind compute_kind = ComputeKind::eight_bit;
};

struct AttentionLayerGroup {
  AttentionKind kind = AttentionKind::full;
  int layer_count = 0;
  int n_q_heads = 0;
  int qk_dim = 0;
  int v_dim = 0;
  std::int64_t window_len = 0;
  std::int64_t kv_token_bytes = 0;
  std::int64_t const_state_bytes = 0;
  std::int64_t const_flops_per_token = 0;
};

struct ModelSpec {
  std::string name;
  std::int64_t total_params = 0;
  std::int64_t activated_params = 0;
  int n_layers = 0;
  int hidden_dim = 0;
  std::vector<AttentionLayerGroup> attention_groups;
  std::int64_t attn_linear_params = 0;
  std::int64_t ffn_activated_params = 0;
  std::int64_t ffn_total_weight_bytes = 0;
  double moe_sparsity = 1.0;
  QuantScheme quant;
  std::int64_t effective_rank = 0;
};

struct AcceleratorSpec {
  std::string name;
  std::optional<double> price_usd_per_hour;
  double flops_16bit = 0.0;
  std::optional<double> flops_8bit;
  double mem_bw = 0.0;
  double net_bw_per_server = 0.0;
  int gpus_per_server = 8;
  double net_efficiency = 1.0;
};

struct Workload {
  std::int64_t avg_ctx = 8192;
  double tpot_sla = 0.05;
  int pipeline_stages = 3;
  double kv_quant_factor = 1.0;
  double mtp_factor = 1.0;
};

struct Catalog {
  std::vector<ModelSpec> models;
  std::vector<AcceleratorSpec> accelerators;
};

enum class PlanMode { afd, colocated };

struct PlanFlags {
  bool sparsity_ok = false;
  bool net_ok = false;
  bool stage_ok = false;
  bool relies_on_large_ep = false;
};

struct DeploymentPlan {
  std::string attn_hw;
  int attn_instances = 1;
  std::string ffn_hw;
  int ffn_instances = 1;
  std::int64_t micro_batch = 0;
  int n_micro = 3;
  std::int64_t total_batch = 0;
  int total_gpus = 0;
  PlanMode mode = PlanMode::afd;
  PlanFlags flags;
  double predicted_tgs = 0.0;
  double theoretical_usd_per_1m = 0.0;
};

struct StageTimes {
  std::vector<double> attn;
  std::vector<double> comm_fwd;
  std::vector<double> comm_bwd;
  std::vector<double> ffn;
  int layers() const { return static_cast<int>(attn.size()); }
};

enum class SimResource : int { attention = 0, fwd_link = 1, ffn = 2, bwd_link = 3 };

struct TraceEvent {
  double time = 0.0;
  SimResource resource = SimResource::attention;
  int layer = 0;
  int micro_batch = 0;
  double duration = 0.0;
};

struct SimResult {
  double tpot = 0.0;
  double tgs = 0.0;
  std::array<double, 4> utilization{};
  std::array<double, 4> bubble_fraction{};
  std::vector<TraceEvent> trace;
};

struct SimOptions {
  int token_steps = 3;
  bool shared_link = false;
};

}  // namespace afd
