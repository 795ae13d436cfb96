// rserve-b200 — POD config structs of include/rserve.h <-> lmmsim types.
#pragma once

#include <sstream>
#include <string>
#include <vector>

#include "lmmsim/simengine.hpp"
#include "lmmsim/workload.hpp"
#include "rserve.h"

namespace rserve {

inline lmmsim::SimConfig to_sim_config(const rs_sim_config& c) {
  using namespace lmmsim;
  if (c.policy < RS_POLICY_VANILLA_PP || c.policy > RS_POLICY_RSERVE)
    throw ConfigError("policy: unknown enum value " + std::to_string(c.policy));
  SimConfig s;
  s.policy = static_cast<Policy>(c.policy);
  if (c.pipeline_mode == RS_PIPELINE_CPP) s.pipeline_mode = PipelineMode::Cpp;
  else if (c.pipeline_mode == RS_PIPELINE_VANILLA) s.pipeline_mode = PipelineMode::Vanilla;
  s.stages = c.stages;
  s.encoder_workers = c.encoder_workers;
  s.token_budget = c.token_budget;
  s.embedding_batch_tokens = c.embedding_batch_tokens;
  s.release_at = c.release_at == RS_RELEASE_FIRST_STAGE ? ReleaseAt::FirstStage
                                                        : ReleaseAt::LastStage;
  s.hidden_size = c.hidden_size;
  const rs_cost_model& m = c.cost;
  s.cost = CostModel{m.alpha_enc_ms,   m.beta_enc_ms_per_token,    m.eps_tx_ms,
                     m.zeta_tx_ms_per_token, m.gamma_stage_ms, m.delta_stage_ms_per_token,
                     m.kappa_attn_ms,  m.tp_speedup};
  return s;
}

inline lmmsim::IntDistribution to_distribution(const rs_int_dist& d) {
  return d.uniform ? lmmsim::IntDistribution::uniform(d.lo, d.hi)
                   : lmmsim::IntDistribution::constant(d.lo);
}

inline lmmsim::WorkloadConfig to_workload_config(const rs_workload_config& w) {
  using namespace lmmsim;
  WorkloadConfig out;
  out.arrival_rate = w.arrival_rate;
  out.duration_s = w.duration_s;
  out.seed = w.seed;
  for (int i = 0; i < w.n_templates; ++i) {
    const rs_template& t = w.templates[i];
    RequestTemplate rt;
    if (t.pattern < RS_LAYOUT_ALTERNATING || t.pattern > RS_LAYOUT_TEXT_FIRST)
      throw ConfigError("workload.templates[" + format_u64(static_cast<std::uint64_t>(i)) +
                        "].pattern: unknown enum value");
    rt.pattern = static_cast<LayoutPattern>(t.pattern);
    rt.num_mm_items = to_distribution(t.num_mm_items);
    rt.mm_item_tokens = to_distribution(t.mm_item_tokens);
    rt.text_segment_tokens = to_distribution(t.text_segment_tokens);
    out.template_mix.emplace_back(rt, t.probability);
  }
  if (w.has_slo) out.slo_ttft_ms = w.slo_ttft_ms;
  return out;
}

inline std::vector<lmmsim::RequestSpec> parse_workload_text(const char* text) {
  std::istringstream is(text ? text : "");
  return lmmsim::read_workload(is);
}

}  // namespace rserve
