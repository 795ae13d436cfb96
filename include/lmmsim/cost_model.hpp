// rserve-b200 — analytic cost model (the reference's execution seam).
//
// Formulas and validation follow reference proj/include/lmmsim/
// cost_model.hpp:37-88 (same floating-point operation order, so virtual
// times are bit-identical). On the B200 these functions are only used by
// the virtual-clock ("lock-step") mode of the engine, where the ORDER of
// events follows the reference while the encode / transfer / stage work is
// executed for real by the sm_100a kernels behind include/rserve.h.
#pragma once

#include <string>

#include "lmmsim/encoder_sched.hpp"
#include "lmmsim/errors.hpp"
#include "lmmsim/request.hpp"

namespace lmmsim {

struct CostModel {
  double alpha_enc_ms = 0;
  double beta_enc_ms_per_token = 0;
  double eps_tx_ms = 0;
  double zeta_tx_ms_per_token = 0;
  double gamma_stage_ms = 0;
  double delta_stage_ms_per_token = 0;
  double kappa_attn_ms = 0;
  double tp_speedup = 1.0;

  void validate() const {
    const struct {
      double value;
      const char* field;
    } knobs[] = {
        {alpha_enc_ms, "alpha_enc_ms"},
        {beta_enc_ms_per_token, "beta_enc_ms_per_token"},
        {eps_tx_ms, "eps_tx_ms"},
        {zeta_tx_ms_per_token, "zeta_tx_ms_per_token"},
        {gamma_stage_ms, "gamma_stage_ms"},
        {delta_stage_ms_per_token, "delta_stage_ms_per_token"},
        {kappa_attn_ms, "kappa_attn_ms"},
    };
    for (const auto& k : knobs)
      if (!(k.value >= 0))  // also rejects NaN
        throw ConfigError(std::string("cost_model.") + k.field +
                          ": must be >= 0");
    if (!(tp_speedup >= 1.0))
      throw ConfigError("cost_model.tp_speedup: must be >= 1");
    if (beta_enc_ms_per_token == 0 && delta_stage_ms_per_token == 0)
      throw ConfigError(
          "cost_model: at least one of beta_enc_ms_per_token and "
          "delta_stage_ms_per_token must be > 0");
  }
};

inline double encode_time_ms(const CostModel& cm, const EncodeBatch& batch) {
  const double tokens = static_cast<double>(batch.total_tokens);
  return cm.alpha_enc_ms + cm.beta_enc_ms_per_token * tokens;
}

inline double stage_time_ms(const CostModel& cm, TokenCount chunk_tokens,
                            double context_tokens) {
  const double m = static_cast<double>(chunk_tokens);
  const double work = cm.gamma_stage_ms + cm.delta_stage_ms_per_token * m +
                      cm.kappa_attn_ms * m * context_tokens;
  return work / cm.tp_speedup;
}

inline double transfer_time_ms(const CostModel& cm, TokenCount tokens) {
  return cm.eps_tx_ms + cm.zeta_tx_ms_per_token * static_cast<double>(tokens);
}

}  // namespace lmmsim
