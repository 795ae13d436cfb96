// rserve-b200 — host-only C-ABI entry points (no device required).
//
// These expose the scheduling core (include/lmmsim/) through include/
// rserve.h: workload generation, the engine over the analytic cost model
// (the reference's run_simulation), one experiment report row, and
// Algorithm 1. The device entry points live in capi_device.cu.
#include <sstream>
#include <string>
#include <vector>

#include "host/config_bridge.hpp"
#include "host/decision_log.hpp"
#include "host/status.hpp"
#include "lmmsim/metrics.hpp"
#include "lmmsim/simengine.hpp"
#include "lmmsim/workload.hpp"
#include "rserve.h"

namespace rserve {
std::string& last_error_slot() {
  thread_local std::string slot;
  return slot;
}
}  // namespace rserve

using namespace rserve;

extern "C" {

const char* rs_last_error(void) { return last_error_slot().c_str(); }
void rs_free(void* p) { std::free(p); }
const char* rs_version(void) { return "rserve-b200 0.1 sm_100a tcgen05/TMA"; }

rs_status rs_generate_workload(const rs_workload_config* cfg, char** out_text) {
  return guarded([&] {
    std::ostringstream os;
    lmmsim::write_workload(os, lmmsim::generate_workload(to_workload_config(*cfg)));
    *out_text = c_string(os.str());
  });
}

rs_status rs_simulate(const char* workload_text, const rs_sim_config* cfg,
                      char** out_result, char** out_journal) {
  return guarded([&] {
    lmmsim::Simulation sim(parse_workload_text(workload_text), to_sim_config(*cfg));
    const lmmsim::SimResult res = sim.run();
    std::vector<ReleaseRecord> rel;
    for (const lmmsim::ReleaseEvent& e : sim.releases()) rel.push_back({e.chunk, e.id, e.range});
    if (out_result) *out_result = c_string(render_decision_log(res, rel, true));
    if (out_journal) *out_journal = c_string(render_journal(sim.journal()));
  });
}

rs_status rs_experiment_cell(const rs_workload_config* wcfg, const rs_sim_config* cfg,
                             double slo_ttft_ms, char** out_csv_row) {
  return guarded([&] {
    const lmmsim::SimConfig sc = to_sim_config(*cfg);
    const lmmsim::SimResult res =
        lmmsim::run_simulation(lmmsim::generate_workload(to_workload_config(*wcfg)), sc);
    std::optional<double> slo;
    if (slo_ttft_ms >= 0) slo = slo_ttft_ms;
    const lmmsim::MetricsReport rep = lmmsim::compute_report(res, slo);
    *out_csv_row = c_string(lmmsim::report_csv_row(lmmsim::to_string(sc.policy),
                                                   wcfg->arrival_rate, wcfg->seed, rep));
  });
}

rs_status rs_plan_batches(const char* layout, uint64_t request_id, uint64_t c_tokens,
                          char** out_text) {
  return guarded([&] {
    lmmsim::RequestSpec req;
    req.id = request_id;
    req.segments = lmmsim::parse_layout(layout ? layout : "");
    std::string text;
    for (const lmmsim::EncodeBatch& b : lmmsim::plan_batches(req, c_tokens)) {
      text += lmmsim::format_u64(b.request_id);
      for (const auto& [idx, r] : b.items)
        text += " " + lmmsim::format_u64(idx) + ":" + lmmsim::format_u64(r.start) + "-" +
                lmmsim::format_u64(r.end);
      text += " total=" + lmmsim::format_u64(b.total_tokens) + "\n";
    }
    *out_text = c_string(text);
  });
}

}  // extern "C"
