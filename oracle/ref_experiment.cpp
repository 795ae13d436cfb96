// ORACLE — test infrastructure only (never linked into the product).
//
// Runs the reference's OWN experiment harness functions, compiled from the
// unmodified /root/reference/proj headers (oracle/Makefile), to produce golden
// outputs for the device-engine harness (scripts/b200_experiment.py):
//
//   ref_experiment <config.json> <out_dir> sweep <C,C,...>
//       ExperimentConfig::load (config.hpp:357-371) + sweep_batch_size
//       (experiment.hpp:296-330): writes <out_dir>/batch_size_sweep.csv
//   ref_experiment <config.json> <out_dir> compare <baseline> <target>
//       run_experiment (experiment.hpp:109-173) + compare_policies
//       (experiment.hpp:222-281): writes report.csv and prints one JSON
//       line per rate (%.17g: exact doubles)
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "lmmsim/experiment.hpp"

using namespace lmmsim;

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s config out_dir sweep C,.. | compare base target\n", argv[0]);
    return 2;
  }
  try {
    ExperimentConfig cfg = ExperimentConfig::load(argv[1]);
    cfg.output_dir = argv[2];
    const std::string cmd = argv[3];
    if (cmd == "sweep" && argc >= 5) {
      std::vector<TokenCount> values;
      std::stringstream ss(argv[4]);
      for (std::string v; std::getline(ss, v, ',');)
        values.push_back(v == "whole_request" ? kWholeRequest : std::strtoull(v.c_str(), nullptr, 10));
      sweep_batch_size(cfg, values);
      return 0;
    }
    if (cmd == "compare" && argc >= 6) {
      const ExperimentOutput out = run_experiment(cfg);
      for (const CompareRow& c :
           compare_policies(out.rows, policy_from_string(argv[4]), policy_from_string(argv[5])))
        std::printf("{\"rate\": %.17g, \"baseline_mean_ttft_ms\": %.17g, \"target_mean_ttft_ms\": %.17g, "
                    "\"ttft_reduction_pct\": %.17g, \"baseline_throughput_tok_s\": %.17g, "
                    "\"target_throughput_tok_s\": %.17g, \"throughput_ratio\": %.17g}\n",
                    c.rate, c.baseline_mean_ttft_ms, c.target_mean_ttft_ms, c.ttft_reduction_pct,
                    c.baseline_throughput_tok_s, c.target_throughput_tok_s, c.throughput_ratio);
      return 0;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "bad arguments\n");
  return 2;
}
