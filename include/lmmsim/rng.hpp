// rserve-b200 — deterministic random source for workload layouts.
//
// Must produce the reference's exact draws (proj/include/lmmsim/rng.hpp:
// 28-64) so generated layouts — and therefore every scheduling decision —
// match: std::mt19937_64 (output fixed by the standard) plus explicit
// arithmetic only (no std::*_distribution, whose mapping is unspecified).
#pragma once

#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace lmmsim {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : mt_(seed) {}

  std::uint64_t next_u64() { return mt_(); }

  /// 53 random mantissa bits scaled into [0, 1).
  double uniform01() { return static_cast<double>(mt_() >> 11) * 0x1.0p-53; }

  /// Exponential variate with the given mean (inverse CDF, u == 0 redrawn).
  double exponential(double mean) {
    double u;
    do {
      u = uniform01();
    } while (u == 0.0);
    return -mean * std::log(u);
  }

  /// Inclusive integer range [lo, hi]; lo >= hi returns lo.
  std::uint64_t uniform_int(std::uint64_t lo, std::uint64_t hi) {
    return lo >= hi ? lo : lo + mt_() % (hi - lo + 1);
  }

  /// Index of the first cumulative bucket above a uniform draw.
  std::size_t pick_cumulative(const std::vector<double>& cumulative) {
    const double u = uniform01();
    const std::size_t n = cumulative.size();
    for (std::size_t i = 0; i + 1 < n; ++i)
      if (u < cumulative[i]) return i;
    return n == 0 ? 0 : n - 1;
  }

 private:
  std::mt19937_64 mt_;
};

}  // namespace lmmsim
