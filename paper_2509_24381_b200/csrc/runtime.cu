// rserve-b200 — process-wide runtime bits: launch counter, device checks.
#include <atomic>

#include "common.cuh"

namespace rserve {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}

void count_launch(std::uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
std::uint64_t launches_so_far() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace rserve
