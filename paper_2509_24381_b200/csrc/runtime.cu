#include <cstdio>
// rserve-b200 — process-wide runtime bits: launch counter, live kernel timing.
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace rserve {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}

void count_launch(std::uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

namespace {
std::atomic<std::uint64_t> g_max_launch_ns{0};
}
void note_launch_ms(double ms) {
  const auto ns = static_cast<std::uint64_t>(ms * 1e6);
  std::uint64_t cur = g_max_launch_ns.load(std::memory_order_relaxed);
  while (ns > cur && !g_max_launch_ns.compare_exchange_weak(cur, ns, std::memory_order_relaxed)) {
  }
}
double take_max_launch_ms() { return static_cast<double>(g_max_launch_ns.exchange(0)) * 1e-6; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RS_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}
std::uint64_t launches_so_far() { return g_launches.load(std::memory_order_relaxed); }

namespace prof {
namespace {
struct Pending {
  cudaEvent_t a, b;
  std::string klass;
  double flops, bytes;
};
struct Agg {
  std::uint64_t n = 0;
  double ms = 0, flops = 0, bytes = 0;
};
std::mutex mu;
bool on = false;
std::vector<Pending> pending;
std::vector<cudaEvent_t> started;  // begin events awaiting end()
std::vector<cudaEvent_t> spare;

cudaEvent_t get_event() {
  if (!spare.empty()) {
    cudaEvent_t e = spare.back();
    spare.pop_back();
    return e;
  }
  cudaEvent_t e;
  RS_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}
}  // namespace

bool enabled() { return on; }
void enable(bool v) {
  std::lock_guard<std::mutex> g(mu);
  on = v;
}

int begin(cudaStream_t st) {
  if (!on) return -1;
  std::lock_guard<std::mutex> g(mu);
  cudaEvent_t e = get_event();
  RS_CUDA_CHECK(cudaEventRecord(e, st));
  started.push_back(e);
  return static_cast<int>(started.size()) - 1;
}

void end(int token, cudaStream_t st, const char* klass, double flops, double bytes) {
  if (token < 0) return;
  std::lock_guard<std::mutex> g(mu);
  cudaEvent_t e = get_event();
  RS_CUDA_CHECK(cudaEventRecord(e, st));
  pending.push_back({started[static_cast<std::size_t>(token)], e, klass, flops, bytes});
}

std::string drain() {
  std::lock_guard<std::mutex> g(mu);
  std::map<std::string, Agg> agg;
  for (Pending& p : pending) {
    RS_CUDA_CHECK(cudaEventSynchronize(p.b));
    float ms = 0;
    RS_CUDA_CHECK(cudaEventElapsedTime(&ms, p.a, p.b));
    Agg& a = agg[p.klass];
    ++a.n;
    a.ms += ms;
    a.flops += p.flops;
    a.bytes += p.bytes;
    spare.push_back(p.a);
    spare.push_back(p.b);
  }
  pending.clear();
  started.clear();
  std::string out;
  for (const auto& [k, a] : agg)
    out += k + " " + std::to_string(a.n) + " " + std::to_string(a.ms) + " " +
           std::to_string(a.flops) + " " + std::to_string(a.bytes) + "\n";
  return out;
}
}  // namespace prof

double host_trace_ms() {
  static const double v = [] {
    const char* e = std::getenv("RS_HOST_TRACE");
    return e != nullptr ? std::atof(e) : 0.0;
  }();
  return v;
}

HostPhase::~HostPhase() {
  const double lim = host_trace_ms();
  if (lim <= 0.0) return;
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > lim) std::fprintf(stderr, "[rs host] %s took %.2f ms\n", label, ms);
}

}  // namespace rserve
