// rserve-b200 — Algorithm 2: schedulable-token micro-batching + policies.
//
// Policy names/traits follow reference proj/include/lmmsim/token_sched.hpp:
// 43-103; policy_schedulable 119-123; build_microbatch 132-180 (budget
// sweep, partial admission, blocked/incomplete requests re-prepended in
// sweep order, intra_only stops after one admission, vanilla admits one
// whole fully-ready prompt ignoring B); on_embeddings_ready 184-187.
// A MicroBatch is exactly one varlen prefill chunk on the B200: its slices
// become the token rows of every LLM GEMM of that chunk.
#pragma once

#include <algorithm>
#include <deque>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "lmmsim/errors.hpp"
#include "lmmsim/tracker.hpp"

namespace lmmsim {

enum class Policy { VanillaPp, EpdBaseline, IntraOnly, Rserve };

namespace detail {
struct PolicyName {
  Policy policy;
  const char* name;
};
inline constexpr PolicyName kPolicyNames[] = {
    {Policy::VanillaPp, "vanilla_pp"},
    {Policy::EpdBaseline, "epd_baseline"},
    {Policy::IntraOnly, "intra_only"},
    {Policy::Rserve, "rserve"},
};
}  // namespace detail

inline const char* to_string(Policy p) {
  for (const auto& entry : detail::kPolicyNames)
    if (entry.policy == p) return entry.name;
  return "?";
}

inline Policy policy_from_string(const std::string& name) {
  for (const auto& entry : detail::kPolicyNames)
    if (name == entry.name) return entry.policy;
  throw ConfigError("policy: unknown name '" + name +
                    "' (expected vanilla_pp, epd_baseline, intra_only or "
                    "rserve)");
}

enum class PipelineMode { Cpp, Vanilla };

struct PolicyTraits {
  Policy policy = Policy::Rserve;
  PipelineMode default_mode = PipelineMode::Cpp;
  bool require_full_encode = false;    // hidden until every item is encoded
  bool single_request_chunks = false;  // one request per micro-batch
  bool whole_prompt_chunks = false;    // a micro-batch is a whole prompt
  bool whole_request_encode = false;   // encode batches = whole request
};

inline PolicyTraits select_policy(Policy policy) {
  PolicyTraits t;
  t.policy = policy;
  const bool vanilla = policy == Policy::VanillaPp;
  const bool epd = policy == Policy::EpdBaseline;
  t.default_mode = vanilla ? PipelineMode::Vanilla : PipelineMode::Cpp;
  t.require_full_encode = vanilla || epd;
  t.whole_request_encode = vanilla || epd;
  t.whole_prompt_chunks = vanilla;
  t.single_request_chunks = vanilla || policy == Policy::IntraOnly;
  return t;
}

struct MicroBatch {
  std::vector<std::pair<RequestId, TokenRange>> slices;  // queue order
  TokenCount total_tokens = 0;
  TimeMs creation_ms = 0;
};

struct SchedulerQueues {
  std::deque<RequestId> waiting;  // FCFS between sweeps
};

inline TokenCount policy_schedulable(const PolicyTraits& traits,
                                     const EmbeddingTracker& tracker) {
  const bool gated = traits.require_full_encode && !tracker.all_encoded();
  return gated ? 0 : tracker.schedulable_tokens();
}

namespace detail {
// vanilla_pp: the first request whose whole remaining prompt is visible.
inline std::optional<MicroBatch> admit_whole_prompt(SchedulerQueues& queues,
                                                    TrackerRegistry& registry,
                                                    const PolicyTraits& traits,
                                                    MicroBatch mb) {
  auto& q = queues.waiting;
  for (auto it = q.begin(); it != q.end(); ++it) {
    EmbeddingTracker& tr = registry.get(*it);
    const TokenCount visible = policy_schedulable(traits, tr);
    if (visible == 0) continue;
    mb.slices.emplace_back(*it, tr.advance_prefill(visible));
    mb.total_tokens = visible;
    q.erase(it);
    return mb;
  }
  return std::nullopt;
}
}  // namespace detail

inline std::optional<MicroBatch> build_microbatch(SchedulerQueues& queues,
                                                  TrackerRegistry& registry,
                                                  TokenCount budget,
                                                  const PolicyTraits& traits,
                                                  TimeMs now) {
  if (budget == 0) throw ConfigError("token_budget_B: must be >= 1");
  MicroBatch mb;
  mb.creation_ms = now;
  if (traits.whole_prompt_chunks)
    return detail::admit_whole_prompt(queues, registry, traits, std::move(mb));

  auto& q = queues.waiting;
  std::vector<RequestId> keep;  // swept but not finished, in sweep order
  TokenCount left = budget;
  while (left > 0 && !q.empty()) {
    const RequestId id = q.front();
    q.pop_front();
    EmbeddingTracker& tr = registry.get(id);
    const TokenCount visible = policy_schedulable(traits, tr);
    if (visible == 0) {
      keep.push_back(id);
      continue;
    }
    const TokenCount take = visible < left ? visible : left;
    mb.slices.emplace_back(id, tr.advance_prefill(take));
    mb.total_tokens += take;
    left -= take;
    if (!tr.fully_prefilled()) keep.push_back(id);
    if (traits.single_request_chunks) break;
  }
  q.insert(q.begin(), keep.begin(), keep.end());
  if (mb.slices.empty()) return std::nullopt;
  return mb;
}

inline void on_embeddings_ready(TrackerRegistry& registry, RequestId id,
                                TokenRange item_range) {
  registry.get(id).mark_encoded(item_range);
}

}  // namespace lmmsim
