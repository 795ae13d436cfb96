// rserve-b200 — Algorithm 1: chunked multimodal encode batching + FCFS queue.
//
// plan_batches reproduces reference proj/include/lmmsim/encoder_sched.hpp:
// 48-74 (threshold tested after each appended item, items never split,
// trailing remainder flushed, C == 0 rejected, kWholeRequest sentinel at
// 32-33); EncoderQueue reproduces 80-100 (global FIFO, no overtaking).
// On B200 each EncodeBatch is one vision-encoder launch sequence: its
// total_tokens * 4 patches form the M dimension of every ViT GEMM.
#pragma once

#include <cstdint>
#include <deque>
#include <limits>
#include <optional>
#include <utility>
#include <vector>

#include "lmmsim/errors.hpp"
#include "lmmsim/request.hpp"

namespace lmmsim {

/// Threshold that is never reached: all items of a request land in one
/// trailing batch (the encode-everything-first baseline).
inline constexpr TokenCount kWholeRequest =
    std::numeric_limits<TokenCount>::max();

struct EncodeBatch {
  RequestId request_id = 0;
  std::vector<std::pair<std::size_t, TokenRange>> items;  // (item idx, range)
  TokenCount total_tokens = 0;
  TimeMs dispatch_ms = -1;
};

inline std::vector<EncodeBatch> plan_batches(const RequestSpec& req,
                                             TokenCount batch_tokens) {
  if (batch_tokens == 0)
    throw ConfigError("embedding_batch_size_C: must be >= 1");

  std::vector<EncodeBatch> plan;
  EncodeBatch open;
  open.request_id = req.id;
  std::size_t item = 0;
  for (const TokenRange& r : req.mm_item_ranges()) {
    open.items.emplace_back(item++, r);
    open.total_tokens += r.length();
    if (open.total_tokens < batch_tokens) continue;
    plan.push_back(std::move(open));
    open = EncodeBatch{};
    open.request_id = req.id;
  }
  if (!open.items.empty()) plan.push_back(std::move(open));
  return plan;
}

class EncoderQueue {
 public:
  void enqueue_request(std::vector<EncodeBatch> planned) {
    for (EncodeBatch& b : planned) fifo_.push_back(std::move(b));
  }

  std::optional<EncodeBatch> next_dispatch(bool encoder_idle, TimeMs now) {
    if (!encoder_idle || fifo_.empty()) return std::nullopt;
    std::optional<EncodeBatch> head(std::move(fifo_.front()));
    fifo_.pop_front();
    head->dispatch_ms = now;
    return head;
  }

  bool empty() const { return fifo_.empty(); }
  std::size_t pending() const { return fifo_.size(); }

 private:
  std::deque<EncodeBatch> fifo_;
};

}  // namespace lmmsim
