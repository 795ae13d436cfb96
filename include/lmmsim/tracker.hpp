// rserve-b200 — per-request embedding tracker (host mirror of the device
// readiness bitmap).
//
// Semantics follow the reference tracker exactly (proj/include/lmmsim/
// tracker.hpp: ctor 44-59, schedulable_tokens 79, mark_encoded 83-105,
// advance_prefill 109-122, release 126-135, registry 158-198), including
// every exception class and message text. The representation is B200-first:
// readiness is a packed uint32 bitmap, bit (i % 32) of word (i / 32) for
// prompt token i — byte-for-byte the layout the device tracker keeps in HBM
// (paper_2509_24381_b200/csrc/elementwise.cu K6/K7), so host and device state
// can be compared word by word. Item lookup is a binary search over the
// (sorted, disjoint) item starts and the ready run advances a word at a time.
//
// The host mirror stays authoritative for every scheduling decision; the
// device bitmap is what the kernels read, and tests assert the two agree.
#pragma once

#include <algorithm>
#include <bit>
#include <cstdint>
#include <unordered_map>
#include <vector>

#include "lmmsim/errors.hpp"
#include "lmmsim/request.hpp"

namespace lmmsim {

namespace bitmap {
inline constexpr std::uint32_t kAll = 0xFFFFFFFFu;

inline std::size_t words_for(TokenCount tokens) {
  return static_cast<std::size_t>((tokens + 31) / 32);
}

/// Sets bits [begin, end) of `words`.
inline void set_range(std::vector<std::uint32_t>& words, TokenIndex begin,
                      TokenIndex end) {
  while (begin < end) {
    const std::size_t w = static_cast<std::size_t>(begin >> 5);
    const unsigned lo = static_cast<unsigned>(begin & 31);
    const TokenIndex word_end = (static_cast<TokenIndex>(w) + 1) << 5;
    const TokenIndex stop = std::min(end, word_end);
    const unsigned span = static_cast<unsigned>(stop - begin);
    const std::uint32_t mask =
        span == 32 ? kAll : (((std::uint32_t{1} << span) - 1u) << lo);
    words[w] |= mask;
    begin = stop;
  }
}

inline bool test(const std::vector<std::uint32_t>& words, TokenIndex i) {
  return (words[static_cast<std::size_t>(i >> 5)] >> (i & 31)) & 1u;
}

/// First index >= from whose bit is clear, capped at `limit`.
inline TokenIndex first_clear(const std::vector<std::uint32_t>& words,
                              TokenIndex from, TokenIndex limit) {
  TokenIndex i = from;
  while (i < limit) {
    const std::size_t w = static_cast<std::size_t>(i >> 5);
    const unsigned lo = static_cast<unsigned>(i & 31);
    // Bits below `lo` are treated as set so they never stop the scan.
    const std::uint32_t seen = words[w] | ((std::uint32_t{1} << lo) - 1u);
    if (seen != kAll) {
      const TokenIndex hit =
          (static_cast<TokenIndex>(w) << 5) +
          static_cast<TokenIndex>(std::countr_one(seen));
      return std::min(hit, limit);
    }
    i = (static_cast<TokenIndex>(w) + 1) << 5;
  }
  return limit;
}
}  // namespace bitmap

class EmbeddingTracker {
 public:
  EmbeddingTracker(const RequestSpec& req, std::uint32_t hidden_size)
      : id_(req.id),
        total_(req.total_tokens()),
        hidden_(hidden_size),
        ready_(bitmap::words_for(total_), 0u),
        items_(req.mm_item_ranges()) {
    TokenIndex cursor = 0;
    for (const SegmentSpec& seg : req.segments) {
      if (seg.kind == SegmentKind::Text)
        bitmap::set_range(ready_, cursor, cursor + seg.tokens);
      cursor += seg.tokens;
    }
    live_ = req.text_tokens();
    peak_ = live_;
    extend_run();
  }

  RequestId request_id() const { return id_; }
  TokenCount total_tokens() const { return total_; }
  std::uint32_t hidden_size() const { return hidden_; }
  TokenIndex prefilled_frontier() const { return frontier_; }
  TokenCount live_embedding_tokens() const { return live_; }
  TokenCount peak_live_embedding_tokens() const { return peak_; }
  std::uint64_t live_embedding_scalars() const { return live_ * hidden_; }
  TokenCount released_tokens() const { return released_; }
  std::size_t mm_item_count() const { return items_.size(); }
  bool all_encoded() const { return encoded_ == items_.size(); }
  bool fully_prefilled() const { return frontier_ == total_; }
  bool fully_released() const { return released_ == total_; }

  /// Contiguous ready run starting at the prefill frontier.
  TokenCount schedulable_tokens() const { return run_end_ - frontier_; }

  /// First token index >= frontier that is not ready (== total when none).
  TokenIndex ready_run_end() const { return run_end_; }

  /// Packed readiness words (bit i%32 of word i/32), the device layout.
  const std::vector<std::uint32_t>& ready_words() const { return ready_; }
  const std::vector<TokenRange>& items() const { return items_; }

  void mark_encoded(TokenRange r) {
    const auto pos = std::lower_bound(
        items_.begin(), items_.end(), r.start,
        [](const TokenRange& item, TokenIndex s) { return item.start < s; });
    const bool aligned =
        pos != items_.end() && pos->start == r.start && pos->end == r.end;
    if (!aligned)
      throw AlignmentError("request " + format_u64(id_) + ": encode range " +
                           span_text(r) + " does not cover one multimodal item");
    if (bitmap::test(ready_, r.start))
      throw DoubleEncodeError("request " + format_u64(id_) + ": range " +
                              span_text(r) + " already encoded");
    bitmap::set_range(ready_, r.start, r.end);
    ++encoded_;
    live_ += r.length();
    if (live_ > peak_) peak_ = live_;
    extend_run();
  }

  TokenRange advance_prefill(TokenCount n) {
    if (n == 0) throw InternalError("advance_prefill: zero-token advance");
    const TokenCount avail = schedulable_tokens();
    if (n > avail)
      throw DependencyViolation(
          "request " + format_u64(id_) + ": advance of " + format_u64(n) +
          " tokens exceeds schedulable frontier (" + format_u64(avail) +
          " at token " + format_u64(frontier_) + ")");
    const TokenRange taken{frontier_, frontier_ + n};
    frontier_ = taken.end;
    return taken;
  }

  void release(TokenRange r) {
    const bool in_order = r.start == released_ && r.end <= frontier_;
    if (!in_order)
      throw InternalError("request " + format_u64(id_) +
                          ": out-of-order release of " + span_text(r) +
                          " at released frontier " + format_u64(released_));
    released_ = r.end;
    live_ -= r.length();
  }

 private:
  static std::string span_text(TokenRange r) {
    return "[" + format_u64(r.start) + "," + format_u64(r.end) + ")";
  }

  // The run end only moves on creation and on mark_encoded; advances of the
  // frontier never pass it, so scanning resumes where it last stopped.
  void extend_run() { run_end_ = bitmap::first_clear(ready_, run_end_, total_); }

  RequestId id_;
  TokenCount total_;
  std::uint32_t hidden_;
  std::vector<std::uint32_t> ready_;
  std::vector<TokenRange> items_;
  TokenIndex frontier_ = 0;
  TokenIndex released_ = 0;
  TokenIndex run_end_ = 0;
  TokenCount live_ = 0;
  TokenCount peak_ = 0;
  std::size_t encoded_ = 0;
};

/// Live trackers by request id. Single-threaded owner (the engine loop).
class TrackerRegistry {
 public:
  EmbeddingTracker& create(const RequestSpec& req, std::uint32_t hidden_size) {
    if (map_.count(req.id))
      throw RegistryError("duplicate request id " + format_u64(req.id));
    return map_.emplace(req.id, EmbeddingTracker(req, hidden_size))
        .first->second;
  }

  EmbeddingTracker& get(RequestId id) {
    const auto it = map_.find(id);
    if (it == map_.end())
      throw RegistryError("unknown request id " + format_u64(id));
    return it->second;
  }

  const EmbeddingTracker* find(RequestId id) const {
    const auto it = map_.find(id);
    return it != map_.end() ? &it->second : nullptr;
  }

  bool contains(RequestId id) const { return map_.find(id) != map_.end(); }
  std::size_t size() const { return map_.size(); }

  void erase(RequestId id) {
    if (!map_.erase(id))
      throw RegistryError("erase of unknown request id " + format_u64(id));
  }

 private:
  std::unordered_map<RequestId, EmbeddingTracker> map_;
};

inline EmbeddingTracker& create_tracker(TrackerRegistry& registry,
                                        const RequestSpec& req,
                                        std::uint32_t hidden_size) {
  req.validate();
  return registry.create(req, hidden_size);
}

}  // namespace lmmsim
