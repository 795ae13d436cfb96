// rserve-b200 — EP topology and control-message codec (host only).
//
// Control messages are fixed-size arrays of kCtrlWords int64 words so that
// every receive knows its byte count up front (NCCL point-to-point requires
// matched sizes). Layout:
//   [0] magic "RSEP"  [1] kind  [2] payload words  [3..] payload
//   ENCODE: slot, request_id, n_items, n_items x (index, start, end, patch_offset)
//   STAGE : chunk_id, n_slices, per slice (request_id, start, end, n_segments,
//           n_segments x (kind, tokens))
//   STOP  : (empty)
// The text form (to_text / from_text) is `ENCODE slot=.. req=.. items=i:s-e@p,..`
// `STAGE chunk=.. slices=req:s-e[T128|M1024],..` / `STOP`.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "lmmsim/request.hpp"

namespace rserve::ep {

struct Topology {
  int stages = 1;    // prefill GPUs P0 .. P_{S-1} = ranks 0 .. S-1
  int encoders = 1;  // encoder GPUs E0 .. E_{W-1} = ranks S .. S+W-1
  int p_rank(int s) const { return s; }
  int e_rank(int w) const { return stages + w; }
  int world() const { return stages + encoders; }
  bool is_encoder(int rank) const { return rank >= stages; }
  /// Directed links (src, dst), in the order every rank creates them:
  /// P0->E_w, E_w->P0 for each w; P_s->P_{s+1}; P_s->P0 for s >= 1.
  std::vector<std::pair<int, int>> links() const;
  /// Index of link (src, dst) in links(); -1 if absent.
  int link_index(int src, int dst) const;
  void validate() const;  // ConfigError
};

constexpr std::size_t kCtrlWords = 4096;  // 32 KB control message
constexpr std::size_t kCtrlBytes = kCtrlWords * sizeof(std::int64_t);
constexpr std::size_t kHeaderBytes = 64;  // ENC-DONE / DONE header
constexpr std::int64_t kMagic = 0x52534550;

enum class Ctrl : std::int64_t { kStop = 0, kEncode = 1, kStage = 2 };

struct EncodeItem {
  std::uint64_t index = 0;           // multimodal item ordinal within the request
  std::uint64_t start = 0, end = 0;  // prompt token range
  std::uint64_t patch_offset = 0;    // first patch of the item in the request payload
  bool operator==(const EncodeItem&) const = default;
};
struct EncodeCmd {  // P0 -> E_w
  std::uint64_t slot = 0, request_id = 0;
  std::vector<EncodeItem> items;
  std::uint64_t tokens() const {
    std::uint64_t n = 0;
    for (const EncodeItem& i : items) n += i.end - i.start;
    return n;
  }
  bool operator==(const EncodeCmd&) const = default;
};
struct SliceCmd {
  std::uint64_t request_id = 0, start = 0, end = 0;
  std::vector<lmmsim::SegmentSpec> segments;  // request layout (KV sizing, M-RoPE ids)
  std::uint64_t total() const {
    std::uint64_t n = 0;
    for (const auto& s : segments) n += s.tokens;
    return n;
  }
  bool operator==(const SliceCmd&) const = default;
};
struct StageCmd {  // P_s -> P_{s+1}
  std::uint64_t chunk_id = 0;
  std::vector<SliceCmd> slices;
  std::uint64_t rows() const {
    std::uint64_t n = 0;
    for (const SliceCmd& s : slices) n += s.end - s.start;
    return n;
  }
  bool operator==(const StageCmd&) const = default;
};

using Words = std::vector<std::int64_t>;
void pack(const EncodeCmd& c, Words& w);
void pack(const StageCmd& c, Words& w);
void pack_stop(Words& w);
Ctrl kind_of(const Words& w);  // DataError on a malformed message
EncodeCmd unpack_encode(const Words& w);
StageCmd unpack_stage(const Words& w);
std::string to_text(const Words& w);
Words from_text(const std::string& text);

}  // namespace rserve::ep
