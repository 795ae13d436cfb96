// rserve-b200 — request payload files.
//
// The reference's workload files carry only layouts (`id,arrival,slo,layout`,
// workload.hpp:217-265): no pixels, no token ids. The engine synthesises
// payloads from per-request hashes (pixels: mix64(run seed, pixel stream of
// (request, item)); text ids: mix64(run seed, 6<<32 | request, position) %
// vocab). A payload file, kept beside the workload file, pins or overrides
// them per segment so CPU and GPU runs (and replays) see identical inputs:
//
//   # rserve payload v1
//   <req_id>,<segment_index>,M,grid=<gh>x<gw>[;seed=<u64>]
//   <req_id>,<segment_index>,T,seed=<u64>
//   <req_id>,<segment_index>,T,ids=<id> <id> ...
//
// M: merged-token grid of the image (gh * gw == the segment's tokens; the
// ViT sees (2gh) x (2gw) patches) and its pixel seed. T: token-id seed or the
// explicit ids (one per token, each < vocab). Segments without a line keep
// the synthesised defaults (grid = the most square factorisation).
// Errors are lmmsim::InputError("payload line N: ...") like the reference's
// workload reader.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "lmmsim/request.hpp"

namespace rserve {

struct ItemPayload {
  int gh = 0, gw = 0;        // 0: default grid
  bool has_seed = false;
  std::uint64_t seed = 0;    // pixel hash seed
};
struct TextPayload {
  bool has_seed = false;
  std::uint64_t seed = 0;
  std::vector<std::int32_t> ids;  // explicit ids (empty: seeded)
};
struct RequestPayload {
  std::map<std::size_t, ItemPayload> items;  // by segment index
  std::map<std::size_t, TextPayload> texts;  // by segment index
};
using PayloadSpec = std::unordered_map<lmmsim::RequestId, RequestPayload>;

PayloadSpec parse_payload(const std::string& text);
std::string format_payload(const PayloadSpec& spec);
/// Checks segment kinds, grids, id counts / ranges and request ids against
/// the workload; throws lmmsim::InputError.
void validate_payload(const PayloadSpec& spec, const std::vector<lmmsim::RequestSpec>& workload,
                      int vocab);
/// A payload for `workload`, keyed by the workload's own seed: per image a
/// grid drawn among the factorisations of its token count with aspect ratio
/// <= 4 and a pixel seed; per text segment a token-id seed.
PayloadSpec generate_payload(const std::vector<lmmsim::RequestSpec>& workload, std::uint64_t seed);

/// Default grid of an item of `tokens` merged tokens (most square factorisation).
void default_item_grid(std::uint64_t tokens, int* gh, int* gw);

/// Resolved payload of one request, in the order the device consumes it.
struct ResolvedPayload {
  std::vector<std::pair<int, int>> item_grids;  // per MM item
  std::vector<std::uint64_t> item_seeds;        // per MM item (pixel seed)
  std::vector<std::int32_t> text_ids;           // all text tokens, prompt order
};
ResolvedPayload resolve_payload(const lmmsim::RequestSpec& req, const RequestPayload* p,
                                std::uint64_t run_seed, int vocab);

}  // namespace rserve
