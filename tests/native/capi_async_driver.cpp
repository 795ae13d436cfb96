// Test driver (tests/test_capi_async_gpu.py): the reference's event loop —
// PipelineEngine with the decision points of Simulation (simengine.hpp:
// 275-441) — driving the B200 device ONLY through the public C-ABI's
// asynchronous seam (include/rserve.h: rs_request_create_segments,
// rs_encode_batch_async, rs_embeddings_ready, rs_prefill_chunk_async,
// rs_release_async, rs_request_erase_async, rs_poll). It is what a
// maintainer of the reference would write to put the device behind its
// Simulation: an ExecutionBackend whose launch_* calls queue device work and
// return the cost model's durations (lock-step clock).
//
// Checks, printed as one JSON line:
//   * the decision log equals rs_simulate's (the reference's run_simulation)
//     byte for byte;
//   * every request's first-token logits equal those of rs_engine_run on the
//     same inputs (lock-step), element for element;
//   * rs_poll delivered every launch's completion exactly once, in
//     non-decreasing time.
// Inputs (pixels, token ids) are generated here from the documented payload
// hash (oracle/model_oracle.py uniform / token_ids), so both runs
// see identical bytes.
//
// usage: capi_async_driver <workload file> <policy 0-3> <C> <B> <payload seed> [model preset]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "host/decision_log.hpp"
#include "lmmsim/simengine.hpp"
#include "lmmsim/workload.hpp"
#include "rserve.h"

namespace {

void check(rs_status s, const char* what) {
  if (s != RS_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, static_cast<int>(s), rs_last_error());
    std::exit(2);
  }
}

std::uint64_t mix64(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + stream * 0xD1B54A32D192ED03ull + i;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint16_t bf16_rne(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

// pixels of item `item` of request `req`: [4 tokens, 1176] bf16
std::vector<std::uint16_t> pixels(std::uint64_t seed, std::uint64_t req, std::uint64_t item, std::uint64_t tokens) {
  const std::uint64_t stream = (5ull << 32) | (req << 12) | item;
  const std::uint64_t n = 4 * tokens * 1176;
  std::vector<std::uint16_t> out(n);
  for (std::uint64_t i = 0; i < n; ++i) {
    const float u = static_cast<float>(mix64(seed, stream, i) >> 40) * (1.0f / 16777216.0f);
    out[i] = bf16_rne((2.0f * u - 1.0f) * 1.7320508076f);
  }
  return out;
}

struct Backend final : lmmsim::ExecutionBackend {
  rs_ctx* ctx;
  lmmsim::CostModel cm;
  std::uint64_t seed;
  int vocab;
  std::map<lmmsim::RequestId, lmmsim::RequestSpec> specs;
  std::map<std::size_t, std::vector<std::uint16_t>> batch_pixels;  // encode slot -> host patches
  std::map<lmmsim::RequestId, std::size_t> last_chunk;
  std::set<std::uint64_t> encodes_open, stages_open;
  std::vector<rs_event> events;

  double launch_encode(int, std::size_t slot, const lmmsim::EncodeBatch& b) override {
    const lmmsim::RequestSpec& req = specs.at(b.request_id);
    const auto items = req.mm_item_ranges();
    std::vector<std::uint64_t> ranges;
    std::vector<std::uint16_t>& px = batch_pixels[slot];
    px.clear();
    for (const auto& [idx, range] : b.items) {
      (void)items;
      ranges.push_back(range.start);
      ranges.push_back(range.end);
      const auto p = pixels(seed, req.id, idx, range.length());
      px.insert(px.end(), p.begin(), p.end());
    }
    check(rs_encode_batch_async(ctx, b.request_id, ranges.data(), static_cast<int32_t>(b.items.size()),
                                px.data(), 1, nullptr, slot),
          "rs_encode_batch_async");
    encodes_open.insert(slot);
    return lmmsim::encode_time_ms(cm, b);
  }
  double launch_transfer(int, std::size_t, const lmmsim::EncodeBatch& b) override {
    return lmmsim::transfer_time_ms(cm, b.total_tokens);  // co-located: the zero-cost link
  }
  void on_embeddings_ready(std::size_t slot, const lmmsim::EncodeBatch&) override {
    check(rs_embeddings_ready(ctx, slot), "rs_embeddings_ready");
  }
  double launch_stage(int, const lmmsim::ChunkView& c) override {
    std::vector<std::uint64_t> sl;
    for (const auto& [id, r] : *c.slices) {
      sl.push_back(id);
      sl.push_back(r.start);
      sl.push_back(r.end);
      last_chunk[id] = c.chunk_id;
    }
    check(rs_prefill_chunk_async(ctx, sl.data(), static_cast<int32_t>(c.slices->size()), nullptr, c.chunk_id),
          "rs_prefill_chunk_async");
    stages_open.insert(c.chunk_id);
    return lmmsim::stage_time_ms(cm, c.total_tokens, c.weighted_context);
  }
  void on_request_created(const lmmsim::RequestSpec& req, const lmmsim::EmbeddingTracker&) override {
    specs[req.id] = req;
    std::vector<rs_segment> segs;
    std::vector<int32_t> ids;
    std::uint64_t pos = 0;
    for (const lmmsim::SegmentSpec& s : req.segments) {
      segs.push_back({s.kind == lmmsim::SegmentKind::Text ? RS_SEG_TEXT : RS_SEG_MULTIMODAL, s.tokens});
      if (s.kind == lmmsim::SegmentKind::Text)
        for (std::uint64_t t = 0; t < s.tokens; ++t)
          ids.push_back(static_cast<int32_t>(mix64(seed, (6ull << 32) | req.id, pos + t) %
                                             static_cast<std::uint64_t>(vocab)));
      pos += s.tokens;
    }
    check(rs_request_create_segments(ctx, req.id, segs.data(), static_cast<int32_t>(segs.size()),
                                     ids.empty() ? nullptr : ids.data()),
          "rs_request_create_segments");
  }
  void on_release(std::size_t chunk, lmmsim::RequestId id, lmmsim::TokenRange r) override {
    check(rs_release_async(ctx, id, r.start, r.end, chunk), "rs_release_async");
  }
  void on_request_erased(lmmsim::RequestId id) override {
    check(rs_request_erase_async(ctx, id, last_chunk.at(id)), "rs_request_erase_async");
  }
  void drain() {
    rs_event ev[64];
    for (;;) {
      int32_t n = 0;
      check(rs_poll(ctx, ev, 64, 1, &n), "rs_poll");
      if (n == 0) break;
      events.insert(events.end(), ev, ev + n);
    }
  }
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 6) {
    std::fprintf(stderr, "usage: %s workload policy C B seed [preset]\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1]);
  std::stringstream wl_text;
  wl_text << f.rdbuf();
  std::istringstream wl_is(wl_text.str());
  const std::vector<lmmsim::RequestSpec> workload = lmmsim::read_workload(wl_is);
  rs_sim_config sc{};
  sc.policy = std::atoi(argv[2]);
  sc.pipeline_mode = RS_PIPELINE_DEFAULT;
  sc.stages = 1;
  sc.encoder_workers = 1;
  sc.embedding_batch_tokens = std::strtoull(argv[3], nullptr, 10);
  sc.token_budget = std::strtoull(argv[4], nullptr, 10);
  sc.release_at = RS_RELEASE_LAST_STAGE;
  sc.cost.alpha_enc_ms = 0.5;
  sc.cost.beta_enc_ms_per_token = 0.01;
  sc.cost.delta_stage_ms_per_token = 0.01;
  sc.cost.tp_speedup = 1.0;
  const std::uint64_t seed = std::strtoull(argv[5], nullptr, 10);
  const int preset = argc > 6 ? std::atoi(argv[6]) : RS_MODEL_TINY;

  rs_model_config m{};
  check(rs_model_preset(preset, &m), "rs_model_preset");
  sc.hidden_size = static_cast<uint32_t>(m.llm_dim);
  rs_ctx_options o{};
  o.device = 0;
  o.max_prompt_tokens = 8192;
  o.slot_tokens = 1 << 15;
  o.kv_tokens = 1 << 15;
  o.max_chunk_tokens = 2048;
  o.max_encode_tokens = 1024;
  o.layer_end = m.llm_layers;
  o.with_vit = 1;
  o.with_lm_head = 1;
  rs_ctx* ctx = nullptr;
  check(rs_ctx_create(&m, &o, &ctx), "rs_ctx_create");

  // 1) the reference's decisions
  char* ref_log = nullptr;
  check(rs_simulate(wl_text.str().c_str(), &sc, &ref_log, nullptr), "rs_simulate");
  // 2) the device engine (lock-step) for the reference logits
  rs_run_options ro{};
  ro.clock = 0;
  ro.payload_seed = seed;
  char* eng_log = nullptr;
  char* eng_journal = nullptr;
  rs_run_stats st{};
  check(rs_engine_run(ctx, wl_text.str().c_str(), &sc, &ro, &eng_log, &eng_journal, &st), "rs_engine_run");
  std::map<lmmsim::RequestId, std::vector<float>> eng_logits;
  std::map<lmmsim::RequestId, int32_t> eng_am;
  for (const auto& r : workload) {
    std::vector<float> row(static_cast<std::size_t>(m.vocab));
    check(rs_logits(ctx, r.id, row.data(), &eng_am[r.id]), "rs_logits (engine)");
    eng_logits[r.id] = std::move(row);
  }
  // 3) our own event loop through the asynchronous C-ABI
  lmmsim::SimConfig cfg;
  cfg.policy = static_cast<lmmsim::Policy>(sc.policy);
  cfg.stages = 1;
  cfg.encoder_workers = 1;
  cfg.token_budget = sc.token_budget;
  cfg.embedding_batch_tokens = sc.embedding_batch_tokens;
  cfg.hidden_size = sc.hidden_size;
  cfg.cost.alpha_enc_ms = sc.cost.alpha_enc_ms;
  cfg.cost.beta_enc_ms_per_token = sc.cost.beta_enc_ms_per_token;
  cfg.cost.delta_stage_ms_per_token = sc.cost.delta_stage_ms_per_token;
  Backend be;
  be.ctx = ctx;
  be.cm = cfg.cost;
  be.seed = seed;
  be.vocab = m.vocab;
  lmmsim::PipelineEngine eng(workload, cfg, be);
  const lmmsim::SimResult res = eng.run();
  be.drain();
  std::vector<rserve::ReleaseRecord> rel;
  for (const lmmsim::ReleaseEvent& e : eng.releases()) rel.push_back({e.chunk, e.id, e.range});
  const std::string our_log = rserve::render_decision_log(res, rel, true);
  const bool decisions_equal = our_log == std::string(ref_log);

  double max_diff = 0;
  bool argmax_equal = true, logits_present = true;
  for (const auto& r : workload) {
    std::vector<float> row(static_cast<std::size_t>(m.vocab));
    int32_t am = -1;
    if (rs_logits(ctx, r.id, row.data(), &am) != RS_OK) {
      logits_present = false;
      continue;
    }
    for (std::size_t i = 0; i < row.size(); ++i)
      max_diff = std::max(max_diff, static_cast<double>(std::fabs(row[i] - eng_logits[r.id][i])));
    argmax_equal = argmax_equal && am == eng_am[r.id];
  }
  std::set<std::uint64_t> enc_seen, stage_seen;
  bool ordered = true, once = true;
  double last = -1;
  int chunk_complete = 0;
  for (const rs_event& e : be.events) {
    ordered = ordered && e.time_ms >= last;
    last = e.time_ms;
    if (e.kind == RS_EV_ENCODE_DONE) once = once && enc_seen.insert(e.tag).second;
    if (e.kind == RS_EV_STAGE_DONE) once = once && stage_seen.insert(e.tag).second;
    if (e.kind == RS_EV_CHUNK_COMPLETE) ++chunk_complete;
  }
  const bool complete = enc_seen == be.encodes_open && stage_seen == be.stages_open;
  std::printf("{\"decisions_equal\": %s, \"logits_present\": %s, \"logits_max_abs_diff\": %.9g, "
              "\"argmax_equal\": %s, \"events\": %zu, \"encodes\": %zu, \"chunks\": %zu, "
              "\"chunk_complete_events\": %d, \"events_ordered\": %s, \"events_once\": %s, "
              "\"events_complete\": %s}\n",
              decisions_equal ? "true" : "false", logits_present ? "true" : "false", max_diff,
              argmax_equal ? "true" : "false", be.events.size(), be.encodes_open.size(), be.stages_open.size(),
              chunk_complete, ordered ? "true" : "false", once ? "true" : "false", complete ? "true" : "false");
  if (!decisions_equal) {
    std::fprintf(stderr, "--- ours\n%s\n--- reference\n%s\n", our_log.c_str(), ref_log);
  }
  rs_free(ref_log);
  rs_free(eng_log);
  rs_free(eng_journal);
  check(rs_ctx_destroy(ctx), "rs_ctx_destroy");
  return 0;
}
