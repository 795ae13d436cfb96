// rserve-b200 — canonical decision log of an engine run.
//
// The text form of a SimResult (+ release order) used to compare the B200
// engine with the reference bit for bit: doubles use shortest round-trip
// formatting, so two equal logs mean equal decisions AND equal (virtual)
// times. Format (one record per line):
//   result chunks=.. encode_batches=.. transfers=.. [first_arrival=.. last_completion=..]
//   req id=.. prompt=.. completed=.. released=.. peak_live=.. [arrival=.. ... prefill_span=..]
//   slice req=.. chunk=.. start=.. end=..
//   trace kind=.. res=.. name=.. owners=a,b tokens=.. [start=.. dur=..]
//   release chunk=.. req=.. start=.. end=..
// Bracketed fields are omitted when times are excluded (real-clock replay).
#pragma once

#include <string>
#include <vector>

#include "lmmsim/simengine.hpp"

namespace rserve {

struct ReleaseRecord {
  std::size_t chunk;
  lmmsim::RequestId id;
  lmmsim::TokenRange range;
};

inline std::string render_decision_log(const lmmsim::SimResult& r,
                                       const std::vector<ReleaseRecord>& releases,
                                       bool with_times) {
  using lmmsim::format_double;
  using lmmsim::format_u64;
  std::string out;
  auto kv = [&out](const char* key, const std::string& v) {
    out += ' ';
    out += key;
    out += '=';
    out += v;
  };
  out += "result";
  kv("chunks", format_u64(r.chunk_count));
  kv("encode_batches", format_u64(r.encode_batch_count));
  kv("transfers", format_u64(r.transfer_count));
  if (with_times) {
    kv("first_arrival", format_double(r.first_arrival_ms));
    kv("last_completion", format_double(r.last_completion_ms));
  }
  out += '\n';
  for (const lmmsim::RequestRecord& q : r.requests) {
    out += "req";
    kv("id", format_u64(q.id));
    kv("prompt", format_u64(q.prompt_tokens));
    kv("completed", q.completed ? "1" : "0");
    kv("released", format_u64(q.released_tokens));
    kv("peak_live", format_u64(q.peak_live_tokens));
    if (with_times) {
      const std::pair<const char*, double> times[] = {
          {"arrival", q.arrival_ms},
          {"first_token", q.first_token_ms},
          {"first_admission", q.first_admission_ms},
          {"encode_dispatch", q.encode_dispatch_ms},
          {"embeddings_ready", q.embeddings_ready_ms},
          {"ttft", q.ttft_ms},
          {"queue", q.queue_delay_ms},
          {"encode_span", q.encode_span_ms},
          {"prefill_span", q.prefill_span_ms},
      };
      for (const auto& [k, v] : times) kv(k, format_double(v));
    }
    out += '\n';
    for (const auto& [chunk, range] : q.slices) {
      out += "slice";
      kv("req", format_u64(q.id));
      kv("chunk", format_u64(chunk));
      kv("start", format_u64(range.start));
      kv("end", format_u64(range.end));
      out += '\n';
    }
  }
  for (const lmmsim::TraceEvent& e : r.trace) {
    out += "trace";
    kv("kind", e.kind == lmmsim::TraceKind::Encode     ? "encode"
               : e.kind == lmmsim::TraceKind::Transfer ? "transfer"
                                                        : "stage");
    kv("res", std::to_string(e.resource));
    kv("name", e.name);
    std::string owners;
    for (std::size_t i = 0; i < e.owners.size(); ++i)
      owners += (i ? "," : "") + format_u64(e.owners[i]);
    kv("owners", owners);
    kv("tokens", format_u64(e.tokens));
    if (with_times) {
      kv("start", format_double(e.start_ms));
      kv("dur", format_double(e.dur_ms));
    }
    out += '\n';
  }
  for (const ReleaseRecord& rel : releases) {
    out += "release";
    kv("chunk", format_u64(rel.chunk));
    kv("req", format_u64(rel.id));
    kv("start", format_u64(rel.range.start));
    kv("end", format_u64(rel.range.end));
    out += '\n';
  }
  return out;
}

inline std::string render_journal(const std::vector<lmmsim::JournalEntry>& j) {
  std::string out;
  for (const lmmsim::JournalEntry& e : j) {
    out += std::to_string(e.kind) + ' ' + std::to_string(e.a) + ' ' +
           lmmsim::format_u64(e.b) + ' ' + lmmsim::format_double(e.time_ms) + '\n';
  }
  return out;
}

}  // namespace rserve
