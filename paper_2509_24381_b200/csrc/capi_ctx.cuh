// rserve-b200 — the C-ABI's opaque rs_ctx (shared by the capi_*.cu units).
#pragma once

#include <memory>
#include <unordered_map>
#include <vector>

#include "device_context.cuh"
#include "lmmsim/tracker.hpp"
#include "rserve.h"

/// State of the asynchronous seam (capi_async.cu): non-blocking launches on
/// the context's encode / stage streams, completions reported by rs_poll.
struct AsyncOp {
  int kind;                 // RS_EV_*
  std::uint64_t tag;
  std::uint64_t seq;        // issue order (tie-break)
  cudaEvent_t done;         // timing event
  std::vector<std::pair<lmmsim::RequestId, int>> finished;  // prefill: (request, slot) whose prompt ends
};
struct AsyncEncode {
  int staging;
  lmmsim::RequestId request;
  std::vector<lmmsim::TokenRange> items;
  cudaEvent_t done;         // ordering event (scatter waits on it)
};
struct AsyncState {
  cudaStream_t enc = nullptr, stage = nullptr;
  cudaEvent_t origin = nullptr;
  bool origin_set = false;
  std::uint64_t seq = 0;
  std::vector<AsyncOp> pending;
  std::vector<cudaEvent_t> timing_pool;
  std::vector<rserve::bf16*> staging;
  std::vector<cudaEvent_t> staging_guard;  // last reader (scatter) of each buffer
  std::vector<bool> staging_busy;
  std::unordered_map<std::uint64_t, AsyncEncode> encodes;  // tag -> in-flight encode
  std::unordered_map<std::uint64_t, cudaEvent_t> stage_guard;  // chunk tag -> completion (release guards)
  cudaEvent_t tracker_snap = nullptr;
};

struct rs_ctx {
  std::unique_ptr<rserve::Context> ctx;
  lmmsim::TrackerRegistry registry;  // host mirrors of the manual API
  rserve::bf16* manual_out = nullptr;        // rs_encode output
  rserve::bf16* manual_in = nullptr;         // rs_encode patches staging (host input)
  rserve::bf16* manual_x = nullptr;          // rs_prefill_chunk residual
  std::unordered_map<lmmsim::RequestId, std::vector<float>> logits;
  std::unordered_map<lmmsim::RequestId, std::int32_t> argmax;
  AsyncState async;
};

/// Releases the asynchronous seam's streams, events and staging (capi_async.cu).
void rs_async_teardown(rs_ctx* c);

inline rs_ctx& need(rs_ctx* c) {
  if (c == nullptr || !c->ctx) throw lmmsim::InputError("null rs_ctx");
  return *c;
}

