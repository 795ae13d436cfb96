// rserve-b200 — the C-ABI's opaque rs_ctx (shared by the capi_*.cu units).
#pragma once

#include <memory>
#include <unordered_map>
#include <vector>

#include "device_context.cuh"
#include "lmmsim/tracker.hpp"
#include "rserve.h"

struct rs_ctx {
  std::unique_ptr<rserve::Context> ctx;
  lmmsim::TrackerRegistry registry;  // host mirrors of the manual API
  rserve::bf16* manual_out = nullptr;        // rs_encode output
  rserve::bf16* manual_in = nullptr;         // rs_encode patches staging (host input)
  rserve::bf16* manual_x = nullptr;          // rs_prefill_chunk residual
  std::unordered_map<lmmsim::RequestId, std::vector<float>> logits;
  std::unordered_map<lmmsim::RequestId, std::int32_t> argmax;
};

inline rs_ctx& need(rs_ctx* c) {
  if (c == nullptr || !c->ctx) throw lmmsim::InputError("null rs_ctx");
  return *c;
}

