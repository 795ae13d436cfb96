// rserve-b200 — the asynchronous seam of the C-ABI (include/rserve.h
// "caller-owned event loop"): POD request creation, non-blocking encode /
// embeddings-ready / prefill / release launches on the context's streams,
// and rs_poll completions in the reference's event classes
// (simengine.hpp:211-248), so a host scheduler that owns its event loop — the
// reference's Simulation handlers (simengine.hpp:275-441) — can drive the
// device directly.
#include <algorithm>
#include <cstring>
#include <thread>

#include "capi_ctx.cuh"
#include "device_context.cuh"
#include "host/status.hpp"
#include "lmmsim/token_sched.hpp"
#include "rserve.h"

using namespace rserve;

namespace {

AsyncState& async_of(rs_ctx& x) {
  AsyncState& a = x.async;
  if (a.enc == nullptr) {
    int lo = 0, hi = 0;
    RS_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // encoder work first (as the engine does): the ViT's kernels take SMs
    // ahead of the prefill stream's, so embeddings run ahead of prefill
    RS_CUDA_CHECK(cudaStreamCreateWithPriority(&a.enc, cudaStreamNonBlocking, hi));
    RS_CUDA_CHECK(cudaStreamCreateWithPriority(&a.stage, cudaStreamNonBlocking, lo));
    RS_CUDA_CHECK(cudaEventCreate(&a.origin));
    RS_CUDA_CHECK(cudaEventCreateWithFlags(&a.tracker_snap, cudaEventDisableTiming));
  }
  return a;
}

cudaEvent_t timing_event(AsyncState& a) {
  if (!a.timing_pool.empty()) {
    cudaEvent_t e = a.timing_pool.back();
    a.timing_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  RS_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void stamp_origin(AsyncState& a, cudaStream_t st) {
  if (a.origin_set) return;
  RS_CUDA_CHECK(cudaEventRecord(a.origin, st));
  a.origin_set = true;
}

int acquire_staging(rs_ctx& x, AsyncState& a) {
  for (std::size_t i = 0; i < a.staging.size(); ++i)
    if (!a.staging_busy[i]) {
      a.staging_busy[i] = true;
      return static_cast<int>(i);
    }
  void* p = nullptr;
  RS_CUDA_CHECK(cudaMalloc(&p, x.ctx->options().max_encode_tokens * x.ctx->shapes().d * sizeof(bf16)));
  a.staging.push_back(static_cast<bf16*>(p));
  a.staging_guard.push_back(nullptr);
  a.staging_busy.push_back(true);
  return static_cast<int>(a.staging.size() - 1);
}

cudaStream_t pick(void* stream, cudaStream_t dflt) {
  return stream != nullptr ? static_cast<cudaStream_t>(stream) : dflt;
}

}  // namespace

void rs_async_teardown(rs_ctx* c) {
  AsyncState& a = c->async;
  if (a.enc == nullptr) return;
  cudaDeviceSynchronize();
  for (AsyncOp& op : a.pending) cudaEventDestroy(op.done);
  for (auto& [tag, e] : a.encodes) cudaEventDestroy(e.done);
  for (cudaEvent_t e : a.timing_pool) cudaEventDestroy(e);
  for (bf16* p : a.staging) cudaFree(p);
  cudaEventDestroy(a.origin);
  cudaEventDestroy(a.tracker_snap);
  cudaStreamDestroy(a.enc);
  cudaStreamDestroy(a.stage);
  a = AsyncState{};
}

extern "C" {

rs_status rs_request_create_segments(rs_ctx* c, uint64_t id, const rs_segment* segs, int32_t n_segs,
                                     const int32_t* text_ids) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (n_segs < 0 || (n_segs > 0 && segs == nullptr))
      throw lmmsim::InputError("rs_request_create_segments: bad segment array");
    lmmsim::RequestSpec req;
    req.id = id;
    for (int i = 0; i < n_segs; ++i) {
      if (segs[i].kind != RS_SEG_TEXT && segs[i].kind != RS_SEG_MULTIMODAL)
        throw lmmsim::InputError("rs_request_create_segments: segment " + std::to_string(i) +
                                 " has unknown kind " + std::to_string(segs[i].kind));
      req.segments.push_back({segs[i].kind == RS_SEG_TEXT ? lmmsim::SegmentKind::Text
                                                          : lmmsim::SegmentKind::Multimodal,
                              segs[i].tokens});
    }
    req.validate();  // the reference's InputError texts (request.hpp:94-102)
    lmmsim::create_tracker(x.registry, req, static_cast<std::uint32_t>(x.ctx->shapes().d));
    try {
      x.ctx->create_request(req, text_ids, 0, x.ctx->tracker_stream());
    } catch (...) {
      x.registry.erase(id);
      throw;
    }
  });
}

rs_status rs_encode_batch_async(rs_ctx* c, uint64_t id, const uint64_t* items, int32_t n_items,
                                const void* patches, int32_t patches_on_host, void* stream, uint64_t tag) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    if (a.encodes.count(tag)) throw lmmsim::InputError("rs_encode_batch_async: tag " + std::to_string(tag) + " in flight");
    DevRequest& r = x.ctx->get(id);
    std::vector<lmmsim::TokenRange> its;
    std::uint64_t tokens = 0;
    for (int i = 0; i < n_items; ++i) {
      its.push_back({items[2 * i], items[2 * i + 1]});
      tokens += items[2 * i + 1] - items[2 * i];
    }
    if (its.empty()) throw lmmsim::InputError("rs_encode_batch_async: empty batch");
    if (tokens > x.ctx->options().max_encode_tokens)
      throw lmmsim::ConfigError("rs_encode_batch_async: batch exceeds max_encode_tokens");
    const Shapes& s = x.ctx->shapes();
    cudaStream_t st = pick(stream, a.enc);
    stamp_origin(a, st);
    const int si = acquire_staging(x, a);
    if (a.staging_guard[static_cast<std::size_t>(si)] != nullptr)
      RS_CUDA_CHECK(cudaStreamWaitEvent(st, a.staging_guard[static_cast<std::size_t>(si)], 0));
    const bf16* src = static_cast<const bf16*>(patches);
    bf16* tmp = nullptr;
    if (patches_on_host) {
      const std::size_t bytes = 4 * tokens * s.pdim * sizeof(bf16);
      RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tmp), bytes, st));
      RS_CUDA_CHECK(cudaMemcpyAsync(tmp, patches, bytes, cudaMemcpyHostToDevice, st));
      src = tmp;
    }
    const VitBatchPlan plan = x.ctx->plan_batch(r, its);
    x.ctx->encode(plan, src, a.staging[static_cast<std::size_t>(si)], st);
    if (tmp != nullptr) RS_CUDA_CHECK(cudaFreeAsync(tmp, st));
    AsyncOp op{RS_EV_ENCODE_DONE, tag, a.seq++, timing_event(a), {}};
    RS_CUDA_CHECK(cudaEventRecord(op.done, st));
    cudaEvent_t order = x.ctx->new_event();
    RS_CUDA_CHECK(cudaEventRecord(order, st));
    a.encodes[tag] = AsyncEncode{si, id, std::move(its), order};
    a.pending.push_back(std::move(op));
  });
}

rs_status rs_embeddings_ready(rs_ctx* c, uint64_t tag) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    auto it = a.encodes.find(tag);
    if (it == a.encodes.end()) throw lmmsim::InputError("rs_embeddings_ready: unknown encode tag " + std::to_string(tag));
    AsyncEncode e = it->second;
    // host mirror first, item by item in item order (simengine.hpp:329-333):
    // AlignmentError / DoubleEncodeError exactly as the reference raises them
    for (const lmmsim::TokenRange& r : e.items) lmmsim::on_embeddings_ready(x.registry, e.request, r);
    a.encodes.erase(it);
    cudaStream_t st = x.ctx->tracker_stream();
    RS_CUDA_CHECK(cudaStreamWaitEvent(st, e.done, 0));
    x.ctx->scatter_items(x.ctx->get(e.request), e.items, a.staging[static_cast<std::size_t>(e.staging)], st);
    cudaEvent_t g = x.ctx->new_event();
    RS_CUDA_CHECK(cudaEventRecord(g, st));
    a.staging_guard[static_cast<std::size_t>(e.staging)] = g;
    a.staging_busy[static_cast<std::size_t>(e.staging)] = false;
  });
}

rs_status rs_prefill_chunk_async(rs_ctx* c, const uint64_t* slices, int32_t n_slices, void* stream,
                                 uint64_t tag) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    if (n_slices <= 0) throw lmmsim::InputError("rs_prefill_chunk_async: empty chunk");
    // validate on scratch trackers, then advance (no partial state on error)
    std::unordered_map<lmmsim::RequestId, lmmsim::EmbeddingTracker> scratch;
    std::vector<SliceRef> refs;
    std::uint64_t total = 0;
    for (int i = 0; i < n_slices; ++i) {
      const lmmsim::RequestId id = slices[3 * i];
      const std::uint64_t b = slices[3 * i + 1], e = slices[3 * i + 2];
      auto sit = scratch.find(id);
      if (sit == scratch.end()) sit = scratch.emplace(id, x.registry.get(id)).first;
      if (b != sit->second.prefilled_frontier() || e <= b)
        throw lmmsim::InternalError("rs_prefill_chunk_async: slice [" + lmmsim::format_u64(b) + "," +
                                    lmmsim::format_u64(e) + ") of request " + lmmsim::format_u64(id) +
                                    " does not start at its frontier");
      sit->second.advance_prefill(e - b);  // DependencyViolation when not ready
      refs.push_back({&x.ctx->get(id), b, e});
      total += e - b;
    }
    if (total > x.ctx->options().max_chunk_tokens)
      throw lmmsim::ConfigError("rs_prefill_chunk_async: chunk exceeds max_chunk_tokens");
    for (int i = 0; i < n_slices; ++i)
      x.registry.get(slices[3 * i]).advance_prefill(slices[3 * i + 2] - slices[3 * i + 1]);
    cudaStream_t st = pick(stream, a.stage);
    stamp_origin(a, st);
    // the chunk reads slots scattered on the tracker stream so far
    RS_CUDA_CHECK(cudaEventRecord(a.tracker_snap, x.ctx->tracker_stream()));
    RS_CUDA_CHECK(cudaStreamWaitEvent(st, a.tracker_snap, 0));
    bf16* xb = nullptr;
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&xb), total * x.ctx->shapes().d * sizeof(bf16), st));
    x.ctx->prefill(refs, xb, st);
    RS_CUDA_CHECK(cudaFreeAsync(xb, st));
    AsyncOp op{RS_EV_STAGE_DONE, tag, a.seq++, timing_event(a), {}};
    if (x.ctx->llm() && x.ctx->llm()->has_head())
      for (const SliceRef& r : refs)
        if (r.end == r.req->total) op.finished.push_back({r.req->id, r.req->slot});
    RS_CUDA_CHECK(cudaEventRecord(op.done, st));
    cudaEvent_t g = x.ctx->new_event();
    RS_CUDA_CHECK(cudaEventRecord(g, st));
    a.stage_guard[tag] = g;
    a.pending.push_back(std::move(op));
  });
}

rs_status rs_release_async(rs_ctx* c, uint64_t id, uint64_t start, uint64_t end, uint64_t after_tag) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    auto g = a.stage_guard.find(after_tag);
    if (g == a.stage_guard.end())
      throw lmmsim::InputError("rs_release_async: unknown chunk tag " + std::to_string(after_tag));
    lmmsim::EmbeddingTracker& t = x.registry.get(id);
    t.release(lmmsim::TokenRange{start, end});  // InternalError on out-of-order release
    // slot pages go back to the pool once the chunk that read them is done
    x.ctx->release_prefix(x.ctx->get(id), t.released_tokens(), g->second);
  });
}

rs_status rs_request_erase_async(rs_ctx* c, uint64_t id, uint64_t after_tag) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    auto g = a.stage_guard.find(after_tag);
    if (g == a.stage_guard.end())
      throw lmmsim::InputError("rs_request_erase_async: unknown chunk tag " + std::to_string(after_tag));
    x.registry.erase(id);
    x.ctx->erase_request(id, g->second);
  });
}

rs_status rs_poll(rs_ctx* c, rs_event* out, int32_t cap, int32_t wait, int32_t* n_out) {
  return guarded([&] {
    rs_ctx& x = need(c);
    AsyncState& a = async_of(x);
    *n_out = 0;
    if (cap <= 0) throw lmmsim::InputError("rs_poll: capacity must be positive");
    std::vector<rs_event> got;
    std::vector<std::uint64_t> seqs;
    for (;;) {
      for (std::size_t i = 0; i < a.pending.size() && static_cast<int>(got.size()) + 2 <= cap;) {
        AsyncOp& op = a.pending[i];
        const cudaError_t q = cudaEventQuery(op.done);
        if (q == cudaErrorNotReady) {
          ++i;
          continue;
        }
        RS_CUDA_CHECK(q);
        float ms = 0;
        RS_CUDA_CHECK(cudaEventElapsedTime(&ms, a.origin, op.done));
        got.push_back({op.kind, 0, op.tag, static_cast<double>(ms)});
        seqs.push_back(op.seq);
        if (!op.finished.empty()) {
          // the last stage: ChunkComplete at the same time (simengine.hpp:399)
          got.push_back({RS_EV_CHUNK_COMPLETE, 0, op.tag, static_cast<double>(ms)});
          seqs.push_back(op.seq);
          const int vocab = x.ctx->shapes().vocab;
          for (const auto& [rid, slot] : op.finished) {
            std::vector<float> row(static_cast<std::size_t>(vocab));
            x.ctx->copy_logits(slot, row.data(), a.stage);
            std::int32_t am = 0;
            RS_CUDA_CHECK(cudaMemcpyAsync(&am, x.ctx->device_argmax() + slot, 4, cudaMemcpyDeviceToHost, a.stage));
            RS_CUDA_CHECK(cudaStreamSynchronize(a.stage));
            x.logits[rid] = std::move(row);
            x.argmax[rid] = am;
          }
        }
        a.timing_pool.push_back(op.done);
        a.pending.erase(a.pending.begin() + static_cast<std::ptrdiff_t>(i));
      }
      if (!got.empty() || !wait || a.pending.empty()) break;
      std::this_thread::yield();
    }
    // completion order; equal times: encode class before stage class, then issue order
    std::vector<std::size_t> idx(got.size());
    for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](std::size_t p, std::size_t q) {
      if (got[p].time_ms != got[q].time_ms) return got[p].time_ms < got[q].time_ms;
      const int cp = got[p].kind <= RS_EV_TRANSFER_DONE ? 0 : 1, cq = got[q].kind <= RS_EV_TRANSFER_DONE ? 0 : 1;
      if (cp != cq) return cp < cq;
      return seqs[p] < seqs[q];
    });
    for (std::size_t i = 0; i < idx.size(); ++i) out[i] = got[idx[i]];
    *n_out = static_cast<int32_t>(idx.size());
  });
}

}  // extern "C"
