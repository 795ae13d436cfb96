// rserve-b200 — device entry points of the C-ABI (include/rserve.h).
#include <cstring>
#include <memory>
#include <sstream>
#include <unordered_map>

#include "device_backend.cuh"
#include "capi_ctx.cuh"
#include "device_context.cuh"
#include "host/config_bridge.hpp"
#include "host/decision_log.hpp"
#include "host/status.hpp"
#include "lmmsim/simengine.hpp"
#include "rserve.h"

using namespace rserve;

extern "C" {

rs_status rs_model_preset(int32_t preset, rs_model_config* out) {
  return guarded([&] {
    rs_model_config m{};
    m.patch_dim = 3 * 2 * 14 * 14;
    m.rope_theta_llm = 1000000.f;
    m.rope_theta_vit = 10000.f;
    m.rms_eps = 1e-6f;
    m.weight_seed = 20250928;
    m.vit_window = 4;  // 112 px windows = 4x4 merged units = 8x8 patches
    switch (preset) {
      case RS_MODEL_TINY:
        m.vit_dim = 256; m.vit_layers = 4; m.vit_heads = 4; m.vit_ff = 1024; m.vit_fullatt_every = 2;
        m.llm_dim = 512; m.llm_layers = 4; m.llm_q_heads = 8; m.llm_kv_heads = 2;
        m.llm_head_dim = 64; m.llm_ff = 1536; m.vocab = 4096;
        break;
      case RS_MODEL_QWEN25VL_7B:
        m.vit_dim = 1280; m.vit_layers = 32; m.vit_heads = 16; m.vit_ff = 3420; m.vit_fullatt_every = 8;
        m.llm_dim = 3584; m.llm_layers = 28; m.llm_q_heads = 28; m.llm_kv_heads = 4;
        m.llm_head_dim = 128; m.llm_ff = 18944; m.vocab = 152064;
        break;
      case RS_MODEL_QWEN25VL_72B_LLM:
        m.vit_dim = 1280; m.vit_layers = 32; m.vit_heads = 16; m.vit_ff = 3420; m.vit_fullatt_every = 8;
        m.llm_dim = 8192; m.llm_layers = 80; m.llm_q_heads = 64; m.llm_kv_heads = 8;
        m.llm_head_dim = 128; m.llm_ff = 29568; m.vocab = 152064;
        break;
      default:
        throw lmmsim::ConfigError("model preset: unknown value " + std::to_string(preset));
    }
    *out = m;
  });
}

rs_status rs_ctx_create(const rs_model_config* model, const rs_ctx_options* opt, rs_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<rs_ctx>();
    c->ctx = std::make_unique<Context>(*model, *opt);
    const Shapes& s = c->ctx->shapes();
    if (opt->with_vit) {
      RS_CUDA_CHECK(cudaMalloc(&c->manual_out, opt->max_encode_tokens * s.d * sizeof(bf16)));
      RS_CUDA_CHECK(cudaMalloc(&c->manual_in, 4 * opt->max_encode_tokens * s.pdim * sizeof(bf16)));
    }
    RS_CUDA_CHECK(cudaMalloc(&c->manual_x, opt->max_chunk_tokens * s.d * sizeof(bf16)));
    *out = c.release();
  });
}

rs_status rs_ctx_destroy(rs_ctx* c) {
  return guarded([&] {
    if (c == nullptr) return;
    cudaDeviceSynchronize();
    rs_async_teardown(c);
    if (c->manual_out) cudaFree(c->manual_out);
    if (c->manual_in) cudaFree(c->manual_in);
    if (c->manual_x) cudaFree(c->manual_x);
    delete c;
  });
}

rs_status rs_request_create(rs_ctx* c, uint64_t id, const char* layout, const int32_t* text_ids) {
  return guarded([&] {
    rs_ctx& x = need(c);
    lmmsim::RequestSpec req;
    req.id = id;
    req.segments = lmmsim::parse_layout(layout ? layout : "");
    lmmsim::create_tracker(x.registry, req, static_cast<std::uint32_t>(x.ctx->shapes().d));
    try {
      x.ctx->create_request(req, text_ids, 0, x.ctx->tracker_stream());
    } catch (...) {
      x.registry.erase(id);
      throw;
    }
  });
}

rs_status rs_mark_encoded(rs_ctx* c, uint64_t id, uint64_t start, uint64_t end,
                          const void* embeddings_dev) {
  return guarded([&] {
    rs_ctx& x = need(c);
    // Host mirror first: alignment / double-encode errors exactly as the
    // reference raises them (tracker.hpp:83-105), before any device write.
    lmmsim::on_embeddings_ready(x.registry, id, lmmsim::TokenRange{start, end});
    x.ctx->scatter_items(x.ctx->get(id), {lmmsim::TokenRange{start, end}},
                         static_cast<const bf16*>(embeddings_dev), x.ctx->tracker_stream());
  });
}

rs_status rs_schedulable(rs_ctx* c, uint64_t id, uint64_t* host_count, uint64_t* device_count) {
  return guarded([&] {
    rs_ctx& x = need(c);
    lmmsim::EmbeddingTracker& t = x.registry.get(id);
    if (host_count) *host_count = t.schedulable_tokens();
    if (device_count) *device_count = x.ctx->device_schedulable(x.ctx->get(id), t.prefilled_frontier());
  });
}

rs_status rs_advance_prefill(rs_ctx* c, uint64_t id, uint64_t n, uint64_t* s, uint64_t* e) {
  return guarded([&] {
    rs_ctx& x = need(c);
    const lmmsim::TokenRange r = x.registry.get(id).advance_prefill(n);
    if (s) *s = r.start;
    if (e) *e = r.end;
  });
}

rs_status rs_release(rs_ctx* c, uint64_t id, uint64_t start, uint64_t end) {
  return guarded([&] {
    rs_ctx& x = need(c);
    lmmsim::EmbeddingTracker& t = x.registry.get(id);
    t.release(lmmsim::TokenRange{start, end});
    RS_CUDA_CHECK(cudaDeviceSynchronize());  // manual mode: readers are done
    x.ctx->release_prefix(x.ctx->get(id), t.released_tokens(), nullptr);
  });
}

rs_status rs_request_erase(rs_ctx* c, uint64_t id) {
  return guarded([&] {
    rs_ctx& x = need(c);
    x.registry.erase(id);
    RS_CUDA_CHECK(cudaDeviceSynchronize());
    x.ctx->erase_request(id, nullptr);
  });
}

rs_status rs_read_bitmap(rs_ctx* c, uint64_t id, uint32_t* out, uint64_t n_words) {
  return guarded([&] {
    rs_ctx& x = need(c);
    DevRequest& r = x.ctx->get(id);
    const std::uint64_t words = (r.total + 31) / 32;
    if (n_words < words) throw lmmsim::InputError("rs_read_bitmap: buffer too small");
    RS_CUDA_CHECK(cudaDeviceSynchronize());
    RS_CUDA_CHECK(cudaMemcpy(out, r.bitmap, words * 4, cudaMemcpyDeviceToHost));
  });
}

rs_status rs_read_slots(rs_ctx* c, uint64_t id, uint64_t start, uint64_t end, void* out) {
  return guarded([&] {
    rs_ctx& x = need(c);
    DevRequest& r = x.ctx->get(id);
    if (end > r.total || start > end) throw lmmsim::InputError("rs_read_slots: bad range");
    RS_CUDA_CHECK(cudaDeviceSynchronize());
    const std::size_t row = static_cast<std::size_t>(x.ctx->shapes().d) * sizeof(bf16);
    for (std::uint64_t t = start; t < end; ++t) {
      if (r.slot_pages[t / kPageTokens] < 0) throw lmmsim::InputError("rs_read_slots: token released");
      RS_CUDA_CHECK(cudaMemcpy(static_cast<std::uint8_t*>(out) + (t - start) * row,
                               x.ctx->slab() + r.slab_row(t) * x.ctx->shapes().d, row,
                               cudaMemcpyDeviceToHost));
    }
  });
}

rs_status rs_tracker_stats(rs_ctx* c, uint64_t id, uint64_t out[6]) {
  return guarded([&] {
    rs_ctx& x = need(c);
    const lmmsim::EmbeddingTracker& t = x.registry.get(id);
    out[0] = t.live_embedding_tokens();
    out[1] = t.peak_live_embedding_tokens();
    out[2] = t.released_tokens();
    out[3] = t.prefilled_frontier();
    out[4] = t.schedulable_tokens();
    out[5] = t.all_encoded() ? 1 : 0;
  });
}

rs_status rs_encode(rs_ctx* c, const uint64_t* items, int32_t n_items, const void* patches,
                    int32_t patches_on_host, void** out_embeddings_dev) {
  return guarded([&] {
    rs_ctx& x = need(c);
    std::vector<lmmsim::TokenRange> its;
    std::uint64_t tokens = 0;
    for (int i = 0; i < n_items; ++i) {
      its.push_back({items[2 * i], items[2 * i + 1]});
      tokens += items[2 * i + 1] - items[2 * i];
    }
    if (tokens > x.ctx->options().max_encode_tokens)
      throw lmmsim::ConfigError("rs_encode: batch exceeds max_encode_tokens");
    const Shapes& s = x.ctx->shapes();
    cudaStream_t st = x.ctx->aux_stream();
    const bf16* src = static_cast<const bf16*>(patches);
    if (patches_on_host) {
      RS_CUDA_CHECK(cudaMemcpyAsync(x.manual_in, patches, 4 * tokens * s.pdim * sizeof(bf16),
                                    cudaMemcpyHostToDevice, st));
      src = x.manual_in;
    }
    DevRequest dummy;
    const VitBatchPlan plan = x.ctx->plan_batch(dummy, its);
    bf16* dst = *out_embeddings_dev != nullptr ? static_cast<bf16*>(*out_embeddings_dev) : x.manual_out;
    x.ctx->encode(plan, src, dst, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    *out_embeddings_dev = dst;
  });
}

rs_status rs_prefill_chunk(rs_ctx* c, const uint64_t* slices, int32_t n_slices) {
  return guarded([&] {
    rs_ctx& x = need(c);
    // Validate every slice on scratch copies of the trackers first (frontier,
    // readiness — the reference's DependencyViolation text — and the chunk
    // size), so a rejected chunk leaves no tracker advanced.
    std::unordered_map<lmmsim::RequestId, lmmsim::EmbeddingTracker> scratch;
    std::vector<SliceRef> refs;
    std::uint64_t total = 0;
    for (int i = 0; i < n_slices; ++i) {
      const lmmsim::RequestId id = slices[3 * i];
      const std::uint64_t b = slices[3 * i + 1], e = slices[3 * i + 2];
      auto it = scratch.find(id);
      if (it == scratch.end()) it = scratch.emplace(id, x.registry.get(id)).first;
      lmmsim::EmbeddingTracker& t = it->second;
      if (b != t.prefilled_frontier() || e <= b)
        throw lmmsim::InternalError("rs_prefill_chunk: slice [" + lmmsim::format_u64(b) + "," +
                                    lmmsim::format_u64(e) + ") of request " +
                                    lmmsim::format_u64(id) + " does not start at its frontier");
      t.advance_prefill(e - b);  // DependencyViolation when not ready
      refs.push_back({&x.ctx->get(id), b, e});
      total += e - b;
    }
    if (total > x.ctx->options().max_chunk_tokens)
      throw lmmsim::ConfigError("rs_prefill_chunk: chunk exceeds max_chunk_tokens");
    for (int i = 0; i < n_slices; ++i)
      x.registry.get(slices[3 * i]).advance_prefill(slices[3 * i + 2] - slices[3 * i + 1]);
    cudaStream_t st = x.ctx->aux_stream();
    RS_CUDA_CHECK(cudaStreamSynchronize(x.ctx->tracker_stream()));
    x.ctx->prefill(refs, x.manual_x, st);
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    const int vocab = x.ctx->shapes().vocab;
    for (const SliceRef& r : refs) {
      if (r.end != r.req->total || !x.ctx->llm()->has_head()) continue;
      std::vector<float> row(static_cast<std::size_t>(vocab));
      x.ctx->copy_logits(r.req->slot, row.data(), st);
      std::int32_t am = 0;
      RS_CUDA_CHECK(cudaMemcpyAsync(&am, x.ctx->device_argmax() + r.req->slot, 4,
                                    cudaMemcpyDeviceToHost, st));
      RS_CUDA_CHECK(cudaStreamSynchronize(st));
      x.logits[r.req->id] = std::move(row);
      x.argmax[r.req->id] = am;
    }
  });
}

rs_status rs_logits(rs_ctx* c, uint64_t id, float* out_host, int32_t* out_argmax) {
  return guarded([&] {
    rs_ctx& x = need(c);
    const auto it = x.logits.find(id);
    if (it == x.logits.end())
      throw lmmsim::RegistryError("no first-token logits for request " + lmmsim::format_u64(id));
    if (out_host) std::memcpy(out_host, it->second.data(), it->second.size() * 4);
    if (out_argmax) *out_argmax = x.argmax.at(id);
  });
}

rs_status rs_synchronize(rs_ctx* c) {
  return guarded([&] {
    need(c);
    RS_CUDA_CHECK(cudaDeviceSynchronize());
  });
}

rs_status rs_engine_run(rs_ctx* c, const char* workload_text, const rs_sim_config* cfg,
                        const rs_run_options* opt, char** out_result, char** out_journal,
                        rs_run_stats* out_stats) {
  return guarded([&] {
    rs_ctx& x = need(c);
    std::vector<lmmsim::RequestSpec> wl = parse_workload_text(workload_text);
    lmmsim::SimConfig sc = to_sim_config(*cfg);
    sc.hidden_size = static_cast<std::uint32_t>(x.ctx->shapes().d);
    const bool realtime = opt != nullptr && opt->clock == 1;
    const bool e2e = opt != nullptr && opt->e2e != 0;
    DeviceBackend backend(*x.ctx, sc, realtime, e2e, opt ? opt->payload_seed : 0,
                          opt != nullptr && opt->serialize != 0);
    if (opt != nullptr && opt->payload_text != nullptr) {
      PayloadSpec spec = parse_payload(opt->payload_text);
      validate_payload(spec, wl, x.ctx->shapes().vocab);
      backend.set_payload(std::move(spec));
    }
    if (opt != nullptr && opt->keep_kv != 0) {
      if (!x.ctx->llm() || !x.ctx->llm()->has_head())
        throw lmmsim::ConfigError("keep_kv: the context holds no LM head");
      backend.set_keep_kv(true);
    }
    backend.prepare(wl);
    lmmsim::PipelineEngine engine(wl, sc, backend);
    backend.start();
    const lmmsim::SimResult res = engine.run();  // ends with backend.finish()
    backend.collect();
    for (const auto& [id, row] : backend.logits()) x.logits[id] = row;
    for (const auto& [id, am] : backend.argmax()) x.argmax[id] = am;
    std::vector<ReleaseRecord> rel;
    for (const lmmsim::ReleaseEvent& e : engine.releases()) rel.push_back({e.chunk, e.id, e.range});
    if (out_result) *out_result = c_string(render_decision_log(res, rel, true));
    if (out_journal) *out_journal = c_string(render_journal(engine.journal()));
    if (out_stats) *out_stats = backend.stats();
  });
}

rs_status rs_decode(rs_ctx* c, const uint64_t* request_ids, int32_t n_requests, int32_t n_steps,
                    int32_t* out_tokens, float* out_logits, double* out_ms) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (n_requests <= 0 || n_steps <= 0 || request_ids == nullptr || out_tokens == nullptr)
      throw lmmsim::ConfigError("rs_decode: need requests, steps > 0 and an output buffer");
    std::vector<lmmsim::RequestId> ids(request_ids, request_ids + n_requests);
    const double ms = x.ctx->decode(ids, n_steps, out_tokens, out_logits, x.ctx->aux_stream());
    if (out_ms) *out_ms = ms;
  });
}

rs_status rs_decode_release(rs_ctx* c, uint64_t request_id) {
  return guarded([&] {
    rs_ctx& x = need(c);
    RS_CUDA_CHECK(cudaDeviceSynchronize());
    x.ctx->free_kept(request_id);
  });
}

}  // extern "C"

extern "C" {

rs_status rs_kv_image_bytes(rs_ctx* c, uint64_t tokens, uint64_t* out_bytes) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (out_bytes == nullptr) throw lmmsim::ConfigError("rs_kv_image_bytes: null output");
    *out_bytes = x.ctx->kv_image_bytes(tokens);
  });
}

rs_status rs_kv_export(rs_ctx* c, uint64_t request_id, void* dst_dev, uint64_t cap_bytes, rs_kv_meta* out_meta,
                       void* stream) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (dst_dev == nullptr || out_meta == nullptr) throw lmmsim::ConfigError("rs_kv_export: null buffer / meta");
    cudaStream_t st = stream != nullptr ? static_cast<cudaStream_t>(stream) : x.ctx->aux_stream();
    x.ctx->export_kv(request_id, dst_dev, cap_bytes, out_meta, st);
  });
}

rs_status rs_kv_import(rs_ctx* c, uint64_t request_id, const rs_kv_meta* meta, const void* src_dev, void* stream) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (src_dev == nullptr || meta == nullptr) throw lmmsim::ConfigError("rs_kv_import: null image / meta");
    cudaStream_t st = stream != nullptr ? static_cast<cudaStream_t>(stream) : x.ctx->aux_stream();
    x.ctx->import_kv(request_id, *meta, src_dev, st);
  });
}

}  // extern "C"

// ---- tensor parallelism across GPUs -------------------------------------------
extern "C" {

rs_status rs_tp_buffer(rs_ctx* c, void** out_dev_ptr, void* out_ipc_handle) {
  return guarded([&] {
    rs_ctx& x = need(c);
    x.ctx->tp_buffer(out_dev_ptr, static_cast<cudaIpcMemHandle_t*>(out_ipc_handle));
  });
}

rs_status rs_tp_connect(rs_ctx* c, const void* const* peer_ptrs, const void* ipc_handles) {
  return guarded([&] {
    rs_ctx& x = need(c);
    x.ctx->tp_connect(peer_ptrs, static_cast<const cudaIpcMemHandle_t*>(ipc_handles));
  });
}

rs_status rs_kv_request_create(rs_ctx* c, uint64_t id, const char* layout) {
  return guarded([&] {
    rs_ctx& x = need(c);
    lmmsim::RequestSpec req;
    req.id = id;
    req.segments = lmmsim::parse_layout(layout ? layout : "");
    req.validate();
    x.ctx->create_kv_request(req, x.ctx->aux_stream());
  });
}

rs_status rs_tp_prefill(rs_ctx* c, const uint64_t* slices, int32_t n_slices, void* x_dev, void* stream) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (x_dev == nullptr || slices == nullptr || n_slices <= 0)
      throw lmmsim::ConfigError("rs_tp_prefill: need slices and the chunk's input rows");
    std::vector<SliceRef> refs;
    std::uint64_t total = 0;
    for (int i = 0; i < n_slices; ++i) {
      const std::uint64_t b = slices[3 * i + 1], e = slices[3 * i + 2];
      DevRequest& r = x.ctx->get(slices[3 * i]);
      if (e <= b || e > r.total)
        throw lmmsim::InternalError("rs_tp_prefill: slice [" + lmmsim::format_u64(b) + "," + lmmsim::format_u64(e) +
                                    ") outside request " + lmmsim::format_u64(r.id));
      refs.push_back({&r, b, e});
      total += e - b;
    }
    if (total > x.ctx->options().max_chunk_tokens)
      throw lmmsim::ConfigError("rs_tp_prefill: chunk exceeds max_chunk_tokens");
    cudaStream_t st = stream != nullptr ? static_cast<cudaStream_t>(stream) : x.ctx->aux_stream();
    x.ctx->prefill(refs, static_cast<bf16*>(x_dev), st);
  });
}

rs_status rs_tp_logits(rs_ctx* c, uint64_t id, float* out_host, int32_t* out_argmax) {
  return guarded([&] {
    rs_ctx& x = need(c);
    if (!x.ctx->llm()->has_head()) throw lmmsim::ConfigError("rs_tp_logits: this rank holds no LM head");
    DevRequest& r = x.ctx->get(id);
    cudaStream_t st = x.ctx->aux_stream();
    if (out_host) x.ctx->copy_logits(r.slot, out_host, st);
    if (out_argmax)
      RS_CUDA_CHECK(cudaMemcpyAsync(out_argmax, x.ctx->device_argmax() + r.slot, 4, cudaMemcpyDeviceToHost, st));
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
