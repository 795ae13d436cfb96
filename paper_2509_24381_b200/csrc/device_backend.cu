// rserve-b200 — the B200 ExecutionBackend (see device_backend.cuh).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "device_backend.cuh"
#include "kernels.cuh"

namespace rserve {
namespace {
// NVTX range over a launch call, named as the reference's TraceEvent for the
// same work (simengine.hpp:296-303,316-323,377-384): encode_r<id>_b<slot>,
// transfer_r<id>_b<slot>, chunk<k>_s<s> — nsys / ncu timelines line up with
// the Chrome trace the engine exports.
struct NvtxRange {
  explicit NvtxRange(const char* fmt, unsigned long long a, unsigned long long b) {
    char name[64];
    std::snprintf(name, sizeof name, fmt, a, b);
    nvtxRangePushA(name);
  }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

DeviceBackend::DeviceBackend(Context& ctx, const lmmsim::SimConfig& cfg, bool realtime, bool e2e,
                             std::uint64_t payload_seed, bool serialize_streams,
                             const ep::Remote* remote)
    : ctx_(ctx), cfg_(cfg), realtime_(realtime), e2e_(e2e), seed_(payload_seed), remote_(remote) {
  if (cfg.stages < 1) throw lmmsim::ConfigError("stages: must be >= 1");
  if (remote_ != nullptr) {
    remote_->topo.validate();
    if (cfg.encoder_workers != remote_->topo.encoders)
      throw lmmsim::ConfigError("encoder_workers: must equal the EP encoder ranks (" +
                                std::to_string(remote_->topo.encoders) + ")");
    if (cfg.stages != remote_->topo.stages)
      throw lmmsim::ConfigError("stages: must equal the EP prefill ranks (" +
                                std::to_string(remote_->topo.stages) + ")");
    if (remote_->topo.stages > 1 && ctx.llm()->has_head())
      throw lmmsim::ConfigError("EP: P0 must not hold the LM head when stages > 1");
  }
  const int workers = cfg.encoder_workers;
  const Shapes& s = ctx.shapes();
  // One prefill stream: all stages of this GPU share the SMs and the per-stage
  // scratch; each chunk owns its residual buffer so stages can interleave.
  // Stream priorities (RS_STREAM_PRIO = enc | prefill | none; default enc):
  // an encode batch unblocks prefill of its span, so its CTAs go first when
  // both streams have work pending; prefill fills the remaining SM time.
  int prio_lo = 0, prio_hi = 0;
  RS_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const char* prio = std::getenv("RS_STREAM_PRIO");
  const std::string pmode = prio != nullptr ? prio : "enc";
  const int enc_prio = pmode == "enc" ? prio_hi : prio_lo;
  const int stage_prio = pmode == "prefill" ? prio_hi : prio_lo;
  stage_streams_.resize(1);
  RS_CUDA_CHECK(cudaStreamCreateWithPriority(&stage_streams_[0], cudaStreamNonBlocking, stage_prio));
  // serialize (profiling; or RS_SERIALIZE=1): encoders share the prefill
  // stream, so per-kernel event times are not inflated by cross-stream queueing.
  const char* ser = std::getenv("RS_SERIALIZE");
  const bool serialize = serialize_streams || (ser != nullptr && ser[0] == '1');
  enc_streams_.resize(static_cast<std::size_t>(workers));
  for (auto& st : enc_streams_) {
    if (serialize) {
      st = stage_streams_[0];
      shared_streams_ = true;
    } else {
      RS_CUDA_CHECK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, enc_prio));
    }
  }
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
  const std::size_t max_tok = ctx.options().max_encode_tokens;
  for (int i = 0; i < workers * kRing; ++i) {
    void* p = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&p, max_tok * s.d * sizeof(bf16)));
    staging_.push_back(static_cast<bf16*>(p));
    staging_free_.push_back(nullptr);
    staging_busy_.push_back(false);
  }
  if (e2e_ && remote_ == nullptr) {
    for (int w = 0; w < workers; ++w) {
      void* p = nullptr;
      RS_CUDA_CHECK(cudaMalloc(&p, 4 * max_tok * s.pdim * sizeof(bf16)));
      enc_input_.push_back(static_cast<bf16*>(p));
    }
  }
  const int n_x = std::max(2, cfg.stages + 2);
  for (int i = 0; i < n_x; ++i) {
    void* p = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&p, ctx.options().max_chunk_tokens * s.d * sizeof(bf16)));
    xbufs_.push_back(static_cast<bf16*>(p));
    xbuf_guard_.push_back(nullptr);
    free_xbufs_.push_back(i);
  }
  RS_CUDA_CHECK(cudaEventCreate(&origin_));
  if (remote_ != nullptr) {
    RS_CUDA_CHECK(cudaStreamCreateWithFlags(&ctrl_stream_, cudaStreamNonBlocking));
    for (int i = 0; i < kCtrlRing; ++i) {
      void* d = nullptr;
      void* h = nullptr;
      RS_CUDA_CHECK(cudaMalloc(&d, ep::kCtrlBytes));
      RS_CUDA_CHECK(cudaMallocHost(&h, ep::kCtrlBytes));
      ctrl_dev_.push_back(d);
      ctrl_host_.push_back(static_cast<std::int64_t*>(h));
      ctrl_free_.push_back(nullptr);
    }
    RS_CUDA_CHECK(cudaMalloc(&header_sink_, ep::kHeaderBytes));
    if (remote_->topo.stages > 1) {
      void* p = nullptr;
      RS_CUDA_CHECK(cudaMalloc(&p, static_cast<std::size_t>(ctx.max_requests()) * s.vocab * 4));
      remote_logits_ = static_cast<float*>(p);
    }
  }
}

DeviceBackend::~DeviceBackend() {
  cudaDeviceSynchronize();
  ctx_.quiesce();  // page guards reference this backend's events
  for (auto& [id, p] : payloads_) {
    if (p.patches_dev) cudaFree(p.patches_dev);
    if (p.patches_host) cudaFreeHost(p.patches_host);
  }
  for (auto& [id, p] : logits_host_) cudaFreeHost(p);
  for (bf16* p : staging_) cudaFree(p);
  for (bf16* p : enc_input_) cudaFree(p);
  for (bf16* p : xbufs_) cudaFree(p);
  for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
  if (origin_) cudaEventDestroy(origin_);
  auto release = [](cudaStream_t st) {  // per-stream kernel workspaces
    gemm_release_stream(st);
    attention_release_stream(st);
  };
  if (!shared_streams_)
    for (auto st : enc_streams_) {
      release(st);
      cudaStreamDestroy(st);
    }
  for (auto st : stage_streams_) {
    release(st);
    cudaStreamDestroy(st);
  }
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  remote_ops_.clear();
  chunk_logits_.clear();
  slot_xfer_.clear();
  for (void* p : ctrl_dev_) cudaFree(p);
  for (std::int64_t* p : ctrl_host_) cudaFreeHost(p);
  if (ctrl_stream_) cudaStreamDestroy(ctrl_stream_);
  if (header_sink_) cudaFree(header_sink_);
  if (remote_logits_) cudaFree(remote_logits_);
}

cudaEvent_t DeviceBackend::timing_event() {
  cudaEvent_t e;
  RS_CUDA_CHECK(cudaEventCreate(&e));
  event_pool_.push_back(e);
  return e;
}

void DeviceBackend::prepare(const std::vector<lmmsim::RequestSpec>& workload) {
  const Shapes& s = ctx_.shapes();
  cudaStream_t st = ctx_.aux_stream();
  for (const lmmsim::RequestSpec& req : workload) {
    const auto pit = payload_.find(req.id);
    const ResolvedPayload& rp = resolved_[req.id] =
        resolve_payload(req, pit != payload_.end() ? &pit->second : nullptr, seed_, s.vocab);
    std::uint64_t patches = 0;
    for (const lmmsim::SegmentSpec& seg : req.segments)
      if (seg.kind == lmmsim::SegmentKind::Multimodal) patches += 4 * seg.tokens;
    Payload p;
    p.patches = patches;
    if (patches > 0 && remote_ == nullptr) {  // EP: pixels live on the encoder ranks
      void* dev = nullptr;
      RS_CUDA_CHECK(cudaMalloc(&dev, patches * s.pdim * sizeof(bf16)));
      p.patches_dev = static_cast<bf16*>(dev);
      std::uint64_t off = 0, item = 0;
      for (const lmmsim::SegmentSpec& seg : req.segments) {
        if (seg.kind != lmmsim::SegmentKind::Multimodal) continue;
        fill_uniform(p.patches_dev + off * s.pdim, static_cast<std::int64_t>(4 * seg.tokens),
                     s.pdim, s.pdim, rp.item_seeds[item], pixel_stream(req.id, item), kPixelScale, 0.f, st);
        off += 4 * seg.tokens;
        ++item;
      }
      if (e2e_) {
        void* host = nullptr;
        RS_CUDA_CHECK(cudaMallocHost(&host, patches * s.pdim * sizeof(bf16)));
        p.patches_host = static_cast<bf16*>(host);
        RS_CUDA_CHECK(cudaMemcpyAsync(host, p.patches_dev, patches * s.pdim * sizeof(bf16),
                                      cudaMemcpyDeviceToHost, st));
      }
    }
    if (e2e_) {
      void* lh = nullptr;
      RS_CUDA_CHECK(cudaMallocHost(&lh, static_cast<std::size_t>(s.vocab) * 4));
      logits_host_[req.id] = static_cast<float*>(lh);
    }
    payloads_[req.id] = p;
  }
  RS_CUDA_CHECK(cudaStreamSynchronize(st));
  if (e2e_) {  // e2e runs read the pixels from pinned host memory only
    for (auto& [id, p] : payloads_) {
      if (p.patches_dev) cudaFree(p.patches_dev);
      p.patches_dev = nullptr;
    }
  }
}

void DeviceBackend::start() {
  RS_CUDA_CHECK(cudaDeviceSynchronize());
  last_poll_ms_ = -1;
  stats_.host_max_gap_ms = 0;
  stats_.host_last_seen_ms = 0;
  stats_.host_max_call_ms = 0;
  stats_.host_max_call_kind = -1;
  take_max_launch_ms();
  launches0_ = launches_so_far();
  upload0_ = ctx_.uploader().bytes_uploaded();
  RS_CUDA_CHECK(cudaEventRecord(origin_, ctx_.tracker_stream()));
  RS_CUDA_CHECK(cudaEventSynchronize(origin_));
  t0_ = std::chrono::steady_clock::now();
}

lmmsim::TimeMs DeviceBackend::clock_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count();
}

void DeviceBackend::track(lmmsim::OpKind k, std::uint32_t a, std::uint64_t b, cudaEvent_t begin,
                          cudaEvent_t end) {
  ops_.push_back({k, a, b, begin, end});
  last_event_ = end;
}

void DeviceBackend::on_request_created(const lmmsim::RequestSpec& req, const lmmsim::EmbeddingTracker&) {
  cudaStream_t st = ctx_.tracker_stream();
  const auto rit = resolved_.find(req.id);
  DevRequest& r = rit != resolved_.end()
                      ? ctx_.create_request(req, rit->second.text_ids.data(), seed_, st, &rit->second.item_grids)
                      : ctx_.create_request(req, nullptr, seed_, st);
  done_slots_[req.id] = r.slot;
  if (remote_ != nullptr) layouts_[req.id] = req.segments;
  if (e2e_) {
    std::uint64_t text = 0;
    for (const auto& [b, e] : r.text_ranges) text += e - b;
    stats_.h2d_bytes += text * 4;  // token ids
  }
  if (!tracker_tail_) tracker_tail_ = ctx_.new_event();
  RS_CUDA_CHECK(cudaEventRecord(tracker_tail_, st));
}

// Host-side stall diagnostics: the longest backend call of a run.
struct CallTimer {
  DeviceBackend* be;
  int kind;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~CallTimer() { be->note_call(kind, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()); }
};

/// A staging buffer for one encode batch's embeddings, held from
/// launch_encode until that batch's on_embeddings_ready has enqueued its
/// scatter (the scatter's event then guards the next writer). Batches whose
/// transfers are still outstanding keep theirs, so with more of them in
/// flight than the initial ring holds (slow links, EP receives posted ahead)
/// the pool grows instead of handing out a buffer that is still unread.
int DeviceBackend::acquire_staging() {
  const std::size_t n = staging_.size();
  for (std::size_t k = 0; k < n; ++k) {
    const std::size_t i = (staging_next_ + k) % n;
    if (staging_busy_[i]) continue;
    staging_busy_[i] = true;
    staging_next_ = (i + 1) % n;
    return static_cast<int>(i);
  }
  void* p = nullptr;
  RS_CUDA_CHECK(cudaMalloc(&p, ctx_.options().max_encode_tokens * ctx_.shapes().d * sizeof(bf16)));
  staging_.push_back(static_cast<bf16*>(p));
  staging_free_.push_back(nullptr);
  staging_busy_.push_back(true);
  return static_cast<int>(staging_.size() - 1);
}

void DeviceBackend::note_call(int kind, double ms) {
  if (ms > stats_.host_max_call_ms) {
    stats_.host_max_call_ms = ms;
    stats_.host_max_call_kind = kind;
  }
}

double DeviceBackend::launch_encode(int worker, std::size_t slot, const lmmsim::EncodeBatch& b) {
  NvtxRange nvtx_("encode_r%llu_b%llu", b.request_id, slot);
  CallTimer timer{this, 0};
  HostPhase phase_("launch_encode");
  if (remote_ != nullptr) {
    launch_remote_encode(worker, slot, b);
    return realtime_ ? 0.0 : lmmsim::encode_time_ms(cfg_.cost, b);
  }
  cudaStream_t st = enc_streams_[static_cast<std::size_t>(worker)];
  DevRequest& r = ctx_.get(b.request_id);
  const Shapes& s = ctx_.shapes();
  const int ring = acquire_staging();
  if (staging_free_[static_cast<std::size_t>(ring)] != nullptr)
    RS_CUDA_CHECK(cudaStreamWaitEvent(st, staging_free_[static_cast<std::size_t>(ring)], 0));
  slot_staging_[slot] = ring;

  std::vector<lmmsim::TokenRange> items;
  for (const auto& it : b.items) items.push_back(it.second);
  const std::size_t first_item = b.items.front().first;
  const std::uint64_t p0 = r.item_patch_offset[first_item];
  const std::uint64_t np = 4 * b.total_tokens;
  cudaEvent_t begin = timing_event(), end = timing_event();
  RS_CUDA_CHECK(cudaEventRecord(begin, st));
  const Payload& pay = payloads_.at(b.request_id);
  const bf16* patches = nullptr;
  if (e2e_) {
    RS_CUDA_CHECK(cudaMemcpyAsync(enc_input_[static_cast<std::size_t>(worker)],
                                  pay.patches_host + p0 * s.pdim, np * s.pdim * sizeof(bf16),
                                  cudaMemcpyHostToDevice, st));
    stats_.h2d_bytes += np * s.pdim * sizeof(bf16);
    patches = enc_input_[static_cast<std::size_t>(worker)];
  } else {
    patches = pay.patches_dev + p0 * s.pdim;
  }
  const VitBatchPlan plan = ctx_.plan_batch(r, items);
  {
    HostPhase ph("launch_encode.ctx_encode");
    ctx_.encode(plan, patches, staging_[static_cast<std::size_t>(ring)], st);
  }
  RS_CUDA_CHECK(cudaEventRecord(end, st));
  slot_done_[slot] = end;
  last_encode_end_ = end;
  track(lmmsim::OpKind::Encode, static_cast<std::uint32_t>(worker), slot, begin, end);
  return realtime_ ? 0.0 : lmmsim::encode_time_ms(cfg_.cost, b);
}

double DeviceBackend::launch_transfer(int /*worker*/, std::size_t slot, const lmmsim::EncodeBatch& b) {
  NvtxRange nvtx_("transfer_r%llu_b%llu", b.request_id, slot);
  if (remote_ != nullptr) {  // EP: the embeddings' receive was posted at launch_encode
    for (RemoteOp& op : remote_ops_)
      if (op.kind == lmmsim::OpKind::Transfer && op.b == slot) op.launched = true;
    return realtime_ ? 0.0 : lmmsim::transfer_time_ms(cfg_.cost, b.total_tokens);
  }
  // Co-located encoder and prefill: the embeddings are already in this GPU's
  // HBM; the link is the reference's zero-cost case.
  if (realtime_) ready_transfers_.emplace_back(slot, slot_done_ms_.count(slot) ? slot_done_ms_[slot] : clock_ms());
  return realtime_ ? 0.0 : lmmsim::transfer_time_ms(cfg_.cost, b.total_tokens);
}

void DeviceBackend::on_embeddings_ready(std::size_t slot, const lmmsim::EncodeBatch& b) {
  CallTimer timer{this, 2};
  HostPhase phase_("on_embeddings_ready");
  cudaStream_t st = ctx_.tracker_stream();
  if (remote_ != nullptr) remote_->t->wait_posted(*slot_xfer_.at(slot));
  RS_CUDA_CHECK(cudaStreamWaitEvent(st, slot_done_.at(slot), 0));
  DevRequest& r = ctx_.get(b.request_id);
  std::vector<lmmsim::TokenRange> items;
  for (const auto& it : b.items) items.push_back(it.second);
  const int ring = slot_staging_.at(slot);
  ctx_.scatter_items(r, items, staging_[static_cast<std::size_t>(ring)], st);
  slot_xfer_.erase(slot);
  cudaEvent_t ev = ctx_.new_event();
  RS_CUDA_CHECK(cudaEventRecord(ev, st));
  staging_free_[static_cast<std::size_t>(ring)] = ev;
  staging_busy_[static_cast<std::size_t>(ring)] = false;  // reusable once `ev` completes
  if (!tracker_tail_) tracker_tail_ = ctx_.new_event();
  RS_CUDA_CHECK(cudaEventRecord(tracker_tail_, st));
}

double DeviceBackend::launch_stage(int stage, const lmmsim::ChunkView& c) {
  NvtxRange nvtx_("chunk%llu_s%llu", c.chunk_id, static_cast<unsigned long long>(stage));
  CallTimer timer{this, 1};
  HostPhase phase_("launch_stage");
  const double cost = realtime_ ? 0.0 : lmmsim::stage_time_ms(cfg_.cost, c.total_tokens, c.weighted_context);
  if (remote_ != nullptr && stage > 0) {  // runs on rank P_stage; completion = its DONE message
    for (RemoteOp& op : remote_ops_)
      if (op.kind == lmmsim::OpKind::Stage && op.a == static_cast<std::uint32_t>(stage) && op.b == c.chunk_id)
        op.launched = true;
    return cost;
  }
  cudaStream_t st = stage_streams_[0];
  ChunkState& cs = chunks_[c.chunk_id];
  static const bool enc_first = [] {
    const char* e = std::getenv("RS_ENCODE_FIRST");
    return e != nullptr && e[0] == '1';
  }();
  if (enc_first && last_encode_end_ != nullptr && !shared_streams_)
    RS_CUDA_CHECK(cudaStreamWaitEvent(st, last_encode_end_, 0));
  if (stage == 0) {
    if (free_xbufs_.empty()) throw DeviceError(RS_ERR_CUDA, "no free chunk buffer");
    cs.buf = free_xbufs_.back();
    free_xbufs_.pop_back();
    cs.x = xbufs_[static_cast<std::size_t>(cs.buf)];
    if (xbuf_guard_[static_cast<std::size_t>(cs.buf)] != nullptr)
      RS_CUDA_CHECK(cudaStreamWaitEvent(st, xbuf_guard_[static_cast<std::size_t>(cs.buf)], 0));
    if (tracker_tail_ != nullptr) {
      // Snapshot: every scatter / creation issued so far precedes this chunk.
      cudaEvent_t snap = ctx_.new_event();
      RS_CUDA_CHECK(cudaEventRecord(snap, ctx_.tracker_stream()));
      RS_CUDA_CHECK(cudaStreamWaitEvent(st, snap, 0));
    }
  }
  std::vector<SliceRef> slices;
  for (const auto& [id, range] : *c.slices) slices.push_back({&ctx_.get(id), range.start, range.end});
  // Layers of this stage within the context's range.
  const int lb = ctx_.llm()->layer_begin(), le = ctx_.llm()->layer_end();
  const int S = remote_ != nullptr ? 1 : cfg_.stages, n = le - lb;  // EP: stage 0 = all local layers
  const int from = lb + n * stage / S, to = lb + n * (stage + 1) / S;
  cudaEvent_t begin = timing_event(), end = timing_event();
  RS_CUDA_CHECK(cudaEventRecord(begin, st));
  {
    HostPhase ph("launch_stage.ctx_prefill");
    ctx_.prefill(slices, cs.x, st, from, to);
  }
  RS_CUDA_CHECK(cudaEventRecord(end, st));
  cs.last = end;
  if (stage == 0) cs.s0_end = end;
  track(lmmsim::OpKind::Stage, static_cast<std::uint32_t>(stage), c.chunk_id, begin, end);
  if (remote_ != nullptr && cfg_.stages > 1) {
    forward_chunk(c, cs);  // sets the residual buffer's guard to its send
    free_xbufs_.push_back(cs.buf);
  } else if (stage + 1 == S) {  // residual buffer free once the last stage ran
    xbuf_guard_[static_cast<std::size_t>(cs.buf)] = end;
    free_xbufs_.push_back(cs.buf);
  }
  return cost;
}

void* DeviceBackend::put_ctrl(const ep::Words& w) {
  const int i = ctrl_pos_;
  ctrl_pos_ = (ctrl_pos_ + 1) % kCtrlRing;
  if (ctrl_free_[static_cast<std::size_t>(i)] != nullptr)  // previous message still in flight
    RS_CUDA_CHECK(cudaEventSynchronize(ctrl_free_[static_cast<std::size_t>(i)]));
  std::memcpy(ctrl_host_[static_cast<std::size_t>(i)], w.data(), ep::kCtrlBytes);
  RS_CUDA_CHECK(cudaMemcpyAsync(ctrl_dev_[static_cast<std::size_t>(i)], ctrl_host_[static_cast<std::size_t>(i)],
                                ep::kCtrlBytes, cudaMemcpyHostToDevice, ctrl_stream_));
  stats_.h2d_bytes += ep::kCtrlBytes;
  return ctrl_dev_[static_cast<std::size_t>(i)];
}

void DeviceBackend::launch_remote_encode(int worker, std::size_t slot, const lmmsim::EncodeBatch& b) {
  const ep::Topology& topo = remote_->topo;
  ep::Transport& t = *remote_->t;
  DevRequest& r = ctx_.get(b.request_id);
  const Shapes& s = ctx_.shapes();
  const int ring = acquire_staging();
  slot_staging_[slot] = ring;
  ep::EncodeCmd cmd;
  cmd.slot = slot;
  cmd.request_id = b.request_id;
  for (const auto& [idx, range] : b.items)
    cmd.items.push_back({idx, range.start, range.end, r.item_patch_offset[idx]});
  ep::Words w;
  ep::pack(cmd, w);
  void* dev = put_ctrl(w);
  cudaEvent_t staged = timing_event();
  RS_CUDA_CHECK(cudaEventRecord(staged, ctrl_stream_));
  const int peer = topo.e_rank(worker);
  ctrl_free_[static_cast<std::size_t>((ctrl_pos_ + kCtrlRing - 1) % kCtrlRing)] =
      t.send(peer, dev, ep::kCtrlBytes, staged);
  auto hdr = t.post_recv(peer, header_sink_, ep::kHeaderBytes, nullptr);
  auto emb = t.post_recv(peer, staging_[static_cast<std::size_t>(ring)], b.total_tokens * s.d * sizeof(bf16),
                         staging_free_[static_cast<std::size_t>(ring)]);
  slot_done_[slot] = emb->done;
  slot_xfer_[slot] = emb;
  remote_ops_.push_back({lmmsim::OpKind::Encode, static_cast<std::uint32_t>(worker), slot, {hdr}, true});
  remote_ops_.push_back({lmmsim::OpKind::Transfer, 0, slot, {emb}, false});
}

void DeviceBackend::forward_chunk(const lmmsim::ChunkView& c, const ChunkState& cs) {
  const ep::Topology& topo = remote_->topo;
  ep::Transport& t = *remote_->t;
  const Shapes& s = ctx_.shapes();
  ep::StageCmd cmd;
  cmd.chunk_id = c.chunk_id;
  for (const auto& [id, range] : *c.slices) cmd.slices.push_back({id, range.start, range.end, layouts_.at(id)});
  ep::Words w;
  ep::pack(cmd, w);
  void* dev = put_ctrl(w);
  cudaEvent_t staged = timing_event();
  RS_CUDA_CHECK(cudaEventRecord(staged, ctrl_stream_));
  const int p1 = topo.p_rank(1);
  ctrl_free_[static_cast<std::size_t>((ctrl_pos_ + kCtrlRing - 1) % kCtrlRing)] =
      t.send(p1, dev, ep::kCtrlBytes, staged);
  // The residual rides behind the control message; its buffer is reusable
  // once sent.
  xbuf_guard_[static_cast<std::size_t>(cs.buf)] =
      t.send(p1, cs.x, c.total_tokens * s.d * sizeof(bf16), cs.s0_end);
  // Completions of the downstream stages: a DONE header each; the last stage
  // then ships the logits row of every prompt that ends in this chunk.
  for (int st = 1; st < topo.stages; ++st) {
    RemoteOp op{lmmsim::OpKind::Stage, static_cast<std::uint32_t>(st), c.chunk_id, {}, false};
    op.xfers.push_back(t.post_recv(topo.p_rank(st), header_sink_, ep::kHeaderBytes, nullptr));
    if (st + 1 == topo.stages) {
      for (const auto& [id, range] : *c.slices) {
        const DevRequest& r = ctx_.get(id);
        if (range.end != r.total) continue;
        op.xfers.push_back(t.post_recv(topo.p_rank(st), remote_logits_ + static_cast<std::int64_t>(r.slot) * s.vocab,
                                       static_cast<std::size_t>(s.vocab) * 4, nullptr));
      }
      chunk_logits_[c.chunk_id] = op.xfers.back();
    }
    remote_ops_.push_back(std::move(op));
  }
}

bool DeviceBackend::remote_done(RemoteOp& op) {
  for (auto& x : op.xfers)
    if (!remote_->t->test(*x)) return false;
  return true;
}

void DeviceBackend::on_release(std::size_t chunk, lmmsim::RequestId id, lmmsim::TokenRange r) {
  const ChunkState& cs = chunks_.at(chunk);
  release_guard_ = remote_ != nullptr ? cs.s0_end : cs.last;
  DevRequest& dr = ctx_.get(id);
  ctx_.release_prefix(dr, r.end, release_guard_);
}

void DeviceBackend::on_request_erased(lmmsim::RequestId id) {
  if (keep_kv_) {  // prompt slab pages are back (release_prefix); KV stays for decode
    kept_.push_back(id);
    return;
  }
  ctx_.erase_request(id, release_guard_, /*keep_slot=*/true);
}

void DeviceBackend::on_request_complete(lmmsim::RequestId id, std::size_t chunk) {
  if (!e2e_) return;
  const ChunkState& cs = chunks_.at(chunk);
  if (remote_logits_ != nullptr) {  // EP: the logits row arrived from the last stage
    for (RemoteOp& op : remote_ops_)
      if (op.kind == lmmsim::OpKind::Stage && op.b == chunk)
        for (auto& x : op.xfers) remote_->t->wait_posted(*x);
    RS_CUDA_CHECK(cudaStreamWaitEvent(copy_stream_, chunk_logits_.at(chunk)->done, 0));
    RS_CUDA_CHECK(cudaMemcpyAsync(logits_host_.at(id),
                                  remote_logits_ + static_cast<std::int64_t>(done_slots_.at(id)) * ctx_.shapes().vocab,
                                  static_cast<std::size_t>(ctx_.shapes().vocab) * 4, cudaMemcpyDeviceToHost,
                                  copy_stream_));
  } else {
    RS_CUDA_CHECK(cudaStreamWaitEvent(copy_stream_, cs.last, 0));
    ctx_.copy_logits(done_slots_.at(id), logits_host_.at(id), copy_stream_);
  }
  stats_.d2h_bytes += static_cast<std::uint64_t>(ctx_.shapes().vocab) * 4;
}

void DeviceBackend::poll(std::vector<lmmsim::OpCompletion>& out) {
  const double now = clock_ms();
  if (last_poll_ms_ >= 0) stats_.host_max_gap_ms = std::max(stats_.host_max_gap_ms, now - last_poll_ms_);
  last_poll_ms_ = now;
  const std::size_t n0 = out.size();
  struct SeenStamp {  // host time of the poll that saw a completion
    std::vector<lmmsim::OpCompletion>& v;
    std::size_t n0;
    double now;
    double& seen;
    ~SeenStamp() {
      if (v.size() > n0) seen = now;
    }
  } stamp{out, n0, now, stats_.host_last_seen_ms};
  for (const auto& [slot, t] : ready_transfers_) out.push_back({lmmsim::OpKind::Transfer, 0, slot, t});
  ready_transfers_.clear();
  for (std::size_t i = 0; i < ops_.size();) {
    const cudaError_t q = cudaEventQuery(ops_[i].end);
    if (q == cudaErrorNotReady) {
      ++i;
      continue;
    }
    RS_CUDA_CHECK(q);
    float ms = 0;
    RS_CUDA_CHECK(cudaEventElapsedTime(&ms, origin_, ops_[i].end));
    if (ops_[i].kind == lmmsim::OpKind::Encode) slot_done_ms_[ops_[i].b] = ms;
    out.push_back({ops_[i].kind, ops_[i].a, ops_[i].b, static_cast<double>(ms)});
    ops_[i] = ops_.back();
    ops_.pop_back();
  }
  for (std::size_t i = 0; i < remote_ops_.size();) {
    RemoteOp& op = remote_ops_[i];
    if (!op.launched || !remote_done(op)) {
      ++i;
      continue;
    }
    float ms = 0;
    RS_CUDA_CHECK(cudaEventElapsedTime(&ms, origin_, op.xfers.back()->done));
    remote_last_ms_ = std::max(remote_last_ms_, static_cast<double>(ms));
    out.push_back({op.kind, op.a, op.b, static_cast<double>(ms)});
    remote_ops_.erase(remote_ops_.begin() + static_cast<std::ptrdiff_t>(i));
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const lmmsim::OpCompletion& x, const lmmsim::OpCompletion& y) {
                     return x.time_ms < y.time_ms;
                   });
}

void DeviceBackend::finish() {
  for (RemoteOp& op : remote_ops_) {  // lock-step EP: arrivals not yet observed
    for (auto& x : op.xfers) remote_->t->wait(*x);
    float ms = 0;
    RS_CUDA_CHECK(cudaEventElapsedTime(&ms, origin_, op.xfers.back()->done));
    remote_last_ms_ = std::max(remote_last_ms_, static_cast<double>(ms));
  }
  remote_ops_.clear();
  const double sync0 = clock_ms();
  RS_CUDA_CHECK(cudaDeviceSynchronize());
  stats_.wall_ms = clock_ms();
  stats_.host_finish_sync_ms = stats_.wall_ms - sync0;
  if (last_event_ != nullptr) {
    float ms = 0;
    RS_CUDA_CHECK(cudaEventElapsedTime(&ms, origin_, last_event_));
    stats_.gpu_ms = ms;
  }
  stats_.gpu_ms = std::max(stats_.gpu_ms, remote_last_ms_);
  stats_.kernel_launches = launches_so_far() - launches0_;
  stats_.host_max_launch_ms = take_max_launch_ms();
  stats_.h2d_bytes += ctx_.uploader().bytes_uploaded() - upload0_;
}

void DeviceBackend::collect() {
  const int vocab = ctx_.shapes().vocab;
  std::vector<std::int32_t> am(static_cast<std::size_t>(ctx_.max_requests()));
  if (ctx_.device_argmax() != nullptr)
    RS_CUDA_CHECK(cudaMemcpy(am.data(), ctx_.device_argmax(), am.size() * 4, cudaMemcpyDeviceToHost));
  for (const auto& [id, slot] : done_slots_) {
    std::vector<float> row(static_cast<std::size_t>(vocab));
    if (e2e_) {
      std::memcpy(row.data(), logits_host_.at(id), row.size() * 4);
    } else if (remote_logits_ != nullptr) {
      RS_CUDA_CHECK(cudaMemcpy(row.data(), remote_logits_ + static_cast<std::int64_t>(slot) * vocab,
                               row.size() * 4, cudaMemcpyDeviceToHost));
    } else {
      ctx_.copy_logits(slot, row.data(), ctx_.aux_stream());
      RS_CUDA_CHECK(cudaStreamSynchronize(ctx_.aux_stream()));
    }
    argmax_[id] = remote_logits_ != nullptr
                      ? static_cast<std::int32_t>(std::max_element(row.begin(), row.end()) - row.begin())
                      : am[static_cast<std::size_t>(slot)];
    logits_[id] = std::move(row);
    if (!keep_kv_) ctx_.free_slot(slot);
  }
  done_slots_.clear();
}

}  // namespace rserve
