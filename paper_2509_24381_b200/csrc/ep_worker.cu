// rserve-b200 — EP worker loops: encoder ranks and downstream prefill stages.
#include <algorithm>

#include "ep.cuh"
#include "kernels.cuh"

namespace rserve::ep {

namespace {
std::vector<std::int64_t> read_ctrl(Transport& t, int peer, void* dev, std::int64_t* host,
                                    cudaStream_t st, void* fwd_dev = nullptr,
                                    cudaEvent_t fwd_free = nullptr) {
  auto x = t.post_recv(peer, dev, kCtrlBytes, nullptr);
  t.wait(*x);
  RS_CUDA_CHECK(cudaStreamWaitEvent(st, x->done, 0));
  RS_CUDA_CHECK(cudaMemcpyAsync(host, dev, kCtrlBytes, cudaMemcpyDeviceToHost, st));
  if (fwd_dev != nullptr) {  // copy kept for forwarding down the pipeline
    if (fwd_free != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(st, fwd_free, 0));
    RS_CUDA_CHECK(cudaMemcpyAsync(fwd_dev, dev, kCtrlBytes, cudaMemcpyDeviceToDevice, st));
  }
  RS_CUDA_CHECK(cudaStreamSynchronize(st));
  return std::vector<std::int64_t>(host, host + kCtrlWords);
}

/// Ring of completion events owned by a worker (guards are only ever waited
/// on; re-recording one later on the same stream is conservative).
struct Ring {
  std::vector<cudaEvent_t> ev;
  std::size_t next = 0;
  explicit Ring(std::size_t n) : ev(n) {
    for (auto& e : ev) RS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~Ring() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaEvent_t take() {
    cudaEvent_t e = ev[next];
    next = (next + 1) % ev.size();
    return e;
  }
};
constexpr int kBufs = 4;
}  // namespace

// ---- encoder ------------------------------------------------------------------------------
EncoderWorker::EncoderWorker(Context& ctx, Transport& t, const Topology& topo)
    : ctx_(ctx), t_(t), topo_(topo) {
  if (ctx.vit() == nullptr) throw lmmsim::ConfigError("EP encoder rank: context has no vision encoder");
  RS_CUDA_CHECK(cudaSetDevice(ctx.options().device));
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  const std::size_t out_bytes = ctx.options().max_encode_tokens * ctx.shapes().d * sizeof(bf16);
  for (int i = 0; i < kBufs; ++i) {
    void* p = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&p, out_bytes));
    out_.push_back(static_cast<bf16*>(p));
    out_free_.push_back(nullptr);
  }
  RS_CUDA_CHECK(cudaMalloc(&ctrl_dev_, kCtrlBytes));
  RS_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&ctrl_host_), kCtrlBytes));
  RS_CUDA_CHECK(cudaMalloc(&header_dev_, kHeaderBytes));
  RS_CUDA_CHECK(cudaMemset(header_dev_, 0, kHeaderBytes));
}

EncoderWorker::~EncoderWorker() {
  cudaDeviceSynchronize();
  for (auto& [id, p] : pay_) {
    if (p.dev) cudaFree(p.dev);
    if (p.host) cudaFreeHost(p.host);
  }
  for (bf16* p : out_) cudaFree(p);
  if (input_) cudaFree(input_);
  cudaFree(ctrl_dev_);
  cudaFreeHost(ctrl_host_);
  cudaFree(header_dev_);
  cudaStreamDestroy(st_);
}

void EncoderWorker::prepare(const std::vector<lmmsim::RequestSpec>& workload, std::uint64_t seed,
                            bool e2e) {
  RS_CUDA_CHECK(cudaSetDevice(ctx_.options().device));
  const Shapes& s = ctx_.shapes();
  RS_CUDA_CHECK(cudaStreamSynchronize(st_));
  for (auto& [id, p] : pay_) {
    if (p.dev) cudaFree(p.dev);
    if (p.host) cudaFreeHost(p.host);
  }
  pay_.clear();
  e2e_ = e2e;
  if (e2e_ && input_ == nullptr) {
    void* p = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&p, 4 * ctx_.options().max_encode_tokens * s.pdim * sizeof(bf16)));
    input_ = static_cast<bf16*>(p);
  }
  for (const lmmsim::RequestSpec& req : workload) {
    std::uint64_t patches = 0;
    for (const auto& seg : req.segments)
      if (seg.kind == lmmsim::SegmentKind::Multimodal) patches += 4 * seg.tokens;
    if (patches == 0) continue;
    Pay p;
    void* dev = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&dev, patches * s.pdim * sizeof(bf16)));
    p.dev = static_cast<bf16*>(dev);
    std::uint64_t off = 0, item = 0;
    for (const auto& seg : req.segments) {
      if (seg.kind != lmmsim::SegmentKind::Multimodal) continue;
      fill_uniform(p.dev + off * s.pdim, static_cast<std::int64_t>(4 * seg.tokens), s.pdim, s.pdim,
                   seed, pixel_stream(req.id, item), kPixelScale, 0.f, st_);
      off += 4 * seg.tokens;
      ++item;
    }
    if (e2e_) {
      void* host = nullptr;
      RS_CUDA_CHECK(cudaMallocHost(&host, patches * s.pdim * sizeof(bf16)));
      RS_CUDA_CHECK(cudaMemcpyAsync(host, p.dev, patches * s.pdim * sizeof(bf16),
                                    cudaMemcpyDeviceToHost, st_));
      RS_CUDA_CHECK(cudaStreamSynchronize(st_));
      cudaFree(p.dev);
      p.dev = nullptr;
      p.host = static_cast<bf16*>(host);
    }
    pay_[req.id] = p;
  }
  RS_CUDA_CHECK(cudaStreamSynchronize(st_));
}

void EncoderWorker::run() {
  RS_CUDA_CHECK(cudaSetDevice(ctx_.options().device));
  const Shapes& s = ctx_.shapes();
  const int p0 = topo_.p_rank(0);
  cudaStream_t ctrl_st;
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&ctrl_st, cudaStreamNonBlocking));
  Ring done(8);
  DevRequest none;
  for (;;) {
    const Words w = read_ctrl(t_, p0, ctrl_dev_, ctrl_host_, ctrl_st);
    if (kind_of(w) == Ctrl::kStop) break;
    const EncodeCmd c = unpack_encode(w);
    const auto it = pay_.find(c.request_id);
    if (it == pay_.end())
      throw lmmsim::RegistryError("EP encoder: no payload for request " + lmmsim::format_u64(c.request_id));
    const int b = static_cast<int>(batches_ % kBufs);
    if (out_free_[static_cast<std::size_t>(b)] != nullptr)
      RS_CUDA_CHECK(cudaStreamWaitEvent(st_, out_free_[static_cast<std::size_t>(b)], 0));
    std::vector<lmmsim::TokenRange> items;
    for (const EncodeItem& i : c.items) items.push_back({i.start, i.end});
    const std::uint64_t first = c.items.front().patch_offset;
    const std::uint64_t np = 4 * c.tokens();
    const bf16* patches = nullptr;
    if (e2e_) {
      RS_CUDA_CHECK(cudaMemcpyAsync(input_, it->second.host + first * s.pdim, np * s.pdim * sizeof(bf16),
                                    cudaMemcpyHostToDevice, st_));
      patches = input_;
    } else {
      patches = it->second.dev + first * s.pdim;
    }
    const VitBatchPlan plan = ctx_.plan_batch(none, items);
    ctx_.encode(plan, patches, out_[static_cast<std::size_t>(b)], st_);
    cudaEvent_t end = done.take();
    RS_CUDA_CHECK(cudaEventRecord(end, st_));
    t_.send(p0, header_dev_, kHeaderBytes, end);
    out_free_[static_cast<std::size_t>(b)] =
        t_.send(p0, out_[static_cast<std::size_t>(b)], c.tokens() * s.d * sizeof(bf16), end);
    ++batches_;
  }
  RS_CUDA_CHECK(cudaDeviceSynchronize());
  cudaStreamDestroy(ctrl_st);
}

// ---- downstream stage ------------------------------------------------------------------------
StageWorker::StageWorker(Context& ctx, Transport& t, const Topology& topo, int stage)
    : ctx_(ctx), t_(t), topo_(topo), stage_(stage), last_(stage + 1 == topo.stages) {
  if (stage < 1 || stage >= topo.stages) throw lmmsim::ConfigError("EP stage worker: bad stage index");
  if (last_ && !ctx.llm()->has_head())
    throw lmmsim::ConfigError("EP last stage: context needs the LM head (with_lm_head=1)");
  RS_CUDA_CHECK(cudaSetDevice(ctx.options().device));
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  const std::size_t x_bytes = ctx.options().max_chunk_tokens * ctx.shapes().d * sizeof(bf16);
  for (int i = 0; i < kBufs; ++i) {
    void* p = nullptr;
    RS_CUDA_CHECK(cudaMalloc(&p, x_bytes));
    x_.push_back(static_cast<bf16*>(p));
    x_free_.push_back(nullptr);
  }
  RS_CUDA_CHECK(cudaMalloc(&ctrl_dev_, kCtrlBytes));
  RS_CUDA_CHECK(cudaMalloc(&ctrl_fwd_dev_, kCtrlBytes));
  RS_CUDA_CHECK(cudaMallocHost(reinterpret_cast<void**>(&ctrl_host_), kCtrlBytes));
  RS_CUDA_CHECK(cudaMalloc(&header_dev_, kHeaderBytes));
  RS_CUDA_CHECK(cudaMemset(header_dev_, 0, kHeaderBytes));
}

StageWorker::~StageWorker() {
  cudaDeviceSynchronize();
  for (bf16* p : x_) cudaFree(p);
  cudaFree(ctrl_dev_);
  cudaFree(ctrl_fwd_dev_);
  cudaFreeHost(ctrl_host_);
  cudaFree(header_dev_);
  cudaStreamDestroy(st_);
}

void StageWorker::reclaim(bool all) {
  for (std::size_t i = 0; i < slot_reclaim_.size();) {
    const auto [slot, ev] = slot_reclaim_[i];
    if (all) {
      RS_CUDA_CHECK(cudaEventSynchronize(ev));
    } else {
      const cudaError_t q = cudaEventQuery(ev);
      if (q == cudaErrorNotReady) {
        ++i;
        continue;
      }
      RS_CUDA_CHECK(q);
    }
    ctx_.free_slot(slot);
    slot_reclaim_[i] = slot_reclaim_.back();
    slot_reclaim_.pop_back();
  }
}

void StageWorker::run() {
  RS_CUDA_CHECK(cudaSetDevice(ctx_.options().device));
  const Shapes& s = ctx_.shapes();
  const int prev = topo_.p_rank(stage_ - 1), next = last_ ? -1 : topo_.p_rank(stage_ + 1);
  const int p0 = topo_.p_rank(0);
  cudaStream_t ctrl_st;
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&ctrl_st, cudaStreamNonBlocking));
  Ring done(8);
  for (;;) {
    const Words w = read_ctrl(t_, prev, ctrl_dev_, ctrl_host_, ctrl_st, last_ ? nullptr : ctrl_fwd_dev_,
                              ctrl_fwd_free_);
    if (kind_of(w) == Ctrl::kStop) {
      if (!last_) t_.send(next, ctrl_fwd_dev_, kCtrlBytes, nullptr);
      break;
    }
    const StageCmd c = unpack_stage(w);
    std::vector<SliceRef> slices;
    for (const SliceCmd& sl : c.slices) {
      DevRequest* r = ctx_.find(sl.request_id);
      if (r == nullptr) {
        lmmsim::RequestSpec spec;
        spec.id = sl.request_id;
        spec.segments = sl.segments;
        r = &ctx_.create_kv_request(spec, st_);
      }
      slices.push_back({r, sl.start, sl.end});
    }
    const std::uint64_t rows = c.rows();
    if (rows > ctx_.options().max_chunk_tokens)
      throw lmmsim::ConfigError("EP stage: chunk of " + lmmsim::format_u64(rows) + " rows exceeds max_chunk_tokens");
    const std::size_t b = static_cast<std::size_t>(chunks_ % kBufs);
    auto xr = t_.post_recv(prev, x_[b], rows * s.d * sizeof(bf16), x_free_[b]);
    RS_CUDA_CHECK(cudaStreamWaitEvent(st_, xr->done, 0));
    ctx_.prefill(slices, x_[b], st_);
    cudaEvent_t end = done.take();
    RS_CUDA_CHECK(cudaEventRecord(end, st_));
    if (!last_) {
      ctrl_fwd_free_ = t_.send(next, ctrl_fwd_dev_, kCtrlBytes, end);
      x_free_[b] = t_.send(next, x_[b], rows * s.d * sizeof(bf16), end);
    } else {
      x_free_[b] = end;
    }
    t_.send(p0, header_dev_, kHeaderBytes, end);
    for (const SliceRef& sl : slices) {
      if (sl.end != sl.req->total) continue;
      const int slot = sl.req->slot;
      if (last_) {
        cudaEvent_t sent = t_.send(p0, ctx_.llm()->logits_row(slot), static_cast<std::size_t>(s.vocab) * 4, end);
        slot_reclaim_.emplace_back(slot, sent);
      }
      ctx_.erase_request(sl.req->id, end, /*keep_slot=*/last_);
    }
    reclaim(false);
    ++chunks_;
  }
  RS_CUDA_CHECK(cudaDeviceSynchronize());
  reclaim(true);
  ctx_.quiesce();
  cudaStreamDestroy(ctrl_st);
}

void stop_workers(Transport& t, const Topology& topo) {
  void* dev = nullptr;
  RS_CUDA_CHECK(cudaMalloc(&dev, kCtrlBytes));
  Words w;
  pack_stop(w);
  RS_CUDA_CHECK(cudaMemcpy(dev, w.data(), kCtrlBytes, cudaMemcpyHostToDevice));
  std::vector<cudaEvent_t> sent;
  for (int e = 0; e < topo.encoders; ++e) sent.push_back(t.send(topo.e_rank(e), dev, kCtrlBytes, nullptr));
  if (topo.stages > 1) sent.push_back(t.send(topo.p_rank(1), dev, kCtrlBytes, nullptr));
  for (cudaEvent_t e : sent) RS_CUDA_CHECK(cudaEventSynchronize(e));
  cudaFree(dev);
}

}  // namespace rserve::ep
