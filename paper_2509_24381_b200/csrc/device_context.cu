// rserve-b200 — per-GPU pipeline context (see device_context.cuh).
#include <algorithm>
#include <cstring>
#include <set>
#include <tuple>

#include "device_context.cuh"
#include "kernels.cuh"

namespace rserve {

// ---- PagePool --------------------------------------------------------------------
void PagePool::reset(std::int64_t pages) {
  free_.clear();
  for (std::int64_t p = 0; p < pages; ++p) free_.emplace_back(static_cast<int>(p), nullptr);
  cap_ = pages;
}

std::vector<int> PagePool::take(std::int64_t n, std::vector<cudaEvent_t>& guards) {
  if (n > static_cast<std::int64_t>(free_.size()))
    throw DeviceError(RS_ERR_CUDA, "page pool exhausted: need " + std::to_string(n) +
                                       " pages, " + std::to_string(free_.size()) + " free of " +
                                       std::to_string(cap_));
  std::vector<int> out;
  out.reserve(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    auto [page, ev] = free_.front();
    free_.pop_front();
    out.push_back(page);
    if (ev != nullptr && (guards.empty() || guards.back() != ev)) guards.push_back(ev);
  }
  return out;
}

void PagePool::give(const std::vector<int>& pages, cudaEvent_t guard) {
  for (int p : pages)
    if (p >= 0) free_.emplace_back(p, guard);
}

// ---- Uploader ---------------------------------------------------------------------
void Uploader::init(std::size_t bytes) {
  cap_ = bytes;
  RS_CUDA_CHECK(cudaMallocHost(&host_, bytes));
  RS_CUDA_CHECK(cudaMalloc(&dev_, bytes));
}

Uploader::~Uploader() {
  marks_.clear();
  if (host_) cudaFreeHost(host_);
  if (dev_) cudaFree(dev_);
}

void* Uploader::put(const void* src, std::size_t n, cudaStream_t st) {
  const std::size_t len = n;
  n = (n + 255) / 256 * 256;
  if (n > cap_ / 4) throw DeviceError(RS_ERR_CUDA, "uploader: descriptor too large");
  if (head_ + n > cap_) head_ = 0;  // wrap
  const std::size_t b = head_, e = head_ + n;
  // Regions still in use by enqueued work must be consumed before reuse.
  for (auto it = marks_.begin(); it != marks_.end();) {
    if (it->begin < e && b < it->end) {
      RS_CUDA_CHECK(cudaEventSynchronize(it->ev.get()));
      it = marks_.erase(it);
    } else {
      ++it;
    }
  }
  if (len > 0) std::memcpy(host_ + b, src, len);
  RS_CUDA_CHECK(cudaMemcpyAsync(dev_ + b, host_ + b, n, cudaMemcpyHostToDevice, st));
  head_ = e;
  uploaded_ += n;
  if (pending_begin_ == kNone) pending_begin_ = b;
  pending_.push_back({b, e});
  return dev_ + b;
}

void Uploader::fence(cudaStream_t st) {
  if (pending_.empty()) return;
  cudaEvent_t raw;
  RS_CUDA_CHECK(cudaEventCreateWithFlags(&raw, cudaEventDisableTiming));
  RS_CUDA_CHECK(cudaEventRecord(raw, st));
  std::shared_ptr<CUevent_st> ev(raw, [](cudaEvent_t e) { cudaEventDestroy(e); });
  for (const auto& [b, e] : pending_) marks_.push_back({b, e, ev});
  pending_.clear();
  pending_begin_ = kNone;
}

// ---- Context ----------------------------------------------------------------------
Context::Context(const rs_model_config& model, const rs_ctx_options& opt) : opt_(opt) {
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
    throw DeviceError(RS_ERR_CUDA, "no CUDA device: the rserve-b200 product path has no CPU fallback");
  RS_CUDA_CHECK(cudaSetDevice(opt.device));
  cudaDeviceProp prop{};
  RS_CUDA_CHECK(cudaGetDeviceProperties(&prop, opt.device));
  if (prop.major != 10)
    throw DeviceError(RS_ERR_CUDA, std::string("device ") + prop.name +
                                       " is not sm_100 (tcgen05 kernels need a B200)");
  // Stream-ordered allocations (per-request tables, decode buffers) must not
  // be trimmed back to the OS at every synchronisation (the default release
  // threshold is 0): keep the pool.
  {
    cudaMemPool_t pool;
    RS_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, opt.device));
    std::uint64_t keep = ~0ull;
    RS_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  s_ = Shapes::from(model);
  if (opt_.layer_end <= 0 || opt_.layer_end > s_.L) opt_.layer_end = s_.L;
  if (opt_.layer_begin < 0) opt_.layer_begin = 0;
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&tracker_, cudaStreamNonBlocking));
  RS_CUDA_CHECK(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
  up_.init(64ull << 20);
  max_requests_ = 512;

  // TP group rank (rs_ctx_options.tp_group): one shard per context, chunk
  // inputs handed in, no embedding slab / vision tower here
  tp_group_ = opt_.tp_group != 0;
  if (tp_group_) {
    if (opt_.tp_size < 2 || opt_.tp_size > kMaxTpRanks || opt_.tp_rank < 0 || opt_.tp_rank >= opt_.tp_size)
      throw lmmsim::ConfigError("tp group: need 2 <= tp_size <= 8 and 0 <= tp_rank < tp_size");
    if (opt_.with_vit) throw lmmsim::ConfigError("tp group: the vision tower does not live on a TP rank");
  }
  const bool first_stage = opt_.layer_begin == 0 && !tp_group_;
  if (opt_.with_vit) {
    vit_ = std::make_unique<Vit>();
    vit_->init(s_, arena_, static_cast<int>(4 * opt_.max_encode_tokens), aux_);
  }
  llm_ = std::make_unique<Llm>();
  const std::int64_t kv_pages = static_cast<std::int64_t>((opt_.kv_tokens + kPageTokens - 1) / kPageTokens);
  const int tp = opt_.tp_size > 1 ? opt_.tp_size : 1;
  if (tp > 1 && (opt_.layer_begin != 0 || opt_.layer_end != s_.L))
    throw lmmsim::ConfigError("tensor parallelism: the context must own every LLM layer");
  llm_->init(s_, arena_, opt_.layer_begin, opt_.layer_end, first_stage, opt_.with_lm_head != 0,
             static_cast<int>(opt_.max_chunk_tokens), kv_pages, kPageTokens, max_requests_, aux_,
             tp_group_ ? opt_.tp_rank : 0, tp);
  if (tp_group_) {
    // exchange buffer: [2 phases][max_chunk, d] bf16 partials + flag slots;
    // cudaMalloc'd on its own so one IPC handle maps it into peer processes
    const std::size_t part = static_cast<std::size_t>(opt_.max_chunk_tokens) * s_.d * sizeof(bf16);
    // + a 64-byte header (magic, rank, ranks, max chunk rows, d) that peers
    // check at connect: ranks with different shapes would read past each
    // other's partials
    tpx_bytes_ = 2 * part + sizeof(unsigned) * kTpBlocks * kMaxTpRanks + kTpHeaderBytes;
    RS_CUDA_CHECK(cudaMalloc(&tpx_, tpx_bytes_));
    RS_CUDA_CHECK(cudaMemsetAsync(tpx_, 0, tpx_bytes_, aux_));
    const std::int32_t hdr[5] = {kTpMagic, opt_.tp_rank, opt_.tp_size, static_cast<std::int32_t>(opt_.max_chunk_tokens),
                                 s_.d};
    RS_CUDA_CHECK(cudaMemcpyAsync(static_cast<std::uint8_t*>(tpx_) + tpx_bytes_ - kTpHeaderBytes, hdr, sizeof hdr,
                                  cudaMemcpyHostToDevice, aux_));
    RS_CUDA_CHECK(cudaStreamSynchronize(aux_));
    tp_ss_ = static_cast<unsigned long long*>(arena_.alloc(static_cast<std::size_t>(opt_.max_chunk_tokens) * 8));
    tpx_peers_.assign(static_cast<std::size_t>(tp), nullptr);
  } else if (tp > 1) {
    const std::int64_t M = static_cast<std::int64_t>(opt_.max_chunk_tokens);
    for (int r = 1; r < tp; ++r) {
      tp_shards_.push_back(std::make_unique<Llm>());
      tp_shards_.back()->init(s_, arena_, opt_.layer_begin, opt_.layer_end, false, false,
                              static_cast<int>(opt_.max_chunk_tokens), kv_pages, kPageTokens, max_requests_,
                              aux_, r, tp);
    }
    for (int r = 0; r < tp; ++r)
      tp_parts_.push_back(static_cast<bf16*>(arena_.alloc(static_cast<std::size_t>(M) * s_.d * sizeof(bf16))));
    tp_parts_dev_ = static_cast<bf16**>(arena_.alloc(sizeof(bf16*) * tp));
    RS_CUDA_CHECK(cudaMemcpyAsync(tp_parts_dev_, tp_parts_.data(), sizeof(bf16*) * tp, cudaMemcpyHostToDevice, aux_));
    tp_ss_ = static_cast<unsigned long long*>(arena_.alloc(static_cast<std::size_t>(M) * 8));
  }
  kv_pages_.reset(kv_pages);
  if (first_stage) {
    const std::int64_t slab_pages =
        static_cast<std::int64_t>((opt_.slot_tokens + kPageTokens - 1) / kPageTokens);
    slab_ = static_cast<bf16*>(arena_.alloc(static_cast<std::size_t>(slab_pages) * kPageTokens *
                                            s_.d * sizeof(bf16)));
    slab_pages_.reset(slab_pages);
  }
  page_tables_dev_ = static_cast<int**>(arena_.alloc(sizeof(int*) * max_requests_));
  RS_CUDA_CHECK(cudaMemsetAsync(page_tables_dev_, 0, sizeof(int*) * max_requests_, aux_));
  page_tables_host_.assign(static_cast<std::size_t>(max_requests_), nullptr);
  for (int i = max_requests_ - 1; i >= 0; --i) free_slots_.push_back(i);
  prefix_dev_ = static_cast<std::uint64_t*>(arena_.alloc(64));
  RS_CUDA_CHECK(cudaMallocHost(&prefix_host_, 64));
  RS_CUDA_CHECK(cudaStreamSynchronize(aux_));
}

Context::~Context() {
  cudaDeviceSynchronize();
  for (std::size_t r = 0; r < tpx_opened_.size(); ++r)
    if (tpx_opened_[r]) cudaIpcCloseMemHandle(tpx_peers_[r]);
  if (tpx_) cudaFree(tpx_);
  if (decode_x_) cudaFree(decode_x_);
  if (decode_ids_) cudaFree(decode_ids_);
  reqs_.clear();
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
  if (prefix_host_) cudaFreeHost(prefix_host_);
  if (tracker_) cudaStreamDestroy(tracker_);
  if (aux_) cudaStreamDestroy(aux_);
}

cudaEvent_t Context::new_event() {
  cudaEvent_t e;
  RS_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  events_.push_back(e);
  return e;
}

int Context::take_request_slot() {
  if (free_slots_.empty())
    throw DeviceError(RS_ERR_CUDA, "too many live requests on the device (max " +
                                       std::to_string(max_requests_) + ")");
  const int s = free_slots_.back();
  free_slots_.pop_back();
  return s;
}

DevRequest* Context::find(lmmsim::RequestId id) {
  const auto it = reqs_.find(id);
  return it == reqs_.end() ? nullptr : it->second.get();
}

DevRequest& Context::get(lmmsim::RequestId id) {
  DevRequest* r = find(id);
  if (r == nullptr) throw lmmsim::RegistryError("unknown request id " + lmmsim::format_u64(id));
  return *r;
}

namespace {
// Qwen2-VL get_rope_index: text advances (t,t,t); an image of merged grid
// (gh, gw) gets (s, s+row, s+col) and the next position is s + max(gh, gw).
void mrope_ids(const lmmsim::RequestSpec& req, const std::vector<std::pair<int, int>>& grids,
               std::vector<std::array<std::int32_t, 3>>& out) {
  std::int32_t cur = 0;
  std::size_t item = 0;
  for (const lmmsim::SegmentSpec& seg : req.segments) {
    if (seg.kind == lmmsim::SegmentKind::Text) {
      for (std::uint64_t i = 0; i < seg.tokens; ++i, ++cur) out.push_back({cur, cur, cur});
    } else {
      int gh, gw;
      if (item < grids.size()) std::tie(gh, gw) = grids[item];
      else item_grid(seg.tokens, &gh, &gw);
      ++item;
      for (int r = 0; r < gh; ++r)
        for (int c = 0; c < gw; ++c) out.push_back({cur, cur + r, cur + c});
      cur += std::max(gh, gw);
    }
  }
}
}  // namespace

void Context::attach_kv(const lmmsim::RequestSpec& req, DevRequest& r, cudaStream_t st) {
  mrope_ids(req, r.item_grids, r.rope);
  r.slot = take_request_slot();
  const std::int64_t pages = static_cast<std::int64_t>((r.total + kPageTokens - 1) / kPageTokens);
  std::vector<cudaEvent_t> kv_guards;  // KV pages: written only on the stage stream, in order
  r.kv_pages = kv_pages_.take(pages, kv_guards);
  RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&r.kv_table),
                                static_cast<std::size_t>(pages) * 4, st));
  const void* kvt = up_.put(r.kv_pages.data(), r.kv_pages.size() * 4, st);
  RS_CUDA_CHECK(cudaMemcpyAsync(r.kv_table, kvt, r.kv_pages.size() * 4, cudaMemcpyDeviceToDevice, st));
  const void* ptr_src = up_.put(&r.kv_table, sizeof(int*), st);
  RS_CUDA_CHECK(cudaMemcpyAsync(page_tables_dev_ + r.slot, ptr_src, sizeof(int*),
                                cudaMemcpyDeviceToDevice, st));
  page_tables_host_[static_cast<std::size_t>(r.slot)] = r.kv_table;
}

DevRequest& Context::create_kv_request(const lmmsim::RequestSpec& req, cudaStream_t st) {
  if (find(req.id) != nullptr)
    throw lmmsim::RegistryError("duplicate request id " + lmmsim::format_u64(req.id));
  auto owned = std::make_unique<DevRequest>();
  DevRequest& r = *owned;
  r.id = req.id;
  r.total = req.total_tokens();
  if (r.total > opt_.kv_tokens)
    throw lmmsim::ConfigError("request " + lmmsim::format_u64(req.id) + ": " +
                              lmmsim::format_u64(r.total) + " tokens exceed the KV pool");
  attach_kv(req, r, st);
  up_.fence(st);
  DevRequest* raw = owned.get();
  reqs_.emplace(req.id, std::move(owned));
  return *raw;
}

DevRequest& Context::create_request(const lmmsim::RequestSpec& req, const std::int32_t* text_ids,
                                    std::uint64_t payload_seed, cudaStream_t st,
                                    const std::vector<std::pair<int, int>>* grids) {
  if (find(req.id) != nullptr)
    throw lmmsim::RegistryError("duplicate request id " + lmmsim::format_u64(req.id));
  if (slab_ == nullptr) throw DeviceError(RS_ERR_CUDA, "context holds no embedding slab (not stage 0)");
  auto owned = std::make_unique<DevRequest>();
  DevRequest& r = *owned;
  r.id = req.id;
  r.total = req.total_tokens();
  if (r.total > opt_.max_prompt_tokens)
    throw lmmsim::ConfigError("request " + lmmsim::format_u64(req.id) + ": " +
                              lmmsim::format_u64(r.total) + " tokens exceed max_prompt_tokens");
  r.items = req.mm_item_ranges();
  std::uint64_t pos = 0, patch = 0;
  for (const lmmsim::SegmentSpec& seg : req.segments) {
    if (seg.kind == lmmsim::SegmentKind::Text) r.text_ranges.emplace_back(pos, pos + seg.tokens);
    else {
      r.item_patch_offset.push_back(patch);
      patch += 4 * seg.tokens;
    }
    pos += seg.tokens;
  }
  r.patches = patch;
  if (grids != nullptr) {
    if (grids->size() != r.items.size())
      throw lmmsim::InputError("request " + lmmsim::format_u64(req.id) + ": " + std::to_string(grids->size()) +
                               " item grids for " + std::to_string(r.items.size()) + " items");
    for (std::size_t i = 0; i < grids->size(); ++i)
      if (static_cast<std::uint64_t>((*grids)[i].first) * static_cast<std::uint64_t>((*grids)[i].second) !=
          r.items[i].length())
        throw lmmsim::InputError("request " + lmmsim::format_u64(req.id) + ": item " + std::to_string(i) +
                                 " grid does not cover its tokens");
    r.item_grids = *grids;
  }
  const std::int64_t pages = static_cast<std::int64_t>((r.total + kPageTokens - 1) / kPageTokens);
  std::vector<cudaEvent_t> guards;
  r.slot_pages = slab_pages_.take(pages, guards);
  for (cudaEvent_t g : guards) RS_CUDA_CHECK(cudaStreamWaitEvent(st, g, 0));
  attach_kv(req, r, st);

  const std::size_t words = static_cast<std::size_t>((r.total + 31) / 32);
  RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&r.bitmap), words * 4, st));
  RS_CUDA_CHECK(cudaMemsetAsync(r.bitmap, 0, words * 4, st));

  // Text: readiness bits + K8 gather of the token embeddings into the slots.
  std::vector<std::uint64_t> ranges;
  std::vector<std::int32_t> ids;
  std::vector<std::int64_t> rows;
  std::size_t k = 0;
  for (const auto& [b, e] : r.text_ranges) {
    ranges.push_back(b);
    ranges.push_back(e);
    for (std::uint64_t t = b; t < e; ++t, ++k) {
      std::int32_t id;
      if (text_ids != nullptr) {
        id = text_ids[k];
        if (id < 0 || id >= s_.vocab)
          throw lmmsim::InputError("request " + lmmsim::format_u64(req.id) + ": token id " +
                                   std::to_string(id) + " outside the vocabulary");
      } else {
        id = static_cast<std::int32_t>(mix64(payload_seed, (6ull << 32) | req.id, t) %
                                       static_cast<std::uint64_t>(s_.vocab));
      }
      ids.push_back(id);
      rows.push_back(r.slab_row(t));
    }
  }
  if (!ranges.empty()) {
    const auto* rng = static_cast<const std::uint64_t*>(up_.put(ranges.data(), ranges.size() * 8, st));
    bitmap_set_ranges(r.bitmap, rng, static_cast<int>(ranges.size() / 2), st);
    const auto* idd = static_cast<const std::int32_t*>(up_.put(ids.data(), ids.size() * 4, st));
    const auto* rwd = static_cast<const std::int64_t*>(up_.put(rows.data(), rows.size() * 8, st));
    gather_text_embeddings(llm_->embed(), idd, static_cast<int>(ids.size()), rwd, slab_, s_.d, st);
  }
  up_.fence(st);
  DevRequest* raw = owned.get();
  reqs_.emplace(req.id, std::move(owned));
  return *raw;
}

void Context::scatter_items(DevRequest& r, const std::vector<lmmsim::TokenRange>& items,
                            const bf16* rows_src, cudaStream_t st) {
  std::vector<std::int64_t> rows;
  std::vector<std::uint64_t> ranges;
  for (const lmmsim::TokenRange& it : items) {
    ranges.push_back(it.start);
    ranges.push_back(it.end);
    for (std::uint64_t t = it.start; t < it.end; ++t) rows.push_back(r.slab_row(t));
  }
  const auto* rwd = static_cast<const std::int64_t*>(up_.put(rows.data(), rows.size() * 8, st));
  const auto* rng = static_cast<const std::uint64_t*>(up_.put(ranges.data(), ranges.size() * 8, st));
  scatter_rows_and_mark(rows_src, static_cast<int>(rows.size()), rwd, slab_, s_.d, r.bitmap, rng,
                        static_cast<int>(ranges.size() / 2), st);
  up_.fence(st);
}

void Context::release_prefix(DevRequest& r, std::uint64_t released_end, cudaEvent_t guard) {
  const std::uint64_t full_pages =
      released_end >= r.total ? r.slot_pages.size() : released_end / kPageTokens;
  std::vector<int> give;
  for (std::uint64_t p = r.slot_freed_tokens / kPageTokens; p < full_pages; ++p) {
    give.push_back(r.slot_pages[p]);
    r.slot_pages[p] = -1;
  }
  r.slot_freed_tokens = full_pages * kPageTokens;
  slab_pages_.give(give, guard);
}

void Context::erase_request(lmmsim::RequestId id, cudaEvent_t guard, bool keep_slot) {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) throw lmmsim::RegistryError("erase of unknown request id " + lmmsim::format_u64(id));
  DevRequest& r = *it->second;
  release_prefix(r, r.total, guard);
  kv_pages_.give(r.kv_pages, guard);
  if (guard != nullptr) RS_CUDA_CHECK(cudaStreamWaitEvent(tracker_, guard, 0));
  if (r.bitmap != nullptr) RS_CUDA_CHECK(cudaFreeAsync(r.bitmap, tracker_));
  RS_CUDA_CHECK(cudaFreeAsync(r.kv_table, tracker_));
  if (!keep_slot) free_slots_.push_back(r.slot);
  reqs_.erase(it);
}

std::uint64_t Context::device_schedulable(DevRequest& r, std::uint64_t frontier) {
  ready_prefix(r.bitmap, frontier, r.total, prefix_dev_, tracker_);
  RS_CUDA_CHECK(cudaMemcpyAsync(prefix_host_, prefix_dev_, 8, cudaMemcpyDeviceToHost, tracker_));
  RS_CUDA_CHECK(cudaStreamSynchronize(tracker_));
  return *prefix_host_ - frontier;
}

VitBatchPlan Context::plan_batch(const DevRequest& r,
                                 const std::vector<lmmsim::TokenRange>& items) const {
  VitBatchPlan plan;
  plan.cu_window.push_back(0);
  plan.cu_item.push_back(0);
  for (const lmmsim::TokenRange& it : items) {
    int gh = 0, gw = 0;
    for (std::size_t k = 0; k < r.item_grids.size() && k < r.items.size(); ++k)
      if (r.items[k].start == it.start) std::tie(gh, gw) = r.item_grids[k];
    if (gh == 0) item_grid(it.length(), &gh, &gw);
    plan_item(gh, gw, s_.win, plan.tokens, plan);
  }
  finalize_plan(plan);
  return plan;
}

void Context::encode(const VitBatchPlan& plan, const bf16* patches_dev, bf16* out, cudaStream_t st) {
  if (!vit_) throw DeviceError(RS_ERR_CUDA, "context holds no vision encoder");
  const auto* pos = static_cast<const std::int32_t*>(up_.put(plan.pos_hw.data(), plan.pos_hw.size() * 4, st));
  const auto* cuw = static_cast<const std::int32_t*>(up_.put(plan.cu_window.data(), plan.cu_window.size() * 4, st));
  const auto* cui = static_cast<const std::int32_t*>(up_.put(plan.cu_item.data(), plan.cu_item.size() * 4, st));
  const auto* orow = static_cast<const std::int32_t*>(up_.put(plan.out_row.data(), plan.out_row.size() * 4, st));
  // window tiles followed by the per-row window table (attention_window_tc)
  std::vector<std::uint8_t> wbuf(plan.win_blocks.size() * sizeof(AttnBlock) + plan.win_row.size() * 4);
  std::memcpy(wbuf.data(), plan.win_blocks.data(), plan.win_blocks.size() * sizeof(AttnBlock));
  std::memcpy(wbuf.data() + plan.win_blocks.size() * sizeof(AttnBlock), plan.win_row.data(), plan.win_row.size() * 4);
  const auto* wb = static_cast<const AttnBlock*>(up_.put(wbuf.data(), wbuf.size(), st));
  const auto* fb = static_cast<const AttnBlock*>(
      up_.put(plan.full_blocks.data(), plan.full_blocks.size() * sizeof(AttnBlock), st));
  vit_->encode(plan, patches_dev, pos, cuw, cui, orow, wb, fb, out, st);
  up_.fence(st);
}

void Context::prefill(const std::vector<SliceRef>& slices, bf16* x, cudaStream_t st,
                      int layer_from, int layer_to) {
  std::vector<ChunkRowInfo> rows;
  std::vector<std::int64_t> gather;
  std::vector<PrefillWork> work;
  std::vector<std::int64_t> done_rows;
  std::vector<std::int32_t> done_slots;
  const int l_from = layer_from < 0 ? llm_->layer_begin() : layer_from;
  const int l_to = layer_to < 0 ? llm_->layer_end() : layer_to;
  const bool first = l_from == 0 && slab_ != nullptr;  // TP group ranks: chunk input handed in
  for (const SliceRef& sl : slices) {
    const int base = static_cast<int>(rows.size());
    for (std::uint64_t p = sl.start; p < sl.end; ++p) {
      const auto& rp = sl.req->rope[p];
      rows.push_back({sl.req->slot, static_cast<std::int32_t>(p), {rp[0], rp[1], rp[2]}, 0});
      if (first) gather.push_back(sl.req->slab_row(p));
    }
    const std::uint64_t unit = static_cast<std::uint64_t>(attn_unit_rows());
    for (std::uint64_t q = sl.start; q < sl.end; q += unit)
      work.push_back({base + static_cast<int>(q - sl.start),
                      static_cast<int>(std::min<std::uint64_t>(unit, sl.end - q)),
                      static_cast<int>(q), sl.req->slot});
    if (sl.end == sl.req->total) {
      done_rows.push_back(base + static_cast<std::int64_t>(sl.end - sl.start) - 1);
      done_slots.push_back(sl.req->slot);
    }
  }
  // Most keys first: the attention grid issues work items in this order
  // (LPT over the SMs; attention_tc.cu).
  std::stable_sort(work.begin(), work.end(), [](const PrefillWork& a, const PrefillWork& b) {
    return a.q_pos0 + a.q_rows > b.q_pos0 + b.q_rows;
  });
  ChunkDev c;
  c.M = static_cast<int>(rows.size());
  c.rows = static_cast<const ChunkRowInfo*>(up_.put(rows.data(), rows.size() * sizeof(ChunkRowInfo), st));
  if (first) c.gather_rows = static_cast<const std::int64_t*>(up_.put(gather.data(), gather.size() * 8, st));
  c.work = static_cast<const PrefillWork*>(up_.put(work.data(), work.size() * sizeof(PrefillWork), st));
  c.work_host = work.data();
  c.n_work = static_cast<int>(work.size());
  c.max_keys = work.empty() ? 0 : work.front().q_pos0 + work.front().q_rows;  // sorted: most keys first
  if (llm_->has_head() && l_to == llm_->layer_end() && !done_rows.empty()) {
    c.done_rows = static_cast<const std::int64_t*>(up_.put(done_rows.data(), done_rows.size() * 8, st));
    c.done_slots = static_cast<const std::int32_t*>(up_.put(done_slots.data(), done_slots.size() * 4, st));
    c.n_done = static_cast<int>(done_rows.size());
  }
  {
    HostPhase ph("prefill.run_llm");
    run_llm(c, slab_, x, st, l_from, l_to);
  }
  HostPhase ph("prefill.fence");
  up_.fence(st);
}

// Tensor-parallel pass over all shards (same device: loopback ranks; the
// reduction reads every shard's partial through the pointer table, which on
// an NVSwitch box holds peer addresses): per layer, every shard's attention
// block -> O partial, reduce into x (shard order, + folded-norm sums of
// squares), every shard's MLP -> down partial, reduce.
void Context::run_llm(const ChunkDev& c, const bf16* slab, bf16* x, cudaStream_t st, int l_from, int l_to) {
  if (tp_group_) {
    if (!tp_connected_) throw lmmsim::ConfigError("tp group: rs_tp_connect first");
    if (l_from < 0) l_from = llm_->layer_begin();
    if (l_to < 0) l_to = llm_->layer_end();
    const int T = opt_.tp_size;
    const std::size_t part = static_cast<std::size_t>(opt_.max_chunk_tokens) * s_.d * sizeof(bf16);
    TpGroupArgs a{};
    a.x = x;
    a.rows = c.M;
    a.d = s_.d;
    a.T = T;
    a.rank = opt_.tp_rank;
    a.ss = tp_ss_;
    for (int r = 0; r < T; ++r)
      a.flags[r] = reinterpret_cast<unsigned*>(static_cast<std::uint8_t*>(tpx_peers_[static_cast<std::size_t>(r)]) + 2 * part);
    auto reduce = [&]() {
      const int ph = static_cast<int>((tp_epoch_ + 1) & 1u);  // = my_part()'s phase
      for (int r = 0; r < T; ++r)
        a.parts[r] = reinterpret_cast<const bf16*>(static_cast<std::uint8_t*>(tpx_peers_[static_cast<std::size_t>(r)]) + ph * part);
      a.epoch = ++tp_epoch_;
      tp_group_reduce(a, st);
    };
    auto my_part = [&]() {  // the partial of the coming reduce (epoch + 1)
      return reinterpret_cast<bf16*>(static_cast<std::uint8_t*>(tpx_) + ((tp_epoch_ + 1) & 1u) * part);
    };
    llm_->tp_begin(c, st);
    for (int l = l_from; l < l_to; ++l) {
      // O partial -> this rank's exchange buffer, then the peer-memory reduction
      // (double-buffered by phase: a rank rewrites a phase buffer only after every
      // rank has signalled the next phase, i.e. finished reading it)
      llm_->tp_attn_partial(l, c, slab, x, l == l_from, tp_ss_, page_tables_dev_, my_part(), st);
      reduce();
      llm_->tp_mlp_partial(l, c, x, tp_ss_, my_part(), st);
      reduce();
    }
    if (l_to == llm_->layer_end()) llm_->head_phase(c, x, st);
    return;
  }
  if (tp_shards_.empty()) {
    llm_->forward_stage(c, slab, x, page_tables_dev_, st, l_from, l_to);
    return;
  }
  if (l_from < 0) l_from = llm_->layer_begin();
  if (l_to < 0) l_to = llm_->layer_end();
  std::vector<Llm*> sh{llm_.get()};
  for (auto& p : tp_shards_) sh.push_back(p.get());
  const int T = static_cast<int>(sh.size());
  for (Llm* l : sh) l->tp_begin(c, st);
  for (int l = l_from; l < l_to; ++l) {
    for (int t = 0; t < T; ++t)
      sh[static_cast<std::size_t>(t)]->tp_attn_partial(l, c, slab, x, l == l_from, tp_ss_, page_tables_dev_,
                                                       tp_parts_[static_cast<std::size_t>(t)], st);
    tp_reduce_residual(x, c.M, s_.d, tp_parts_dev_, T, tp_ss_, st);
    for (int t = 0; t < T; ++t)
      sh[static_cast<std::size_t>(t)]->tp_mlp_partial(l, c, x, tp_ss_, tp_parts_[static_cast<std::size_t>(t)], st);
    tp_reduce_residual(x, c.M, s_.d, tp_parts_dev_, T, tp_ss_, st);
  }
  if (l_to == llm_->layer_end()) llm_->head_phase(c, x, st);
}

double Context::decode(const std::vector<lmmsim::RequestId>& ids, int steps, std::int32_t* out_tokens,
                       float* out_logits, cudaStream_t st) {
  if (!llm_ || !llm_->has_head() || llm_->layer_begin() != 0)
    throw lmmsim::ConfigError("decode needs the whole LLM and its head on this context");
  if (tp_group_) throw lmmsim::ConfigError("decode: not on a TP group rank (prefill only)");
  const int n = static_cast<int>(ids.size());
  if (n <= 0 || steps <= 0) return 0.0;
  if (n > opt_.max_chunk_tokens) throw lmmsim::ConfigError("decode: more requests than max_chunk_tokens");
  std::vector<DevRequest*> reqs;
  std::vector<std::int32_t> slots;
  std::vector<std::int32_t> next_rope;
  for (lmmsim::RequestId id : ids) {
    DevRequest& r = get(id);
    reqs.push_back(&r);
    slots.push_back(r.slot);
    if (r.next_rope < 0) {  // first decode call: generated text continues after the prompt's max id
      std::int32_t mx = -1;
      for (const auto& p : r.rope) mx = std::max({mx, p[0], p[1], p[2]});
      r.next_rope = mx + 1;
    }
    next_rope.push_back(r.next_rope);
    // KV pages for every decoded token, appended to the request's page table
    const std::uint64_t need = (r.total + static_cast<std::uint64_t>(steps) + kPageTokens - 1) / kPageTokens;
    if (need > r.kv_pages.size()) {
      std::vector<cudaEvent_t> guards;
      const std::vector<int> more = kv_pages_.take(static_cast<std::int64_t>(need - r.kv_pages.size()), guards);
      for (cudaEvent_t g : guards) RS_CUDA_CHECK(cudaStreamWaitEvent(st, g, 0));
      r.kv_pages.insert(r.kv_pages.end(), more.begin(), more.end());
      int* table = nullptr;
      RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&table), r.kv_pages.size() * 4, st));
      const void* src = up_.put(r.kv_pages.data(), r.kv_pages.size() * 4, st);
      RS_CUDA_CHECK(cudaMemcpyAsync(table, src, r.kv_pages.size() * 4, cudaMemcpyDeviceToDevice, st));
      RS_CUDA_CHECK(cudaFreeAsync(r.kv_table, st));
      r.kv_table = table;
      const void* ptr_src = up_.put(&r.kv_table, sizeof(int*), st);
      RS_CUDA_CHECK(cudaMemcpyAsync(page_tables_dev_ + r.slot, ptr_src, sizeof(int*), cudaMemcpyDeviceToDevice, st));
      page_tables_host_[static_cast<std::size_t>(r.slot)] = r.kv_table;
    }
  }
  if (decode_x_cap_ < n) {
    if (decode_x_ != nullptr) RS_CUDA_CHECK(cudaFreeAsync(decode_x_, st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&decode_x_), static_cast<std::size_t>(n) * s_.d * 2, st));
    RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&decode_ids_), static_cast<std::size_t>(n) * 4, st));
    decode_x_cap_ = n;
  }
  std::int32_t* tok_dev = nullptr;
  RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&tok_dev), static_cast<std::size_t>(steps) * n * 4, st));
  std::vector<std::int64_t> done_rows(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) done_rows[static_cast<std::size_t>(i)] = i;
  const auto* rows_idx = static_cast<const std::int64_t*>(up_.put(done_rows.data(), done_rows.size() * 8, st));
  const auto* slots_dev = static_cast<const std::int32_t*>(up_.put(slots.data(), slots.size() * 4, st));
  up_.fence(st);
  cudaEvent_t e0, e1;
  RS_CUDA_CHECK(cudaEventCreate(&e0));
  RS_CUDA_CHECK(cudaEventCreate(&e1));
  RS_CUDA_CHECK(cudaEventRecord(e0, st));
  for (int step = 0; step < steps; ++step) {
    std::vector<ChunkRowInfo> info;
    std::vector<PrefillWork> work;
    for (int i = 0; i < n; ++i) {
      const DevRequest& r = *reqs[static_cast<std::size_t>(i)];
      const std::int32_t pos = static_cast<std::int32_t>(r.total) + step;
      const std::int32_t rp = next_rope[static_cast<std::size_t>(i)] + step;
      info.push_back({r.slot, pos, {rp, rp, rp}, 0});
      work.push_back({i, 1, pos, r.slot});
    }
    ChunkDev c;
    c.M = n;
    c.rows = static_cast<const ChunkRowInfo*>(up_.put(info.data(), info.size() * sizeof(ChunkRowInfo), st));
    c.work = static_cast<const PrefillWork*>(up_.put(work.data(), work.size() * sizeof(PrefillWork), st));
    c.work_host = work.data();
    c.n_work = n;
    c.done_rows = rows_idx;
    c.done_slots = slots_dev;
    c.n_done = n;
    static const bool tc_decode = [] {  // RS_DECODE_ATTN=tc: prefill kernel (A/B)
      const char* e = std::getenv("RS_DECODE_ATTN");
      return e != nullptr && std::string(e) == "tc";
    }();
    c.decode = !tc_decode;
    for (const PrefillWork& wk : work) c.max_keys = std::max(c.max_keys, wk.q_pos0 + 1);
    // previous token (prefill argmax, then each step's) -> embedding rows
    gather_slots_i32(llm_->argmax_dev(), slots_dev, n, decode_ids_, st);
    gather_text_embeddings(llm_->embed(), decode_ids_, n, rows_idx, decode_x_, s_.d, st);
    run_llm(c, nullptr, decode_x_, st, -1, -1);
    gather_slots_i32(llm_->argmax_dev(), slots_dev, n, tok_dev + static_cast<std::int64_t>(step) * n, st);
    if (out_logits != nullptr)
      for (int i = 0; i < n; ++i)
        RS_CUDA_CHECK(cudaMemcpyAsync(out_logits + (static_cast<std::int64_t>(step) * n + i) * s_.vocab,
                                      llm_->logits_row(slots[static_cast<std::size_t>(i)]),
                                      static_cast<std::size_t>(s_.vocab) * 4, cudaMemcpyDeviceToHost, st));
    up_.fence(st);
  }
  RS_CUDA_CHECK(cudaEventRecord(e1, st));
  RS_CUDA_CHECK(cudaMemcpyAsync(out_tokens, tok_dev, static_cast<std::size_t>(steps) * n * 4,
                                cudaMemcpyDeviceToHost, st));
  RS_CUDA_CHECK(cudaFreeAsync(tok_dev, st));
  RS_CUDA_CHECK(cudaStreamSynchronize(st));
  float ms = 0;
  RS_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  RS_CUDA_CHECK(cudaEventDestroy(e0));
  RS_CUDA_CHECK(cudaEventDestroy(e1));
  for (DevRequest* r : reqs) {  // KV now holds the decoded tokens; M-RoPE ids move on with them
    r->total += static_cast<std::uint64_t>(steps);
    r->next_rope += steps;
  }
  return ms;
}

void Context::free_kept(lmmsim::RequestId id) {
  DevRequest& r = get(id);
  const int slot = r.slot;
  r.slot_freed_tokens = r.total;  // slab pages were released with the prompt
  kv_pages_.give(r.kv_pages, nullptr);
  if (r.bitmap != nullptr) RS_CUDA_CHECK(cudaFreeAsync(r.bitmap, tracker_));
  RS_CUDA_CHECK(cudaFreeAsync(r.kv_table, tracker_));
  reqs_.erase(id);
  free_slots_.push_back(slot);
}

std::uint64_t Context::chunk_flops(const std::vector<SliceRef>& slices) const {
  std::uint64_t tokens = 0, att = 0;
  const std::uint64_t layers = static_cast<std::uint64_t>(llm_->layer_end() - llm_->layer_begin());
  for (const SliceRef& sl : slices) {
    tokens += sl.end - sl.start;
    // causal attention over the prefix: 4 * hq * hd per (q, k) pair, k <= q
    for (std::uint64_t q = sl.start; q < sl.end; ++q)
      att += 4ull * static_cast<std::uint64_t>(s_.hq * s_.hd) * (q + 1);
  }
  return llm_->dense_flops(tokens) + att * layers;
}

void Context::copy_logits(int slot, float* host, cudaStream_t st) {
  RS_CUDA_CHECK(cudaMemcpyAsync(host, llm_->logits_row(slot), static_cast<std::size_t>(s_.vocab) * 4,
                                cudaMemcpyDeviceToHost, st));
}

}  // namespace rserve

// ---- PD (prefill -> decode) KV transfer ----------------------------------------
namespace rserve {
namespace {
constexpr std::uint64_t kKvImageHeader = 64;  // [0] first token (i32), [4] next M-RoPE id, [8] tokens (u64)
}

std::uint64_t Context::kv_image_bytes(std::uint64_t tokens) const {
  if (!llm_) throw lmmsim::ConfigError("KV image: this context holds no LLM layers");
  const Shapes& ls = llm_->shapes();
  const std::uint64_t pages = (tokens + kPageTokens - 1) / kPageTokens;
  const std::uint64_t page_bytes = static_cast<std::uint64_t>(ls.hkv) * kPageTokens * ls.hd * 2;
  const std::uint64_t shards = 1 + tp_shards_.size();
  const std::uint64_t layers = static_cast<std::uint64_t>(llm_->layer_end() - llm_->layer_begin());
  return kKvImageHeader + shards * layers * pages * 2 * page_bytes;
}

namespace {
// (src, dst) page pairs of a request's KV image, in image order.
std::vector<PageCopy> kv_image_pages(const std::vector<Llm*>& shards, const std::vector<int>& kv_pages,
                                     std::uint64_t n_pages, std::uint8_t* image, std::size_t page_bytes,
                                     bool to_image) {
  std::vector<PageCopy> list;
  list.reserve(shards.size() * n_pages * 2 * 80);
  std::uint8_t* cur = image + kKvImageHeader;
  for (Llm* sh : shards) {
    for (int l = sh->layer_begin(); l < sh->layer_end(); ++l) {
      for (std::uint64_t i = 0; i < n_pages; ++i) {
        for (int kv = 0; kv < 2; ++kv) {
          std::uint8_t* page = reinterpret_cast<std::uint8_t*>(kv == 0 ? sh->k_cache(l) : sh->v_cache(l)) +
                               static_cast<std::size_t>(kv_pages[i]) * page_bytes;
          list.push_back(to_image ? PageCopy{page, cur} : PageCopy{cur, page});
          cur += page_bytes;
        }
      }
    }
  }
  return list;
}
}  // namespace

void Context::export_kv(lmmsim::RequestId id, void* dst, std::uint64_t cap, rs_kv_meta* meta, cudaStream_t st) {
  DevRequest& r = get(id);
  if (!llm_ || !llm_->has_head())
    throw lmmsim::ConfigError("KV export: the request's first token lives on the last stage (needs the LM head)");
  if (r.kv_pages.empty()) throw lmmsim::InternalError("KV export: request " + lmmsim::format_u64(id) + " holds no KV");
  if (r.slot_freed_tokens < r.total)  // a kept request has been prefilled (and its slab released) to the end
    throw lmmsim::InternalError("KV export: request " + lmmsim::format_u64(id) + " is not fully prefilled");
  const std::uint64_t bytes = kv_image_bytes(r.total);
  if (cap < bytes)
    throw lmmsim::ConfigError("KV export: buffer of " + lmmsim::format_u64(cap) + " bytes < image of " +
                              lmmsim::format_u64(bytes));
  if (r.next_rope < 0) {  // as Context::decode: generated text continues after the prompt's max id
    std::int32_t mx = -1;
    for (const auto& p : r.rope) mx = std::max({mx, p[0], p[1], p[2]});
    r.next_rope = mx + 1;
  }
  const Shapes& ls = llm_->shapes();
  const std::size_t page_bytes = static_cast<std::size_t>(ls.hkv) * kPageTokens * ls.hd * 2;
  const std::uint64_t n_pages = (r.total + kPageTokens - 1) / kPageTokens;
  std::vector<Llm*> shards{llm_.get()};
  for (auto& p : tp_shards_) shards.push_back(p.get());
  auto* image = static_cast<std::uint8_t*>(dst);
  const std::vector<PageCopy> list = kv_image_pages(shards, r.kv_pages, n_pages, image, page_bytes, true);
  struct {
    std::int32_t rope;
    std::int32_t pad;
    std::uint64_t tokens;
  } hdr{r.next_rope, 0, r.total};
  RS_CUDA_CHECK(cudaMemcpyAsync(image, llm_->argmax_dev() + r.slot, 4, cudaMemcpyDeviceToDevice, st));
  RS_CUDA_CHECK(cudaMemcpyAsync(image + 4, up_.put(&hdr, sizeof hdr, st), sizeof hdr, cudaMemcpyDeviceToDevice, st));
  const auto* ld = static_cast<const PageCopy*>(up_.put(list.data(), list.size() * sizeof(PageCopy), st));
  copy_pages(ld, static_cast<int>(list.size()), page_bytes, st, "kv_image_pack");
  up_.fence(st);
  rs_kv_meta m{};
  m.tokens = r.total;
  m.image_bytes = bytes;
  m.next_rope = r.next_rope;
  m.layer_begin = llm_->layer_begin();
  m.layer_end = llm_->layer_end();
  m.kv_heads = ls.hkv * static_cast<int>(shards.size());
  m.head_dim = ls.hd;
  m.page_tokens = kPageTokens;
  m.tp_size = static_cast<int>(shards.size());
  *meta = m;
}

void Context::import_kv(lmmsim::RequestId id, const rs_kv_meta& meta, const void* src, cudaStream_t st) {
  if (!llm_ || !llm_->has_head() || llm_->layer_begin() != 0)
    throw lmmsim::ConfigError("KV import: decode needs the whole LLM and its head on this context");
  if (find(id) != nullptr) throw lmmsim::RegistryError("duplicate request id " + lmmsim::format_u64(id));
  const Shapes& ls = llm_->shapes();
  const int shards_n = 1 + static_cast<int>(tp_shards_.size());
  if (meta.layer_begin != llm_->layer_begin() || meta.layer_end != llm_->layer_end() ||
      meta.kv_heads != ls.hkv * shards_n || meta.head_dim != ls.hd || meta.page_tokens != kPageTokens ||
      meta.tp_size != shards_n)
    throw lmmsim::ConfigError("KV import: image of layers [" + std::to_string(meta.layer_begin) + ", " +
                              std::to_string(meta.layer_end) + "), " + std::to_string(meta.kv_heads) +
                              " kv heads x " + std::to_string(meta.head_dim) + ", TP " +
                              std::to_string(meta.tp_size) + " does not match this context");
  if (meta.tokens == 0 || meta.tokens > opt_.kv_tokens)
    throw lmmsim::ConfigError("KV import: " + lmmsim::format_u64(meta.tokens) + " tokens exceed the KV pool");
  if (meta.image_bytes != kv_image_bytes(meta.tokens)) throw lmmsim::InputError("KV import: image size mismatch");
  auto owned = std::make_unique<DevRequest>();
  DevRequest& r = *owned;
  r.id = id;
  r.total = meta.tokens;
  r.next_rope = meta.next_rope;
  r.slot_freed_tokens = r.total;  // no embedding slot on the decode side
  r.slot = take_request_slot();
  const std::int64_t pages = static_cast<std::int64_t>((r.total + kPageTokens - 1) / kPageTokens);
  std::vector<cudaEvent_t> guards;
  r.kv_pages = kv_pages_.take(pages, guards);
  for (cudaEvent_t g : guards) RS_CUDA_CHECK(cudaStreamWaitEvent(st, g, 0));
  RS_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&r.kv_table), static_cast<std::size_t>(pages) * 4, st));
  RS_CUDA_CHECK(cudaMemcpyAsync(r.kv_table, up_.put(r.kv_pages.data(), r.kv_pages.size() * 4, st),
                                r.kv_pages.size() * 4, cudaMemcpyDeviceToDevice, st));
  RS_CUDA_CHECK(cudaMemcpyAsync(page_tables_dev_ + r.slot, up_.put(&r.kv_table, sizeof(int*), st), sizeof(int*),
                                cudaMemcpyDeviceToDevice, st));
  page_tables_host_[static_cast<std::size_t>(r.slot)] = r.kv_table;
  // the prefill's first token -> this slot's argmax (rs_decode embeds it first)
  RS_CUDA_CHECK(cudaMemcpyAsync(llm_->argmax_dev() + r.slot, src, 4, cudaMemcpyDeviceToDevice, st));
  std::vector<Llm*> shards{llm_.get()};
  for (auto& p : tp_shards_) shards.push_back(p.get());
  const std::size_t page_bytes = static_cast<std::size_t>(ls.hkv) * kPageTokens * ls.hd * 2;
  const std::vector<PageCopy> list =
      kv_image_pages(shards, r.kv_pages, static_cast<std::uint64_t>(pages),
                     static_cast<std::uint8_t*>(const_cast<void*>(src)), page_bytes, false);
  const auto* ld = static_cast<const PageCopy*>(up_.put(list.data(), list.size() * sizeof(PageCopy), st));
  copy_pages(ld, static_cast<int>(list.size()), page_bytes, st, "kv_image_unpack");
  up_.fence(st);
  reqs_.emplace(id, std::move(owned));
}

}  // namespace rserve

// ---- tensor parallelism across GPUs: exchange buffers -------------------------
namespace rserve {
void Context::tp_buffer(void** dev, cudaIpcMemHandle_t* handle) {
  if (!tp_group_) throw lmmsim::ConfigError("tp buffer: not a TP group rank (rs_ctx_options.tp_group)");
  if (dev) *dev = tpx_;
  if (handle) RS_CUDA_CHECK(cudaIpcGetMemHandle(handle, tpx_));
}

void Context::tp_connect(const void* const* ptrs, const cudaIpcMemHandle_t* handles) {
  if (!tp_group_) throw lmmsim::ConfigError("tp connect: not a TP group rank");
  if (tp_connected_) throw lmmsim::ConfigError("tp connect: already connected");
  const int T = opt_.tp_size;
  tpx_opened_.assign(static_cast<std::size_t>(T), false);
  for (int r = 0; r < T; ++r) {
    void*& p = tpx_peers_[static_cast<std::size_t>(r)];
    if (r == opt_.tp_rank) {
      p = tpx_;
    } else if (ptrs != nullptr && ptrs[r] != nullptr) {  // a rank of this process (same address space)
      p = const_cast<void*>(ptrs[r]);
    } else {
      if (handles == nullptr) throw lmmsim::ConfigError("tp connect: rank " + std::to_string(r) + " has no address");
      RS_CUDA_CHECK(cudaIpcOpenMemHandle(&p, handles[r], cudaIpcMemLazyEnablePeerAccess));
      tpx_opened_[static_cast<std::size_t>(r)] = true;
    }
  }
  // every rank's header: same group size / chunk rows / width, rank r at slot r
  for (int r = 0; r < T; ++r) {
    std::int32_t h[5];
    RS_CUDA_CHECK(cudaMemcpy(h, static_cast<std::uint8_t*>(tpx_peers_[static_cast<std::size_t>(r)]) + tpx_bytes_ -
                                    kTpHeaderBytes, sizeof h, cudaMemcpyDeviceToHost));
    if (h[0] != kTpMagic || h[1] != r || h[2] != T || h[3] != static_cast<std::int32_t>(opt_.max_chunk_tokens) ||
        h[4] != s_.d)
      throw lmmsim::ConfigError("tp connect: rank " + std::to_string(r) + "'s exchange buffer is not a rank " +
                                std::to_string(r) + " of this group (ranks " + std::to_string(h[2]) + ", chunk rows " +
                                std::to_string(h[3]) + ", width " + std::to_string(h[4]) + ")");
  }
  RS_CUDA_CHECK(cudaStreamSynchronize(aux_));  // the zeroed flags are in place before any peer signals
  tp_connected_ = true;
}
}  // namespace rserve
