// rserve-b200 — per-GPU pipeline context: model weights, embedding-slot
// slab + readiness bitmaps (the device tracker), paged KV pools, streams,
// metadata uploads. Used by the C-ABI (capi_device.cu) both directly
// (tracker-level entry points) and through the engine backend
// (device_backend.cu).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <deque>
#include <list>
#include <memory>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "lmmsim/tracker.hpp"
#include "model.cuh"
#include "rserve.h"

namespace rserve {

constexpr int kPageTokens = 64;  // slot pages and KV pages
constexpr std::size_t kTpHeaderBytes = 64;       // TP exchange buffer header (at its end)
constexpr std::int32_t kTpMagic = 0x52535450;    // "RSTP"

/// Hash stream of the synthetic pixels of multimodal item `item` of request `req`.
inline std::uint64_t pixel_stream(std::uint64_t req, std::uint64_t item) {
  return (5ull << 32) | (req << 12) | item;
}

/// Free list of fixed-size pages; a freed page may carry the CUDA event
/// after which it is safe to overwrite (its last reader's completion).
class PagePool {
 public:
  void reset(std::int64_t pages);
  /// Takes n pages; appends guard events that writers must wait on.
  std::vector<int> take(std::int64_t n, std::vector<cudaEvent_t>& guards);
  void give(const std::vector<int>& pages, cudaEvent_t guard);
  /// Drops all guard events (call only when the device is idle).
  void clear_guards() {
    for (auto& p : free_) p.second = nullptr;
  }
  std::int64_t available() const { return static_cast<std::int64_t>(free_.size()); }
  std::int64_t capacity() const { return cap_; }

 private:
  std::deque<std::pair<int, cudaEvent_t>> free_;
  std::int64_t cap_ = 0;
};

/// Pinned-host -> device ring for per-op metadata (chunk / batch descriptors).
class Uploader {
 public:
  void init(std::size_t bytes);
  ~Uploader();
  /// Copies `n` bytes from host to a device region (async on `st`), returns
  /// the device pointer. Regions are recycled after the fence covering them.
  void* put(const void* src, std::size_t n, cudaStream_t st);
  /// Marks everything put so far as consumed once work now on `st` finishes.
  void fence(cudaStream_t st);
  std::uint64_t bytes_uploaded() const { return uploaded_; }

 private:
  static constexpr std::size_t kNone = ~std::size_t{0};
  std::uint8_t* host_ = nullptr;
  std::uint8_t* dev_ = nullptr;
  std::size_t cap_ = 0, head_ = 0, pending_begin_ = kNone;
  struct Mark {
    std::size_t begin, end;
    std::shared_ptr<CUevent_st> ev;
  };
  std::list<Mark> marks_;
  std::vector<std::pair<std::size_t, std::size_t>> pending_;
  std::uint64_t uploaded_ = 0;
};

struct DevRequest {
  lmmsim::RequestId id = 0;
  int slot = -1;                       // request table / logits slot
  std::uint64_t total = 0;
  std::vector<lmmsim::TokenRange> items;
  std::vector<std::pair<std::uint64_t, std::uint64_t>> text_ranges;
  std::vector<int> slot_pages;         // embedding slab pages (-1 once freed)
  std::uint64_t slot_freed_tokens = 0; // prefix whose pages are back in the pool
  std::vector<int> kv_pages;
  std::uint32_t* bitmap = nullptr;     // device readiness words
  int* kv_table = nullptr;             // device page table (kv_pages)
  std::vector<std::array<std::int32_t, 3>> rope;  // M-RoPE ids per token
  std::int32_t next_rope = -1;         // decode: M-RoPE id of the next generated token (-1: not started)
  std::vector<std::uint64_t> item_patch_offset;   // first patch of each item
  std::vector<std::pair<int, int>> item_grids;     // merged-token grid of each item
  std::uint64_t patches = 0;

  std::int64_t slab_row(std::uint64_t pos) const {
    return static_cast<std::int64_t>(slot_pages[pos / kPageTokens]) * kPageTokens +
           static_cast<std::int64_t>(pos % kPageTokens);
  }
};

/// One prefill slice (request, [start, end)).
struct SliceRef {
  DevRequest* req;
  std::uint64_t start, end;
};

class Context {
 public:
  Context(const rs_model_config& model, const rs_ctx_options& opt);
  ~Context();

  const Shapes& shapes() const { return s_; }
  const rs_ctx_options& options() const { return opt_; }
  Vit* vit() { return vit_.get(); }
  Llm* llm() { return llm_.get(); }
  cudaStream_t tracker_stream() const { return tracker_; }
  cudaStream_t aux_stream() const { return aux_; }
  Uploader& uploader() { return up_; }

  // ---- device tracker data plane ----
  /// Slot pages, bitmap (text bits set), KV pages + table, M-RoPE ids, and
  /// the K8 text gather (ids from host, or hashed on device when null).
  /// grids: merged-token grid per MM item (payload files, host/payload.hpp);
  /// null = the most square factorisation.
  DevRequest& create_request(const lmmsim::RequestSpec& req, const std::int32_t* text_ids,
                             std::uint64_t payload_seed, cudaStream_t st,
                             const std::vector<std::pair<int, int>>* grids = nullptr);
  /// Downstream pipeline stage: KV pages, page table and M-RoPE ids only
  /// (no embedding slot, no bitmap).
  DevRequest& create_kv_request(const lmmsim::RequestSpec& req, cudaStream_t st);
  DevRequest* find(lmmsim::RequestId id);
  DevRequest& get(lmmsim::RequestId id);
  /// K6: rows [n, d] (LLM order, items concatenated) -> slots; set bits.
  void scatter_items(DevRequest& r, const std::vector<lmmsim::TokenRange>& items,
                     const bf16* rows, cudaStream_t st);
  /// Frees slot pages whose tokens are all below `released_end`.
  void release_prefix(DevRequest& r, std::uint64_t released_end, cudaEvent_t guard);
  /// Frees the request's device state. keep_slot: its request / logits slot
  /// stays reserved until free_slot() (logits not yet read back).
  void erase_request(lmmsim::RequestId id, cudaEvent_t guard, bool keep_slot = false);
  void free_slot(int slot) { free_slots_.push_back(slot); }
  /// After a device-wide synchronize: forget page guard events (their
  /// owners — e.g. an engine run's backend — may be destroyed next).
  void quiesce() {
    slab_pages_.clear_guards();
    kv_pages_.clear_guards();
  }
  /// K7 on the device: schedulable count from `frontier` (synchronous).
  std::uint64_t device_schedulable(DevRequest& r, std::uint64_t frontier);

  // ---- compute ----
  /// Builds + uploads the batch plan, runs the ViT; out = [tokens, d].
  VitBatchPlan plan_batch(const DevRequest& r, const std::vector<lmmsim::TokenRange>& items) const;
  void encode(const VitBatchPlan& plan, const bf16* patches_dev, bf16* out, cudaStream_t st);
  /// One chunk through the local layers. x: [M, d] residual (per chunk).
  /// Greedy decode after the first token, batched over
  /// `ids` (requests kept alive after their prefill, rs_run_options.keep_kv):
  /// each step embeds the previous argmax, runs all layers for one row per
  /// request against its paged KV (appending the new K/V), LM head + argmax.
  /// out_tokens [steps][n]; out_logits optional [steps][n][vocab] (host);
  /// returns the device milliseconds of the decode loop.
  double decode(const std::vector<lmmsim::RequestId>& ids, int steps, std::int32_t* out_tokens,
                float* out_logits, cudaStream_t st);
  /// Frees a request kept for decode (KV pages, tables, request slot).
  void free_kept(lmmsim::RequestId id);
  // ---- TP group across GPUs ----
  /// This rank's exchange buffer and its CUDA IPC handle.
  void tp_buffer(void** dev, cudaIpcMemHandle_t* handle);
  /// Maps every rank's exchange buffer: ptrs[r] (same process) or handles[r] (IPC).
  void tp_connect(const void* const* ptrs, const cudaIpcMemHandle_t* handles);
  // ---- PD (prefill -> decode) KV transfer ----
  /// Bytes of a kept request's KV image: [shard][layer][page][K | V^T page].
  std::uint64_t kv_image_bytes(std::uint64_t tokens) const;
  /// Packs a kept request's KV pages (+ its first token) into `dst` (device,
  /// >= kv_image_bytes + kKvImageHeader) on `st`; fills the host metadata.
  void export_kv(lmmsim::RequestId id, void* dst, std::uint64_t cap, rs_kv_meta* meta, cudaStream_t st);
  /// Creates kept request `id` from an image exported by a context with the
  /// same LLM (layers, kv heads, TP): KV pages unpacked, first token into its
  /// argmax slot; rs_decode continues it.
  void import_kv(lmmsim::RequestId id, const rs_kv_meta& meta, const void* src, cudaStream_t st);
  void prefill(const std::vector<SliceRef>& slices, bf16* x, cudaStream_t st,
               int layer_from = -1, int layer_to = -1);
  std::uint64_t chunk_flops(const std::vector<SliceRef>& slices) const;

  bf16* slab() { return slab_; }
  const std::int32_t* argmax_host(int slot);
  void copy_logits(int slot, float* host, cudaStream_t st);
  std::int32_t* device_argmax() { return llm_ ? llm_->argmax_dev() : nullptr; }
  int max_requests() const { return max_requests_; }
  cudaEvent_t new_event();  // owned by the context

 private:
  int take_request_slot();
  void attach_kv(const lmmsim::RequestSpec& req, DevRequest& r, cudaStream_t st);
  Shapes s_;
  rs_ctx_options opt_;
  DeviceArena arena_;
  std::unique_ptr<Vit> vit_;
  std::unique_ptr<Llm> llm_;
  bf16* slab_ = nullptr;
  PagePool slab_pages_, kv_pages_;
  int** page_tables_dev_ = nullptr;   // [max_requests] -> kv page table
  // tensor parallelism: shards 1..T-1 of the LLM (shard 0 is
  // llm_), their O / down partials and the reduction's sums of squares
  std::vector<std::unique_ptr<Llm>> tp_shards_;
  // TP group rank (f4 across GPUs): exchange buffer (partials x 2 phases +
  // flag slots), every rank's mapping of it, reduction epoch
  bool tp_group_ = false, tp_connected_ = false;
  void* tpx_ = nullptr;
  std::size_t tpx_bytes_ = 0;
  std::vector<void*> tpx_peers_;
  std::vector<bool> tpx_opened_;
  unsigned tp_epoch_ = 0;
  std::vector<bf16*> tp_parts_;
  bf16** tp_parts_dev_ = nullptr;
  unsigned long long* tp_ss_ = nullptr;
  void run_llm(const ChunkDev& c, const bf16* slab, bf16* x, cudaStream_t st, int l_from, int l_to);
  bf16* decode_x_ = nullptr;          // decode: [n, d] residual of the step
  std::int32_t* decode_ids_ = nullptr;
  int decode_x_cap_ = 0;
  std::vector<int*> page_tables_host_;
  std::vector<int> free_slots_;
  int max_requests_ = 0;
  std::unordered_map<lmmsim::RequestId, std::unique_ptr<DevRequest>> reqs_;
  cudaStream_t tracker_ = nullptr, aux_ = nullptr;
  Uploader up_;
  std::vector<cudaEvent_t> events_;
  std::uint64_t* prefix_dev_ = nullptr;
  std::uint64_t* prefix_host_ = nullptr;
};

}  // namespace rserve
