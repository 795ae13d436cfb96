// rserve-b200 — the B200 ExecutionBackend of the pipeline engine.
//
// Receives every decision of lmmsim::PipelineEngine (the reference's event
// handlers, simengine.hpp:275-441) and turns it into device work on one GPU:
//   launch_encode      -> ViT forward of the Algorithm-1 batch on an encoder
//                         stream (encode_time_ms seam, cost_model.hpp:68-71)
//   launch_transfer    -> co-located: nothing to move (0-cost link, the
//                         reference's eps = zeta = 0 case, cost_model.hpp:84-88)
//   on_embeddings_ready-> K6 scatter + bitmap on the tracker stream
//                         (mark_encoded, tracker.hpp:83-105)
//   launch_stage       -> LLM layers of the stage over the micro-batch
//                         (stage_time_ms seam, cost_model.hpp:76-82)
//   on_release / erase -> slot pages back to the pool, guarded by the CUDA
//                         event of the chunk that read them (tracker.hpp:126-135)
// Lock-step mode returns cost-model durations (event order = reference);
// real-clock mode is `deferred`: completions come from CUDA events, stamped
// with GPU time relative to the run's origin event.
#pragma once

#include <chrono>
#include <cstdint>
#include <unordered_map>
#include <vector>

#include "device_context.cuh"
#include "ep.cuh"
#include "host/payload.hpp"
#include "lmmsim/simengine.hpp"

namespace rserve {

/// Synthetic request payloads (pixels, text ids) prepared before a timed run.
struct Payload {
  bf16* patches_dev = nullptr;   // [patches, pdim] (resident mode)
  bf16* patches_host = nullptr;  // pinned (e2e mode)
  std::uint64_t patches = 0;
};

class DeviceBackend final : public lmmsim::ExecutionBackend {
 public:
  /// remote != nullptr: EP mode — this is P0; encoders and stages >= 1 are
  /// other ranks reached through remote->t (see ep.cuh).
  DeviceBackend(Context& ctx, const lmmsim::SimConfig& cfg, bool realtime, bool e2e,
                std::uint64_t payload_seed, bool serialize = false,
                const ep::Remote* remote = nullptr);
  ~DeviceBackend() override;

  /// Payload file overrides (grids, pixel seeds, token ids); before prepare().
  void set_payload(PayloadSpec spec) { payload_ = std::move(spec); }
  /// Keep completed requests' KV pages and request slots for decode (f3).
  void set_keep_kv(bool on) { keep_kv_ = on; }
  const std::vector<lmmsim::RequestId>& kept() const { return kept_; }
  /// Generates pixel payloads of `workload` (device or pinned host). Untimed.
  void prepare(const std::vector<lmmsim::RequestSpec>& workload);
  /// Starts the clock: records the origin event.
  void start();

  bool deferred() const override { return realtime_; }
  void on_request_created(const lmmsim::RequestSpec& req, const lmmsim::EmbeddingTracker&) override;
  double launch_encode(int worker, std::size_t slot, const lmmsim::EncodeBatch& b) override;
  double launch_transfer(int worker, std::size_t slot, const lmmsim::EncodeBatch& b) override;
  void on_embeddings_ready(std::size_t slot, const lmmsim::EncodeBatch& b) override;
  double launch_stage(int stage, const lmmsim::ChunkView& c) override;
  void on_release(std::size_t chunk, lmmsim::RequestId id, lmmsim::TokenRange r) override;
  void on_request_erased(lmmsim::RequestId id) override;
  void on_request_complete(lmmsim::RequestId id, std::size_t chunk) override;
  void poll(std::vector<lmmsim::OpCompletion>& out) override;
  lmmsim::TimeMs clock_ms() override;
  void idle_wait() override {}
  void finish() override;
  /// After the timed region: copies logits / argmax of completed requests
  /// to host and returns their request slots to the context.
  void collect();

  rs_run_stats stats() const { return stats_; }
  void note_call(int kind, double ms);
  /// Logits / argmax of completed requests (host copies after finish()).
  const std::unordered_map<lmmsim::RequestId, std::vector<float>>& logits() const { return logits_; }
  const std::unordered_map<lmmsim::RequestId, std::int32_t>& argmax() const { return argmax_; }

 private:
  struct Op {
    lmmsim::OpKind kind;
    std::uint32_t a;
    std::uint64_t b;
    cudaEvent_t begin, end;
  };
  struct ChunkState {
    bf16* x = nullptr;
    int buf = -1;
    cudaEvent_t last = nullptr;  // completion of the latest stage launched
    cudaEvent_t s0_end = nullptr;  // stage 0 (the only reader of the slab rows)
  };
  /// EP: an op whose completion is the arrival of one or more messages.
  struct RemoteOp {
    lmmsim::OpKind kind;
    std::uint32_t a;
    std::uint64_t b;
    std::vector<std::shared_ptr<ep::Xfer>> xfers;
    bool launched;  // engine has started it (completions before that are held)
  };
  void* put_ctrl(const ep::Words& w);
  void launch_remote_encode(int worker, std::size_t slot, const lmmsim::EncodeBatch& b);
  void forward_chunk(const lmmsim::ChunkView& c, const ChunkState& cs);
  bool remote_done(RemoteOp& op);
  cudaEvent_t timing_event();
  void track(lmmsim::OpKind k, std::uint32_t a, std::uint64_t b, cudaEvent_t begin, cudaEvent_t end);
  int stage_of_layer_split(int s, int* lb, int* le) const;

  Context& ctx_;
  lmmsim::SimConfig cfg_;
  bool realtime_, e2e_;
  std::uint64_t seed_;
  std::vector<cudaStream_t> enc_streams_;
  bool shared_streams_ = false;
  std::vector<cudaStream_t> stage_streams_;
  cudaStream_t copy_stream_ = nullptr;
  cudaEvent_t origin_ = nullptr;
  cudaEvent_t tracker_tail_ = nullptr;  // latest scatter / creation on the tracker stream
  std::chrono::steady_clock::time_point t0_;
  std::unordered_map<lmmsim::RequestId, Payload> payloads_;
  // encode staging: ring per worker
  static constexpr int kRing = 4;       // initial staging buffers per encoder worker (pool grows)
  std::vector<bf16*> staging_;          // [>= workers * kRing] x [max_encode_tokens, d]
  std::vector<cudaEvent_t> staging_free_;
  std::vector<bool> staging_busy_;      // held by a batch not yet scattered
  std::size_t staging_next_ = 0;
  int acquire_staging();
  std::vector<bf16*> enc_input_;        // [workers] patches input (e2e)
  std::unordered_map<std::size_t, int> slot_staging_;     // encode slot -> staging index
  std::unordered_map<std::size_t, cudaEvent_t> slot_done_; // encode slot -> completion
  std::unordered_map<std::size_t, double> slot_done_ms_;
  std::vector<std::pair<std::size_t, double>> ready_transfers_;
  // chunks
  std::vector<bf16*> xbufs_;
  std::vector<cudaEvent_t> xbuf_guard_;
  std::vector<int> free_xbufs_;
  std::unordered_map<std::size_t, ChunkState> chunks_;
  cudaEvent_t release_guard_ = nullptr;
  std::vector<Op> ops_;
  std::vector<cudaEvent_t> event_pool_;
  std::unordered_map<lmmsim::RequestId, float*> logits_host_;
  std::unordered_map<lmmsim::RequestId, int> done_slots_;
  std::unordered_map<lmmsim::RequestId, std::vector<float>> logits_;
  std::unordered_map<lmmsim::RequestId, std::int32_t> argmax_;
  std::vector<int> deferred_slot_free_;
  rs_run_stats stats_{};
  std::uint64_t launches0_ = 0, upload0_ = 0;
  cudaEvent_t last_event_ = nullptr;
  cudaEvent_t last_encode_end_ = nullptr;  // RS_ENCODE_FIRST experiment
  // EP (remote_ != nullptr)
  const ep::Remote* remote_ = nullptr;
  std::unordered_map<lmmsim::RequestId, std::vector<lmmsim::SegmentSpec>> layouts_;
  std::vector<RemoteOp> remote_ops_;
  std::unordered_map<std::size_t, std::shared_ptr<ep::Xfer>> slot_xfer_;
  // chunk -> its last logits arrival: the transfer itself is held (its event
  // goes back to the transport's pool, and is re-recorded, once released)
  std::unordered_map<std::size_t, std::shared_ptr<ep::Xfer>> chunk_logits_;
  static constexpr int kCtrlRing = 16;
  std::vector<void*> ctrl_dev_;
  std::vector<std::int64_t*> ctrl_host_;
  std::vector<cudaEvent_t> ctrl_free_;
  int ctrl_pos_ = 0;
  cudaStream_t ctrl_stream_ = nullptr;
  void* header_sink_ = nullptr;
  float* remote_logits_ = nullptr;  // [max_requests, vocab] when the LM head is remote
  double remote_last_ms_ = 0;
  double last_poll_ms_ = -1;  // host-side stall diagnostics (rs_run_stats)
  PayloadSpec payload_;
  bool keep_kv_ = false;
  std::vector<lmmsim::RequestId> kept_;
  std::unordered_map<lmmsim::RequestId, ResolvedPayload> resolved_;
};

}  // namespace rserve
