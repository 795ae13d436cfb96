// rserve-b200 — EP entry points of the C-ABI (include/rserve.h, "EP disaggregation").
#include <cstring>
#include <exception>
#include <memory>
#include <thread>

#include "capi_ctx.cuh"
#include "device_backend.cuh"
#include "ep.cuh"
#include "host/config_bridge.hpp"
#include "host/decision_log.hpp"
#include "host/status.hpp"
#include "lmmsim/metrics.hpp"
#include "lmmsim/workload.hpp"

using namespace rserve;

struct rs_ep {
  ep::Topology topo;
  int transport = 0;
  int rank = 0;
  std::unique_ptr<ep::LoopbackHub> hub;                    // loopback
  std::vector<std::unique_ptr<ep::Transport>> endpoints;   // loopback: one per rank; NCCL: this rank
  std::vector<lmmsim::RequestSpec> workload;               // worker_prepare
  std::unique_ptr<ep::EncoderWorker> encoder;              // NCCL worker state
  std::unique_ptr<ep::StageWorker> stage;
  rs_ctx* worker_ctx = nullptr;
};

namespace {
rs_ep& need_ep(rs_ep* e) {
  if (e == nullptr) throw lmmsim::InputError("null rs_ep");
  return *e;
}

/// The worker role of `rank` on context `ctx` (encoder or downstream stage).
void run_worker(rs_ep& e, ep::Transport& t, int rank, rs_ctx& ctx,
                const std::vector<lmmsim::RequestSpec>& workload, std::uint64_t seed, bool e2e) {
  if (e.topo.is_encoder(rank)) {
    ep::EncoderWorker w(*ctx.ctx, t, e.topo);
    w.prepare(workload, seed, e2e);
    w.run();
  } else {
    ep::StageWorker w(*ctx.ctx, t, e.topo, rank);
    w.run();
  }
}
}  // namespace

extern "C" {

rs_status rs_ep_links(int32_t stages, int32_t encoders, int32_t* n_links, int32_t* pairs) {
  return guarded([&] {
    ep::Topology topo{stages, encoders};
    topo.validate();
    const auto links = topo.links();
    if (n_links) *n_links = static_cast<int32_t>(links.size());
    if (pairs)
      for (std::size_t i = 0; i < links.size(); ++i) {
        pairs[2 * i] = links[i].first;
        pairs[2 * i + 1] = links[i].second;
      }
  });
}

rs_status rs_nccl_unique_id(void* out128) {
  return guarded([&] { ep::nccl_unique_id(out128); });
}

rs_status rs_ep_create(const rs_ep_options* opt, rs_ep** out) {
  return guarded([&] {
    if (opt == nullptr || out == nullptr) throw lmmsim::InputError("rs_ep_create: null argument");
    auto e = std::make_unique<rs_ep>();
    e->topo = ep::Topology{opt->stages, opt->encoders};
    e->topo.validate();
    e->transport = opt->transport;
    e->rank = opt->rank;
    if (opt->transport == 0) {
      e->hub = std::make_unique<ep::LoopbackHub>(e->topo.world());
      for (int r = 0; r < e->topo.world(); ++r)
        e->endpoints.push_back(ep::make_loopback(*e->hub, r, opt->device));
    } else if (opt->transport == 1) {
      if (opt->nccl_ids == nullptr) throw lmmsim::InputError("rs_ep_create: NCCL needs nccl_ids");
      if (opt->rank < 0 || opt->rank >= e->topo.world())
        throw lmmsim::ConfigError("ep.rank: outside [0, world)");
      e->endpoints.push_back(ep::make_nccl(e->topo, opt->rank, opt->device, opt->nccl_ids));
    } else if (opt->transport == 2) {
      if (opt->shm_name == nullptr || opt->slot_bytes == 0)
        throw lmmsim::InputError("rs_ep_create: IPC needs shm_name and slot_bytes");
      if (opt->rank < 0 || opt->rank >= e->topo.world())
        throw lmmsim::ConfigError("ep.rank: outside [0, world)");
      e->endpoints.push_back(ep::make_ipc(e->topo, opt->rank, opt->device, opt->slot_bytes, opt->shm_name));
    } else {
      throw lmmsim::ConfigError("ep.transport: 0 (loopback), 1 (NCCL) or 2 (CUDA IPC)");
    }
    *out = e.release();
  });
}

rs_status rs_ep_destroy(rs_ep* e) {
  return guarded([&] { delete e; });
}

rs_status rs_ep_ipc_export(rs_ep* e, void* out, uint64_t capacity, uint64_t* size) {
  return guarded([&] {
    rs_ep& x = need_ep(e);
    const std::vector<char> blob = ep::ipc_export(*x.endpoints.at(0));
    if (size) *size = blob.size();
    if (out != nullptr) {
      if (capacity < blob.size()) throw lmmsim::InputError("rs_ep_ipc_export: buffer too small");
      std::memcpy(out, blob.data(), blob.size());
    }
  });
}

rs_status rs_ep_ipc_connect(rs_ep* e, const void* blobs, const uint64_t* sizes, int32_t n) {
  return guarded([&] {
    rs_ep& x = need_ep(e);
    std::vector<std::vector<char>> all;
    const char* p = static_cast<const char*>(blobs);
    for (int32_t i = 0; i < n; ++i) {
      all.emplace_back(p, p + sizes[i]);
      p += sizes[i];
    }
    ep::ipc_connect(*x.endpoints.at(0), all);
  });
}

rs_status rs_ep_worker_prepare(rs_ep* e, rs_ctx* c, const char* workload_text, uint64_t seed, int32_t e2e) {
  return guarded([&] {
    rs_ep& x = need_ep(e);
    rs_ctx& ctx = need(c);
    if (x.transport == 0) throw lmmsim::ConfigError("rs_ep_worker_prepare: multi-process transports only");
    if (x.rank == 0) throw lmmsim::ConfigError("rs_ep_worker_prepare: rank 0 runs the engine");
    x.stage.reset();
    x.encoder.reset();
    if (x.topo.is_encoder(x.rank)) {
      x.encoder = std::make_unique<ep::EncoderWorker>(*ctx.ctx, *x.endpoints[0], x.topo);
      x.encoder->prepare(parse_workload_text(workload_text), seed, e2e != 0);
    } else {
      x.stage = std::make_unique<ep::StageWorker>(*ctx.ctx, *x.endpoints[0], x.topo, x.rank);
    }
    x.worker_ctx = c;
  });
}

rs_status rs_ep_worker_run(rs_ep* e, rs_ctx* c) {
  return guarded([&] {
    rs_ep& x = need_ep(e);
    if (c != x.worker_ctx) throw lmmsim::InputError("rs_ep_worker_run: context differs from prepare");
    if (x.encoder) x.encoder->run();
    else if (x.stage) x.stage->run();
    else throw lmmsim::ConfigError("rs_ep_worker_run: call rs_ep_worker_prepare first");
  });
}

}  // extern "C"

namespace {
struct EngineOutputs {
  lmmsim::SimResult res;
  std::vector<ReleaseRecord> releases;
  std::string journal;
  rs_run_stats stats{};
};

/// One engine run on the device: co-located on `c0` (ep == nullptr) or EP
/// with `c0` as P0 (loopback worker ranks run on threads of this call).
EngineOutputs run_engine(rs_ctx& c0, rs_ep* ep, rs_ctx* const* workers, std::vector<lmmsim::RequestSpec> wl,
                         lmmsim::SimConfig sc, const rs_run_options* opt) {
  sc.hidden_size = static_cast<std::uint32_t>(c0.ctx->shapes().d);
  const bool realtime = opt != nullptr && opt->clock == 1;
  const bool e2e = opt != nullptr && opt->e2e != 0;
  const bool serialize = opt != nullptr && opt->serialize != 0;
  const std::uint64_t seed = opt ? opt->payload_seed : 0;
  if (ep != nullptr && opt != nullptr && opt->payload_text != nullptr)
    throw lmmsim::ConfigError("payload files: co-located engine runs only (EP encoder ranks derive "
                              "pixels and grids from the layout)");
  EngineOutputs out;
  auto finish = [&](DeviceBackend& backend, lmmsim::PipelineEngine& engine) {
    backend.collect();
    for (const auto& [id, row] : backend.logits()) c0.logits[id] = row;
    for (const auto& [id, am] : backend.argmax()) c0.argmax[id] = am;
    for (const lmmsim::ReleaseEvent& ev : engine.releases()) out.releases.push_back({ev.chunk, ev.id, ev.range});
    out.journal = render_journal(engine.journal());
    out.stats = backend.stats();
  };
  if (ep == nullptr) {
    DeviceBackend backend(*c0.ctx, sc, realtime, e2e, seed, serialize);
    if (opt != nullptr && opt->payload_text != nullptr) {
      PayloadSpec spec = parse_payload(opt->payload_text);
      validate_payload(spec, wl, c0.ctx->shapes().vocab);
      backend.set_payload(std::move(spec));
    }
    backend.prepare(wl);
    lmmsim::PipelineEngine engine(wl, sc, backend);
    backend.start();
    out.res = engine.run();
    finish(backend, engine);
    return out;
  }
  rs_ep& x = *ep;
  if (x.transport != 0 && x.rank != 0) throw lmmsim::ConfigError("EP engine run: rank 0 only");
  // Loopback: worker ranks are threads of this call.
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errors(static_cast<std::size_t>(x.topo.world()));
  if (x.transport == 0) {
    if (workers == nullptr) throw lmmsim::InputError("EP engine run: loopback needs worker contexts");
    for (int r = 1; r < x.topo.world(); ++r) {
      rs_ctx& wc = need(workers[r - 1]);
      threads.emplace_back([&x, &wc, &wl, &errors, r, seed, e2e] {
        try {
          run_worker(x, *x.endpoints[static_cast<std::size_t>(r)], r, wc, wl, seed, e2e);
        } catch (...) {
          errors[static_cast<std::size_t>(r)] = std::current_exception();
        }
      });
    }
  }
  ep::Transport& t = *x.endpoints[0];
  ep::Remote remote{&t, x.topo};
  try {
    DeviceBackend backend(*c0.ctx, sc, realtime, e2e, seed, serialize, &remote);
    backend.prepare(wl);
    lmmsim::PipelineEngine engine(wl, sc, backend);
    backend.start();
    out.res = engine.run();
    ep::stop_workers(t, x.topo);
    for (auto& th : threads) th.join();
    threads.clear();
    finish(backend, engine);
  } catch (...) {
    if (!threads.empty()) {  // unblock the worker threads before propagating
      try {
        ep::stop_workers(t, x.topo);
      } catch (...) {
      }
      for (auto& th : threads) th.join();
    }
    throw;
  }
  for (auto& err : errors)
    if (err) std::rethrow_exception(err);
  return out;
}
}  // namespace

extern "C" {

rs_status rs_ep_engine_run(rs_ep* e, rs_ctx* p0, rs_ctx* const* workers, const char* workload_text,
                           const rs_sim_config* cfg, const rs_run_options* opt, char** out_result,
                           char** out_journal, rs_run_stats* out_stats) {
  return guarded([&] {
    rs_ep& x = need_ep(e);
    EngineOutputs o = run_engine(need(p0), &x, workers, parse_workload_text(workload_text), to_sim_config(*cfg), opt);
    if (out_result) *out_result = c_string(render_decision_log(o.res, o.releases, true));
    if (out_journal) *out_journal = c_string(o.journal);
    if (out_stats) *out_stats = o.stats;
  });
}

rs_status rs_engine_cell(rs_ctx* ctx, rs_ep* ep, rs_ctx* const* workers, const rs_workload_config* wcfg,
                         const rs_sim_config* cfg, double slo_ttft_ms, const rs_run_options* opt,
                         char** out_csv_row, char** out_trace_json, rs_run_stats* out_stats) {
  return guarded([&] {
    if (wcfg == nullptr || cfg == nullptr) throw lmmsim::InputError("rs_engine_cell: null config");
    const lmmsim::SimConfig sc = to_sim_config(*cfg);
    EngineOutputs o = run_engine(need(ctx), ep, workers, lmmsim::generate_workload(to_workload_config(*wcfg)), sc, opt);
    std::optional<double> slo;
    if (slo_ttft_ms >= 0) slo = slo_ttft_ms;
    const lmmsim::MetricsReport rep = lmmsim::compute_report(o.res, slo);
    if (out_csv_row)
      *out_csv_row = c_string(lmmsim::report_csv_row(lmmsim::to_string(sc.policy), wcfg->arrival_rate, wcfg->seed, rep));
    if (out_trace_json) *out_trace_json = c_string(lmmsim::trace_to_json_text(o.res));
    if (out_stats) *out_stats = o.stats;
  });
}

rs_status rs_ep_ctrl_pack(const char* text, void* out_msg, uint64_t msg_bytes) {
  return guarded([&] {
    if (text == nullptr || out_msg == nullptr) throw lmmsim::InputError("rs_ep_ctrl_pack: null argument");
    if (msg_bytes != ep::kCtrlBytes)
      throw lmmsim::InputError("rs_ep_ctrl_pack: message buffer must be " + std::to_string(ep::kCtrlBytes) + " bytes");
    const ep::Words w = ep::from_text(text);
    std::memcpy(out_msg, w.data(), ep::kCtrlBytes);
  });
}

rs_status rs_ep_ctrl_unpack(const void* msg, uint64_t msg_bytes, char** out_text) {
  return guarded([&] {
    if (msg == nullptr || out_text == nullptr) throw lmmsim::InputError("rs_ep_ctrl_unpack: null argument");
    if (msg_bytes != ep::kCtrlBytes)
      throw lmmsim::DataError("rs_ep_ctrl_unpack: message must be " + std::to_string(ep::kCtrlBytes) + " bytes");
    ep::Words w(ep::kCtrlWords);
    std::memcpy(w.data(), msg, ep::kCtrlBytes);
    *out_text = c_string(ep::to_text(w));
  });
}

}  // extern "C"
