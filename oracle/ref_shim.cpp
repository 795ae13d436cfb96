// ORACLE — test infrastructure only (never linked into the product).
//
// C-ABI over the UNMODIFIED reference headers (/root/reference/proj/include,
// built by oracle/Makefile into oracle/_ref/liblmmsim_ref.so). Used by
// tests/ (ctypes) and by bench.py's reference arm to obtain the reference's
// own answers on identical inputs:
//   ref_generate_workload  -> generate_workload   (workload.hpp:139-172)
//   ref_simulate           -> run_simulation      (simengine.hpp:522-526)
//   ref_experiment_cell    -> run_cell semantics  (experiment.hpp:72-101)
//   ref_plan_batches       -> plan_batches        (encoder_sched.hpp:48-74)
//   ref_replay             -> drives create_tracker / plan_batches /
//                             EncoderQueue / build_microbatch /
//                             on_embeddings_ready / release in the order of a
//                             journal recorded by the B200 engine (real-clock
//                             runs), emitting the same decision log.
//   ref_time_simulate      -> wall time of run_simulation (CPU baseline).
// The decision-log text format is defined in DESIGN.md ("Decision log") and
// emitted independently by the product (paper_2509_24381_b200/csrc/host/
// decision_log.hpp); equal text means bit-identical decisions and times.

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "lmmsim/cost_model.hpp"
#include "lmmsim/encoder_sched.hpp"
#include "lmmsim/simengine.hpp"
#include "lmmsim/token_sched.hpp"
#include "lmmsim/tracker.hpp"
#include "lmmsim/workload.hpp"

// Only the POD config structs of the boundary header.
#include "../include/rserve.h"

#define REF_API __attribute__((visibility("default")))

using namespace lmmsim;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ConfigError*>(&e)) return RS_ERR_CONFIG;
  if (dynamic_cast<const RegistryError*>(&e)) return RS_ERR_REGISTRY;
  if (dynamic_cast<const DoubleEncodeError*>(&e)) return RS_ERR_DOUBLE_ENCODE;
  if (dynamic_cast<const AlignmentError*>(&e)) return RS_ERR_ALIGNMENT;
  if (dynamic_cast<const DependencyViolation*>(&e)) return RS_ERR_DEPENDENCY_VIOLATION;
  if (dynamic_cast<const InputError*>(&e)) return RS_ERR_INPUT;
  if (dynamic_cast<const InternalError*>(&e)) return RS_ERR_INTERNAL;
  if (dynamic_cast<const SimError*>(&e)) return RS_ERR_SIM;
  return RS_ERR_UNKNOWN;
}

SimConfig to_sim(const rs_sim_config& c) {
  SimConfig s;
  s.policy = static_cast<Policy>(c.policy);
  if (c.pipeline_mode == RS_PIPELINE_CPP) s.pipeline_mode = PipelineMode::Cpp;
  if (c.pipeline_mode == RS_PIPELINE_VANILLA) s.pipeline_mode = PipelineMode::Vanilla;
  s.stages = c.stages;
  s.encoder_workers = c.encoder_workers;
  s.token_budget = c.token_budget;
  s.embedding_batch_tokens = c.embedding_batch_tokens;
  s.release_at = c.release_at == RS_RELEASE_FIRST_STAGE ? ReleaseAt::FirstStage
                                                        : ReleaseAt::LastStage;
  s.hidden_size = c.hidden_size;
  s.cost.alpha_enc_ms = c.cost.alpha_enc_ms;
  s.cost.beta_enc_ms_per_token = c.cost.beta_enc_ms_per_token;
  s.cost.eps_tx_ms = c.cost.eps_tx_ms;
  s.cost.zeta_tx_ms_per_token = c.cost.zeta_tx_ms_per_token;
  s.cost.gamma_stage_ms = c.cost.gamma_stage_ms;
  s.cost.delta_stage_ms_per_token = c.cost.delta_stage_ms_per_token;
  s.cost.kappa_attn_ms = c.cost.kappa_attn_ms;
  s.cost.tp_speedup = c.cost.tp_speedup;
  return s;
}

IntDistribution to_dist(const rs_int_dist& d) {
  return d.uniform ? IntDistribution::uniform(d.lo, d.hi)
                   : IntDistribution::constant(d.lo);
}

WorkloadConfig to_wcfg(const rs_workload_config& w) {
  WorkloadConfig out;
  out.arrival_rate = w.arrival_rate;
  out.duration_s = w.duration_s;
  out.seed = w.seed;
  for (int i = 0; i < w.n_templates; ++i) {
    const rs_template& t = w.templates[i];
    RequestTemplate rt;
    rt.pattern = static_cast<LayoutPattern>(t.pattern);
    rt.num_mm_items = to_dist(t.num_mm_items);
    rt.mm_item_tokens = to_dist(t.mm_item_tokens);
    rt.text_segment_tokens = to_dist(t.text_segment_tokens);
    out.template_mix.emplace_back(rt, t.probability);
  }
  if (w.has_slo) out.slo_ttft_ms = w.slo_ttft_ms;
  return out;
}

std::vector<RequestSpec> parse_workload(const char* text) {
  std::istringstream is(text ? text : "");
  return read_workload(is);
}

const char* kind_name(TraceKind k) {
  return k == TraceKind::Encode ? "encode" : k == TraceKind::Transfer ? "transfer" : "stage";
}

std::string d(double v) { return format_double(v); }
std::string u(std::uint64_t v) { return format_u64(v); }

// Canonical decision log. `with_times` = false
// drops every time/duration field (real-clock replay compares decisions
// only).
std::string render(const SimResult& r, const std::vector<std::string>& releases,
                   bool with_times) {
  std::string o;
  o += "result chunks=" + u(r.chunk_count) + " encode_batches=" +
       u(r.encode_batch_count) + " transfers=" + u(r.transfer_count);
  if (with_times)
    o += " first_arrival=" + d(r.first_arrival_ms) + " last_completion=" +
         d(r.last_completion_ms);
  o += "\n";
  for (const RequestRecord& q : r.requests) {
    o += "req id=" + u(q.id) + " prompt=" + u(q.prompt_tokens) +
         " completed=" + u(q.completed ? 1 : 0) + " released=" +
         u(q.released_tokens) + " peak_live=" + u(q.peak_live_tokens);
    if (with_times)
      o += " arrival=" + d(q.arrival_ms) + " first_token=" + d(q.first_token_ms) +
           " first_admission=" + d(q.first_admission_ms) + " encode_dispatch=" +
           d(q.encode_dispatch_ms) + " embeddings_ready=" +
           d(q.embeddings_ready_ms) + " ttft=" + d(q.ttft_ms) + " queue=" +
           d(q.queue_delay_ms) + " encode_span=" + d(q.encode_span_ms) +
           " prefill_span=" + d(q.prefill_span_ms);
    o += "\n";
    for (const auto& [chunk, range] : q.slices)
      o += "slice req=" + u(q.id) + " chunk=" + u(chunk) + " start=" +
           u(range.start) + " end=" + u(range.end) + "\n";
  }
  for (const TraceEvent& e : r.trace) {
    o += std::string("trace kind=") + kind_name(e.kind) + " res=" +
         std::to_string(e.resource) + " name=" + e.name + " owners=";
    for (std::size_t i = 0; i < e.owners.size(); ++i) o += (i ? "," : "") + u(e.owners[i]);
    o += " tokens=" + u(e.tokens);
    if (with_times) o += " start=" + d(e.start_ms) + " dur=" + d(e.dur_ms);
    o += "\n";
  }
  for (const std::string& rel : releases) o += rel + "\n";
  return o;
}

// Release order is not part of SimResult; derive it exactly as the
// reference emits it: chunk completion order, slices in chunk order. For a
// cost-model run we reconstruct it from the trace (the last stage's events
// are in completion order because the pipeline is FIFO per stage).
std::vector<std::string> releases_from(const SimResult& r, int stages, bool first_stage) {
  std::map<std::size_t, std::vector<std::pair<RequestId, TokenRange>>> by_chunk;
  for (const RequestRecord& q : r.requests)
    for (const auto& [chunk, range] : q.slices) by_chunk[chunk].push_back({q.id, range});
  // slices within a chunk are in queue order; the trace owners give it.
  std::map<std::size_t, std::vector<RequestId>> owners;
  std::vector<std::size_t> order;
  const int wanted = first_stage ? 0 : stages - 1;
  for (const TraceEvent& e : r.trace) {
    if (e.kind != TraceKind::Stage || e.resource != kStageResourceBase + wanted) continue;
    std::size_t chunk = std::stoull(e.name.substr(5, e.name.find('_') - 5));
    order.push_back(chunk);
    owners[chunk] = e.owners;
  }
  std::vector<std::string> out;
  for (std::size_t chunk : order) {
    auto slices = by_chunk[chunk];
    const auto& own = owners[chunk];
    for (std::size_t i = 0; i < own.size(); ++i) {
      for (const auto& [id, range] : slices)
        if (id == own[i]) {
          out.push_back("release chunk=" + u(chunk) + " req=" + u(id) + " start=" +
                        u(range.start) + " end=" + u(range.end));
          break;
        }
    }
  }
  return out;
}

}  // namespace

extern "C" {

REF_API const char* ref_last_error(void) { return g_err.c_str(); }
REF_API void ref_free(void* p) { std::free(p); }

REF_API int ref_generate_workload(const rs_workload_config* w, char** out) {
  try {
    std::ostringstream os;
    write_workload(os, generate_workload(to_wcfg(*w)));
    *out = dup(os.str());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_API int ref_simulate(const char* workload, const rs_sim_config* cfg, char** out) {
  try {
    const SimConfig sc = to_sim(*cfg);
    const SimResult r = run_simulation(parse_workload(workload), sc);
    *out = dup(render(r, releases_from(r, sc.stages, sc.release_at == ReleaseAt::FirstStage), true));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Wall-clock of run_simulation over `reps` repetitions (ns per run).
REF_API int ref_time_simulate(const char* workload, const rs_sim_config* cfg, int reps,
                      double* ns_per_run) {
  try {
    const SimConfig sc = to_sim(*cfg);
    const std::vector<RequestSpec> wl = parse_workload(workload);
    std::size_t sink = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) sink += run_simulation(wl, sc).chunk_count;
    const auto t1 = std::chrono::steady_clock::now();
    *ns_per_run = std::chrono::duration<double, std::nano>(t1 - t0).count() / reps +
                  (sink == 0xFFFFFFFFFFFFull ? 1 : 0);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_API int ref_experiment_cell(const rs_workload_config* w, const rs_sim_config* cfg,
                        double slo, char** out) {
  try {
    const SimConfig sc = to_sim(*cfg);
    const SimResult r = run_simulation(generate_workload(to_wcfg(*w)), sc);
    std::optional<double> s;
    if (slo >= 0) s = slo;
    // metrics.hpp pulls nlohmann; the report row is assembled here from the
    // reference's nearest_rank with the metrics.hpp:49-86 definitions.
    std::vector<double> t;
    double sum = 0;
    TokenCount tok = 0;
    std::size_t with = 0, met = 0;
    for (const auto& q : r.requests) {
      t.push_back(q.ttft_ms);
      sum += q.ttft_ms;
      tok += q.prompt_tokens;
      const std::optional<double> dl = q.slo_ttft_ms ? q.slo_ttft_ms : s;
      if (dl) {
        ++with;
        if (q.ttft_ms <= *dl) ++met;
      }
    }
    std::sort(t.begin(), t.end());
    std::string row = std::string(to_string(sc.policy)) + "," + d(w->arrival_rate) + "," + u(w->seed) + ",";
    if (r.empty()) {
      row += "0,0,0,0,0,";
    } else {
      const double ms = r.makespan_ms();
      row += d(sum / static_cast<double>(r.requests.size())) + "," + d(nearest_rank(t, 50)) + "," +
             d(nearest_rank(t, 90)) + "," + d(nearest_rank(t, 99)) + "," +
             d(ms > 0 ? static_cast<double>(tok) / (ms / 1000.0) : 0) + ",";
      if (with) row += d(static_cast<double>(met) / static_cast<double>(with));
    }
    *out = dup(row);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_API int ref_plan_batches(const char* layout, std::uint64_t id, std::uint64_t c, char** out) {
  try {
    RequestSpec r;
    r.id = id;
    r.segments = parse_layout(layout);
    std::string o;
    for (const EncodeBatch& b : plan_batches(r, c)) {
      o += u(b.request_id);
      for (const auto& [idx, range] : b.items)
        o += " " + u(idx) + ":" + u(range.start) + "-" + u(range.end);
      o += " total=" + u(b.total_tokens) + "\n";
    }
    *out = dup(o);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Journal replay. Journal lines: "<kind> <a> <b> <time>" with kind
// 0 arrival(b = request index in (arrival,id) order), 1 encode done
// (a = worker, b = slot), 2 transfer done (b = slot), 3 stage done
// (a = stage, b = chunk), 4 chunk complete (b = chunk). The handlers below
// are the reference engine's (simengine.hpp:275-441) written over the
// reference components; only the ORDER comes from the journal. Output:
// decision log without times.
REF_API int ref_replay(const char* workload, const rs_sim_config* cfg, const char* journal,
               char** out) {
  try {
    const SimConfig sc = to_sim(*cfg);
    sc.validate();
    const PolicyTraits traits = select_policy(sc.policy);
    const PipelineMode mode = sc.effective_mode();
    std::vector<RequestSpec> reqs = parse_workload(workload);
    std::sort(reqs.begin(), reqs.end(), [](const RequestSpec& a, const RequestSpec& b) {
      return a.arrival_ms != b.arrival_ms ? a.arrival_ms < b.arrival_ms : a.id < b.id;
    });
    std::map<RequestId, RequestRecord> rec;
    for (const auto& q : reqs) {
      rec[q.id].id = q.id;
      rec[q.id].prompt_tokens = q.total_tokens();
    }
    TrackerRegistry reg;
    SchedulerQueues queues;
    EncoderQueue encq;
    std::vector<EncodeBatch> batches;
    std::vector<bool> enc_busy(static_cast<std::size_t>(sc.encoder_workers), false);
    struct St { bool busy = false; std::deque<std::size_t> pending; };
    std::vector<St> st(static_cast<std::size_t>(sc.stages));
    struct Ch { std::vector<std::pair<RequestId, TokenRange>> slices; TokenCount tokens = 0; bool released = false; };
    std::vector<Ch> chunks;
    std::size_t in_flight = 0, completed = 0;
    SimResult res;
    std::vector<std::string> releases;

    auto stage_trace = [&](int s, std::size_t c) {
      TraceEvent ev;
      ev.kind = TraceKind::Stage;
      ev.resource = kStageResourceBase + s;
      ev.name = "chunk" + u(c) + "_s" + u(static_cast<std::uint64_t>(s));
      for (const auto& sl : chunks[c].slices) ev.owners.push_back(sl.first);
      ev.tokens = chunks[c].tokens;
      res.trace.push_back(ev);
      st[static_cast<std::size_t>(s)].busy = true;
    };
    auto dispatch = [&]() {
      for (std::size_t w = 0; w < enc_busy.size(); ++w) {
        if (enc_busy[w]) continue;
        auto b = encq.next_dispatch(true, 0);
        if (!b) return;
        const std::size_t slot = batches.size();
        TraceEvent ev;
        ev.kind = TraceKind::Encode;
        ev.resource = kEncoderResourceBase + static_cast<int>(w);
        ev.name = "encode_r" + u(b->request_id) + "_b" + u(slot);
        ev.owners = {b->request_id};
        ev.tokens = b->total_tokens;
        res.trace.push_back(ev);
        ++res.encode_batch_count;
        enc_busy[w] = true;
        batches.push_back(std::move(*b));
      }
    };
    auto release_chunk = [&](std::size_t c) {
      if (chunks[c].released) throw InternalError("double release");
      chunks[c].released = true;
      for (const auto& [id, range] : chunks[c].slices) {
        EmbeddingTracker& t = reg.get(id);
        t.release(range);
        releases.push_back("release chunk=" + u(c) + " req=" + u(id) + " start=" +
                           u(range.start) + " end=" + u(range.end));
        rec[id].released_tokens += range.length();
        if (t.fully_prefilled() && t.fully_released()) {
          rec[id].peak_live_tokens = t.peak_live_embedding_tokens();
          reg.erase(id);
        }
      }
    };
    auto try_schedule = [&]() {
      if (queues.waiting.empty()) return;
      const bool admit = mode == PipelineMode::Vanilla ? in_flight == 0 : !st[0].busy;
      if (!admit) return;
      auto mb = build_microbatch(queues, reg, sc.token_budget, traits, 0);
      if (!mb) return;
      const std::size_t c = chunks.size();
      chunks.push_back({mb->slices, mb->total_tokens, false});
      for (const auto& [id, range] : mb->slices) rec[id].slices.emplace_back(c, range);
      ++in_flight;
      stage_trace(0, c);
    };

    // Journal lines "<kind> <a> <b> <time>" parsed without iostream numeric
    // facets (this .so may carry its own static C++ runtime).
    std::vector<std::string_view> lines = split(journal ? journal : "", '\n');
    for (std::string_view line : lines) {
      if (line.empty()) continue;
      const std::vector<std::string_view> f = split(line, ' ');
      if (f.size() != 4) throw InputError("journal: bad line '" + std::string(line) + "'");
      const int kind = static_cast<int>(parse_u64(f[0], "journal kind"));
      const std::uint32_t a = static_cast<std::uint32_t>(parse_u64(f[1], "journal a"));
      const std::uint64_t b = parse_u64(f[2], "journal b");
      switch (kind) {
        case 0: {
          const RequestSpec& q = reqs.at(b);
          create_tracker(reg, q, sc.hidden_size);
          encq.enqueue_request(plan_batches(q, traits.whole_request_encode ? kWholeRequest : sc.embedding_batch_tokens));
          queues.waiting.push_back(q.id);
          dispatch();
          try_schedule();
          break;
        }
        case 1: {
          enc_busy.at(a) = false;
          TraceEvent ev;
          ev.kind = TraceKind::Transfer;
          ev.resource = kTransferResource;
          ev.name = "transfer_r" + u(batches.at(b).request_id) + "_b" + u(b);
          ev.owners = {batches[b].request_id};
          ev.tokens = batches[b].total_tokens;
          res.trace.push_back(ev);
          ++res.transfer_count;
          dispatch();
          break;
        }
        case 2: {
          for (const auto& [idx, range] : batches.at(b).items)
            on_embeddings_ready(reg, batches[b].request_id, range);
          try_schedule();
          break;
        }
        case 3: {
          St& s = st.at(a);
          s.busy = false;
          if (static_cast<int>(a) + 1 < sc.stages) {
            St& nx = st[a + 1];
            if (!nx.busy) stage_trace(static_cast<int>(a) + 1, b);
            else nx.pending.push_back(b);
          }
          if (sc.release_at == ReleaseAt::FirstStage && a == 0) release_chunk(b);
          if (!s.busy && !s.pending.empty()) {
            const std::size_t nc = s.pending.front();
            s.pending.pop_front();
            stage_trace(static_cast<int>(a), nc);
          }
          try_schedule();
          break;
        }
        case 4: {
          if (sc.release_at == ReleaseAt::LastStage) release_chunk(b);
          for (const auto& [id, range] : chunks.at(b).slices)
            if (range.end == rec[id].prompt_tokens) {
              rec[id].completed = true;
              ++completed;
            }
          --in_flight;
          try_schedule();
          break;
        }
        default:
          throw InputError("journal: bad event kind");
      }
    }
    for (auto& [id, r] : rec) res.requests.push_back(r);
    res.chunk_count = chunks.size();
    *out = dup(render(res, releases, false));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
