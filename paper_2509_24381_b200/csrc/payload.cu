// rserve-b200 — request payload files (host code; see host/payload.hpp).
#include <algorithm>
#include <sstream>
#include <tuple>

#include "host/payload.hpp"
#include "kernels.cuh"
#include "lmmsim/errors.hpp"
#include "lmmsim/util.hpp"
#include "host/config_bridge.hpp"
#include "host/status.hpp"
#include "rserve.h"

namespace rserve {

void default_item_grid(std::uint64_t tokens, int* gh, int* gw) {
  std::uint64_t best = 1;
  for (std::uint64_t h = 1; h * h <= tokens; ++h)
    if (tokens % h == 0) best = h;
  *gh = static_cast<int>(best);
  *gw = static_cast<int>(tokens / best);
}

namespace {

std::string trim(const std::string& s) {
  std::size_t a = 0, b = s.size();
  while (a < b && (s[a] == ' ' || s[a] == '\t' || s[a] == '\r')) ++a;
  while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
  return s.substr(a, b - a);
}

std::vector<std::string> split_on(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  out.push_back(cur);
  return out;
}

std::uint64_t parse_u64_field(const std::string& v, const std::string& where) {
  return lmmsim::parse_u64(trim(v), where);
}

}  // namespace

PayloadSpec parse_payload(const std::string& text) {
  PayloadSpec spec;
  std::istringstream is(text);
  std::string line;
  std::size_t lineno = 0;
  while (std::getline(is, line)) {
    ++lineno;
    const std::string t = trim(line);
    if (t.empty() || t[0] == '#') continue;
    const std::string where = "payload line " + lmmsim::format_u64(lineno);
    const auto f = split_on(t, ',');
    if (f.size() != 4) throw lmmsim::InputError(where + ": expected 4 comma-separated fields");
    const lmmsim::RequestId id = parse_u64_field(f[0], where + " request id");
    const std::size_t seg = static_cast<std::size_t>(parse_u64_field(f[1], where + " segment index"));
    const std::string kind = trim(f[2]);
    RequestPayload& rp = spec[id];
    if (kind == "M") {
      if (rp.items.count(seg)) throw lmmsim::InputError(where + ": duplicate segment " + f[1]);
      ItemPayload ip;
      for (const std::string& kv : split_on(f[3], ';')) {
        const auto p = kv.find('=');
        if (p == std::string::npos) throw lmmsim::InputError(where + ": expected key=value, got '" + kv + "'");
        const std::string k = trim(kv.substr(0, p)), v = trim(kv.substr(p + 1));
        if (k == "grid") {
          const auto x = v.find('x');
          if (x == std::string::npos) throw lmmsim::InputError(where + ": grid must be <gh>x<gw>");
          ip.gh = static_cast<int>(parse_u64_field(v.substr(0, x), where + " grid"));
          ip.gw = static_cast<int>(parse_u64_field(v.substr(x + 1), where + " grid"));
          if (ip.gh <= 0 || ip.gw <= 0) throw lmmsim::InputError(where + ": grid must be positive");
        } else if (k == "seed") {
          ip.has_seed = true;
          ip.seed = parse_u64_field(v, where + " seed");
        } else {
          throw lmmsim::InputError(where + ": unknown multimodal key '" + k + "'");
        }
      }
      rp.items[seg] = ip;
    } else if (kind == "T") {
      if (rp.texts.count(seg)) throw lmmsim::InputError(where + ": duplicate segment " + f[1]);
      TextPayload tp;
      const auto p = f[3].find('=');
      if (p == std::string::npos) throw lmmsim::InputError(where + ": expected seed=<u64> or ids=<list>");
      const std::string k = trim(f[3].substr(0, p)), v = trim(f[3].substr(p + 1));
      if (k == "seed") {
        tp.has_seed = true;
        tp.seed = parse_u64_field(v, where + " seed");
      } else if (k == "ids") {
        std::istringstream vs(v);
        std::string tok;
        while (vs >> tok) {
          const std::uint64_t x = parse_u64_field(tok, where + " token id");
          if (x > 0x7FFFFFFFull) throw lmmsim::InputError(where + ": token id " + tok + " out of range");
          tp.ids.push_back(static_cast<std::int32_t>(x));
        }
        if (tp.ids.empty()) throw lmmsim::InputError(where + ": empty id list");
      } else {
        throw lmmsim::InputError(where + ": unknown text key '" + k + "'");
      }
      rp.texts[seg] = tp;
    } else {
      throw lmmsim::InputError(where + ": segment kind must be T or M, got '" + kind + "'");
    }
  }
  return spec;
}

std::string format_payload(const PayloadSpec& spec) {
  std::vector<lmmsim::RequestId> ids;
  for (const auto& kv : spec) ids.push_back(kv.first);
  std::sort(ids.begin(), ids.end());
  std::ostringstream os;
  os << "# rserve payload v1\n";
  for (lmmsim::RequestId id : ids) {
    const RequestPayload& rp = spec.at(id);
    std::map<std::size_t, std::string> lines;
    for (const auto& [seg, ip] : rp.items) {
      std::string s = lmmsim::format_u64(id) + "," + lmmsim::format_u64(seg) + ",M,";
      std::string kv;
      if (ip.gh > 0) kv += "grid=" + std::to_string(ip.gh) + "x" + std::to_string(ip.gw);
      if (ip.has_seed) kv += (kv.empty() ? "" : ";") + std::string("seed=") + lmmsim::format_u64(ip.seed);
      lines[seg] = s + kv;
    }
    for (const auto& [seg, tp] : rp.texts) {
      std::string s = lmmsim::format_u64(id) + "," + lmmsim::format_u64(seg) + ",T,";
      if (!tp.ids.empty()) {
        s += "ids=";
        for (std::size_t i = 0; i < tp.ids.size(); ++i) s += (i ? " " : "") + std::to_string(tp.ids[i]);
      } else {
        s += "seed=" + lmmsim::format_u64(tp.seed);
      }
      lines[seg] = s;
    }
    for (const auto& [seg, s] : lines) os << s << '\n';
  }
  return os.str();
}

void validate_payload(const PayloadSpec& spec, const std::vector<lmmsim::RequestSpec>& workload,
                      int vocab) {
  std::unordered_map<lmmsim::RequestId, const lmmsim::RequestSpec*> by_id;
  for (const auto& r : workload) by_id[r.id] = &r;
  for (const auto& [id, rp] : spec) {
    const auto it = by_id.find(id);
    const std::string who = "payload: request " + lmmsim::format_u64(id);
    if (it == by_id.end()) throw lmmsim::InputError(who + " is not in the workload");
    const auto& segs = it->second->segments;
    for (const auto& [seg, ip] : rp.items) {
      if (seg >= segs.size() || segs[seg].kind != lmmsim::SegmentKind::Multimodal)
        throw lmmsim::InputError(who + " segment " + lmmsim::format_u64(seg) + " is not multimodal");
      if (ip.gh > 0 && static_cast<std::uint64_t>(ip.gh) * static_cast<std::uint64_t>(ip.gw) != segs[seg].tokens)
        throw lmmsim::InputError(who + " segment " + lmmsim::format_u64(seg) + ": grid " +
                                 std::to_string(ip.gh) + "x" + std::to_string(ip.gw) + " != " +
                                 lmmsim::format_u64(segs[seg].tokens) + " tokens");
    }
    for (const auto& [seg, tp] : rp.texts) {
      if (seg >= segs.size() || segs[seg].kind != lmmsim::SegmentKind::Text)
        throw lmmsim::InputError(who + " segment " + lmmsim::format_u64(seg) + " is not text");
      if (!tp.ids.empty()) {
        if (tp.ids.size() != segs[seg].tokens)
          throw lmmsim::InputError(who + " segment " + lmmsim::format_u64(seg) + ": " +
                                   std::to_string(tp.ids.size()) + " ids for " +
                                   lmmsim::format_u64(segs[seg].tokens) + " tokens");
        for (std::int32_t x : tp.ids)
          if (x < 0 || x >= vocab)
            throw lmmsim::InputError(who + " segment " + lmmsim::format_u64(seg) + ": token id " +
                                     std::to_string(x) + " outside the vocabulary");
      }
    }
  }
}

PayloadSpec generate_payload(const std::vector<lmmsim::RequestSpec>& workload, std::uint64_t seed) {
  PayloadSpec spec;
  for (const auto& r : workload) {
    RequestPayload& rp = spec[r.id];
    for (std::size_t s = 0; s < r.segments.size(); ++s) {
      const auto& seg = r.segments[s];
      const std::uint64_t h = mix64(seed, (7ull << 32) | r.id, s);
      if (seg.kind == lmmsim::SegmentKind::Multimodal) {
        std::vector<std::pair<int, int>> grids;
        for (std::uint64_t a = 1; a * a <= seg.tokens; ++a) {
          if (seg.tokens % a != 0) continue;
          const std::uint64_t b = seg.tokens / a;
          if (b > 4 * a) continue;
          grids.emplace_back(static_cast<int>(a), static_cast<int>(b));
          if (a != b) grids.emplace_back(static_cast<int>(b), static_cast<int>(a));
        }
        ItemPayload ip;
        if (grids.empty()) default_item_grid(seg.tokens, &ip.gh, &ip.gw);
        else std::tie(ip.gh, ip.gw) = grids[h % grids.size()];
        ip.has_seed = true;
        ip.seed = mix64(h, 1, 0);
        rp.items[s] = ip;
      } else {
        TextPayload tp;
        tp.has_seed = true;
        tp.seed = mix64(h, 2, 0);
        rp.texts[s] = tp;
      }
    }
  }
  return spec;
}

ResolvedPayload resolve_payload(const lmmsim::RequestSpec& req, const RequestPayload* p,
                                std::uint64_t run_seed, int vocab) {
  ResolvedPayload out;
  std::uint64_t pos = 0;
  for (std::size_t s = 0; s < req.segments.size(); ++s) {
    const auto& seg = req.segments[s];
    if (seg.kind == lmmsim::SegmentKind::Multimodal) {
      int gh = 0, gw = 0;
      std::uint64_t pseed = run_seed;
      if (p != nullptr) {
        const auto it = p->items.find(s);
        if (it != p->items.end()) {
          gh = it->second.gh;
          gw = it->second.gw;
          if (it->second.has_seed) pseed = it->second.seed;
        }
      }
      if (gh == 0) default_item_grid(seg.tokens, &gh, &gw);
      out.item_grids.emplace_back(gh, gw);
      out.item_seeds.push_back(pseed);
    } else {
      const TextPayload* tp = nullptr;
      if (p != nullptr) {
        const auto it = p->texts.find(s);
        if (it != p->texts.end()) tp = &it->second;
      }
      for (std::uint64_t i = 0; i < seg.tokens; ++i) {
        std::int32_t id;
        if (tp != nullptr && !tp->ids.empty()) {
          id = tp->ids[i];
        } else {
          const std::uint64_t sd = tp != nullptr ? tp->seed : run_seed;
          id = static_cast<std::int32_t>(mix64(sd, (6ull << 32) | req.id, pos + i) %
                                         static_cast<std::uint64_t>(vocab));
        }
        out.text_ids.push_back(id);
      }
    }
    pos += seg.tokens;
  }
  return out;
}

}  // namespace rserve

using namespace rserve;

extern "C" {

RS_API rs_status rs_payload_generate(const char* workload_text, uint64_t seed, char** out_text) {
  return guarded([&] {
    const std::string t = format_payload(generate_payload(parse_workload_text(workload_text), seed));
    *out_text = c_string(t);
  });
}

RS_API rs_status rs_payload_validate(const char* workload_text, const char* payload_text, int32_t vocab,
                                     char** out_normalized) {
  return guarded([&] {
    const PayloadSpec spec = parse_payload(payload_text ? payload_text : "");
    validate_payload(spec, parse_workload_text(workload_text), vocab);
    if (out_normalized) *out_normalized = c_string(format_payload(spec));
  });
}

}  // extern "C"
