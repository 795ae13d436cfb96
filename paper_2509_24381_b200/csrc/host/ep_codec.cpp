// rserve-b200 — EP topology and control-message codec (see ep_codec.hpp).
#include "ep_codec.hpp"

#include <string_view>

#include "lmmsim/errors.hpp"
#include "lmmsim/util.hpp"

namespace rserve::ep {

using lmmsim::format_u64;
using lmmsim::parse_u64;

std::vector<std::pair<int, int>> Topology::links() const {
  std::vector<std::pair<int, int>> out;
  for (int w = 0; w < encoders; ++w) {
    out.emplace_back(p_rank(0), e_rank(w));
    out.emplace_back(e_rank(w), p_rank(0));
  }
  for (int s = 0; s + 1 < stages; ++s) out.emplace_back(p_rank(s), p_rank(s + 1));
  for (int s = 1; s < stages; ++s) out.emplace_back(p_rank(s), p_rank(0));
  return out;
}

int Topology::link_index(int src, int dst) const {
  const auto l = links();
  for (std::size_t i = 0; i < l.size(); ++i)
    if (l[i].first == src && l[i].second == dst) return static_cast<int>(i);
  return -1;
}

void Topology::validate() const {
  if (stages < 1) throw lmmsim::ConfigError("ep.stages: must be >= 1");
  if (encoders < 1) throw lmmsim::ConfigError("ep.encoders: must be >= 1 (EP needs encoder GPUs)");
}

namespace {
constexpr std::size_t kHead = 3;

void put_header(Words& w, Ctrl k) {
  w.assign(kCtrlWords, 0);
  w[0] = kMagic;
  w[1] = static_cast<std::int64_t>(k);
}

struct Writer {
  Words& w;
  std::size_t pos = kHead;
  void put(std::uint64_t v) {
    if (pos >= w.size())
      throw lmmsim::ConfigError("ep control message: more than " + format_u64(kCtrlWords) +
                                " words (too many slices / items in one message)");
    w[pos++] = static_cast<std::int64_t>(v);
  }
  void done() { w[2] = static_cast<std::int64_t>(pos - kHead); }
};

struct Reader {
  const Words& w;
  std::size_t pos = kHead;
  std::size_t end;
  explicit Reader(const Words& words) : w(words) {
    end = kHead + static_cast<std::size_t>(words[2]);
  }
  std::uint64_t get() {
    if (pos >= end) throw lmmsim::DataError("ep control message: truncated payload");
    return static_cast<std::uint64_t>(w[pos++]);
  }
  void finish() const {
    if (pos != end) throw lmmsim::DataError("ep control message: trailing payload words");
  }
};
}  // namespace

void pack(const EncodeCmd& c, Words& w) {
  if (c.items.empty()) throw lmmsim::DataError("ep ENCODE: batch without items");
  for (const EncodeItem& it : c.items)
    if (it.end <= it.start) throw lmmsim::DataError("ep ENCODE: empty item range");
  put_header(w, Ctrl::kEncode);
  Writer out{w};
  out.put(c.slot);
  out.put(c.request_id);
  out.put(c.items.size());
  for (const EncodeItem& it : c.items) {
    out.put(it.index);
    out.put(it.start);
    out.put(it.end);
    out.put(it.patch_offset);
  }
  out.done();
}

void pack(const StageCmd& c, Words& w) {
  if (c.slices.empty()) throw lmmsim::DataError("ep STAGE: chunk without slices");
  for (const SliceCmd& s : c.slices)
    if (s.end <= s.start || s.end > s.total()) throw lmmsim::DataError("ep STAGE: slice outside its request");
  put_header(w, Ctrl::kStage);
  Writer out{w};
  out.put(c.chunk_id);
  out.put(c.slices.size());
  for (const SliceCmd& s : c.slices) {
    out.put(s.request_id);
    out.put(s.start);
    out.put(s.end);
    out.put(s.segments.size());
    for (const lmmsim::SegmentSpec& seg : s.segments) {
      out.put(seg.kind == lmmsim::SegmentKind::Multimodal ? 1 : 0);
      out.put(seg.tokens);
    }
  }
  out.done();
}

void pack_stop(Words& w) {
  put_header(w, Ctrl::kStop);
  w[2] = 0;
}

Ctrl kind_of(const Words& w) {
  if (w.size() != kCtrlWords) throw lmmsim::DataError("ep control message: wrong size");
  if (w[0] != kMagic) throw lmmsim::DataError("ep control message: bad magic");
  if (w[1] < 0 || w[1] > 2) throw lmmsim::DataError("ep control message: unknown kind");
  if (w[2] < 0 || static_cast<std::size_t>(w[2]) > kCtrlWords - kHead)
    throw lmmsim::DataError("ep control message: bad payload length");
  return static_cast<Ctrl>(w[1]);
}

EncodeCmd unpack_encode(const Words& w) {
  if (kind_of(w) != Ctrl::kEncode) throw lmmsim::DataError("ep control message: not ENCODE");
  Reader in(w);
  EncodeCmd c;
  c.slot = in.get();
  c.request_id = in.get();
  const std::uint64_t n = in.get();
  for (std::uint64_t i = 0; i < n; ++i) {
    EncodeItem it;
    it.index = in.get();
    it.start = in.get();
    it.end = in.get();
    it.patch_offset = in.get();
    if (it.end <= it.start) throw lmmsim::DataError("ep ENCODE: empty item range");
    c.items.push_back(it);
  }
  in.finish();
  if (c.items.empty()) throw lmmsim::DataError("ep ENCODE: batch without items");
  return c;
}

StageCmd unpack_stage(const Words& w) {
  if (kind_of(w) != Ctrl::kStage) throw lmmsim::DataError("ep control message: not STAGE");
  Reader in(w);
  StageCmd c;
  c.chunk_id = in.get();
  const std::uint64_t n = in.get();
  for (std::uint64_t i = 0; i < n; ++i) {
    SliceCmd s;
    s.request_id = in.get();
    s.start = in.get();
    s.end = in.get();
    const std::uint64_t segs = in.get();
    for (std::uint64_t k = 0; k < segs; ++k) {
      lmmsim::SegmentSpec seg;
      seg.kind = in.get() != 0 ? lmmsim::SegmentKind::Multimodal : lmmsim::SegmentKind::Text;
      seg.tokens = in.get();
      s.segments.push_back(seg);
    }
    if (s.end <= s.start || s.end > s.total())
      throw lmmsim::DataError("ep STAGE: slice outside its request");
    c.slices.push_back(std::move(s));
  }
  in.finish();
  if (c.slices.empty()) throw lmmsim::DataError("ep STAGE: chunk without slices");
  return c;
}

std::string to_text(const Words& w) {
  switch (kind_of(w)) {
    case Ctrl::kStop:
      return "STOP";
    case Ctrl::kEncode: {
      const EncodeCmd c = unpack_encode(w);
      std::string t = "ENCODE slot=" + format_u64(c.slot) + " req=" + format_u64(c.request_id) + " items=";
      const char* sep = "";
      for (const EncodeItem& it : c.items) {
        t += sep + format_u64(it.index) + ":" + format_u64(it.start) + "-" + format_u64(it.end) + "@" +
             format_u64(it.patch_offset);
        sep = ",";
      }
      return t;
    }
    case Ctrl::kStage: {
      const StageCmd c = unpack_stage(w);
      std::string t = "STAGE chunk=" + format_u64(c.chunk_id) + " slices=";
      const char* sep = "";
      for (const SliceCmd& s : c.slices) {
        t += sep + format_u64(s.request_id) + ":" + format_u64(s.start) + "-" + format_u64(s.end) + "[" +
             lmmsim::format_layout(s.segments) + "]";
        sep = ",";
      }
      return t;
    }
  }
  throw lmmsim::InternalError("unreachable");
}

namespace {
std::string_view after(std::string_view field, std::string_view key) {
  if (field.substr(0, key.size()) != key)
    throw lmmsim::InputError("ep control text: expected '" + std::string(key) + "' in '" +
                             std::string(field) + "'");
  return field.substr(key.size());
}
std::pair<std::uint64_t, std::uint64_t> range_of(std::string_view s) {
  const auto f = lmmsim::split(s, '-');
  if (f.size() != 2) throw lmmsim::InputError("ep control text: bad range '" + std::string(s) + "'");
  return {parse_u64(f[0], "range start"), parse_u64(f[1], "range end")};
}
}  // namespace

Words from_text(const std::string& text) {
  const auto f = lmmsim::split(text, ' ');
  Words w;
  if (f[0] == "STOP" && f.size() == 1) {
    pack_stop(w);
    return w;
  }
  if (f[0] == "ENCODE" && f.size() == 4) {
    EncodeCmd c;
    c.slot = parse_u64(after(f[1], "slot="), "slot");
    c.request_id = parse_u64(after(f[2], "req="), "req");
    for (std::string_view item : lmmsim::split(after(f[3], "items="), ',')) {
      const auto colon = lmmsim::split(item, ':');
      if (colon.size() != 2) throw lmmsim::InputError("ep control text: bad item");
      const auto at = lmmsim::split(colon[1], '@');
      if (at.size() != 2) throw lmmsim::InputError("ep control text: bad item");
      const auto [b, e] = range_of(at[0]);
      c.items.push_back({parse_u64(colon[0], "item"), b, e, parse_u64(at[1], "patch offset")});
    }
    pack(c, w);
    return w;
  }
  if (f[0] == "STAGE" && f.size() == 3) {
    StageCmd c;
    c.chunk_id = parse_u64(after(f[1], "chunk="), "chunk");
    for (std::string_view sl : lmmsim::split(after(f[2], "slices="), ',')) {
      const std::size_t lb = sl.find('[');
      if (lb == std::string_view::npos || sl.back() != ']')
        throw lmmsim::InputError("ep control text: bad slice");
      const auto colon = lmmsim::split(sl.substr(0, lb), ':');
      if (colon.size() != 2) throw lmmsim::InputError("ep control text: bad slice");
      SliceCmd s;
      s.request_id = parse_u64(colon[0], "request");
      std::tie(s.start, s.end) = range_of(colon[1]);
      s.segments = lmmsim::parse_layout(sl.substr(lb + 1, sl.size() - lb - 2));
      c.slices.push_back(std::move(s));
    }
    pack(c, w);
    return w;
  }
  throw lmmsim::InputError("ep control text: unknown message '" + text + "'");
}

}  // namespace rserve::ep
