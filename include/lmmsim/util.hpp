// rserve-b200 — number formatting / parsing shared by messages and reports.
//
// Error messages and CSV rows must be byte-identical to the reference's, so
// doubles are printed in shortest round-trip form via std::to_chars, exactly
// the convention of the reference (proj/include/lmmsim/util.hpp:30-40).
#pragma once

#include <charconv>
#include <cstdint>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "lmmsim/errors.hpp"

namespace lmmsim {

namespace detail {
template <typename T>
inline std::string to_chars_string(T v) {
  char buf[64];
  const std::to_chars_result r = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, static_cast<std::size_t>(r.ptr - buf));
}

template <typename T>
inline T from_chars_exact(std::string_view s, const std::string& what,
                          const char* kind) {
  T v{};
  const char* first = s.data();
  const char* last = first + s.size();
  const std::from_chars_result r = std::from_chars(first, last, v);
  if (r.ec != std::errc{} || r.ptr != last)
    throw InputError(what + ": not " + kind + ": '" + std::string(s) + "'");
  return v;
}
}  // namespace detail

/// Shortest decimal text that parses back to exactly `v`.
inline std::string format_double(double v) { return detail::to_chars_string(v); }
inline std::string format_u64(std::uint64_t v) { return detail::to_chars_string(v); }

inline double parse_double(std::string_view s, const std::string& what) {
  return detail::from_chars_exact<double>(s, what, "a number");
}
inline std::uint64_t parse_u64(std::string_view s, const std::string& what) {
  return detail::from_chars_exact<std::uint64_t>(s, what,
                                                 "an unsigned integer");
}

/// Splits on `sep`, keeping empty fields (n separators -> n+1 fields).
inline std::vector<std::string_view> split(std::string_view s, char sep) {
  std::vector<std::string_view> fields;
  std::string_view rest = s;
  for (;;) {
    const std::size_t cut = rest.find(sep);
    fields.push_back(rest.substr(0, cut));
    if (cut == std::string_view::npos) break;
    rest.remove_prefix(cut + 1);
  }
  return fields;
}

}  // namespace lmmsim
