// Byte-stable number formatting / strict parsing.
// Semantics follow the reference's text_format.cpp:27-82.
#include "dreamsched/text_format.hpp"

#include <cctype>
#include <charconv>
#include <cmath>
#include <system_error>

#include "dreamsched/errors.hpp"

namespace dreamsched {

std::string format_real(double value) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, value);
  std::string s(buf, res.ptr);
  const bool typed = s.find_first_of(".e") != std::string::npos ||
                     s.find("inf") != std::string::npos || s.find("nan") != std::string::npos;
  return typed ? s : s + ".0";
}

namespace {
[[noreturn]] void bad_field(std::string_view what, std::string_view text) {
  throw ParseError("invalid " + std::string(what) + ": '" + std::string(text) + "'");
}
}  // namespace

std::uint64_t parse_u64_field(std::string_view text, std::string_view what) {
  text = trim(text);
  std::uint64_t v = 0;
  const char* end = text.data() + text.size();
  const auto res = std::from_chars(text.data(), end, v);
  if (res.ec != std::errc() || res.ptr != end) bad_field(what, text);
  return v;
}

double parse_real_field(std::string_view text, std::string_view what) {
  text = trim(text);
  double v = 0.0;
  const char* end = text.data() + text.size();
  const auto res = std::from_chars(text.data(), end, v);
  if (res.ec != std::errc() || res.ptr != end || !std::isfinite(v)) bad_field(what, text);
  return v;
}

std::vector<std::string_view> split(std::string_view line, char sep) {
  std::vector<std::string_view> out;
  for (;;) {
    const auto cut = line.find(sep);
    out.push_back(line.substr(0, cut));
    if (cut == std::string_view::npos) return out;
    line.remove_prefix(cut + 1);
  }
}

std::string_view trim(std::string_view text) {
  auto is_space = [](char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; };
  std::size_t b = 0, e = text.size();
  while (b < e && is_space(text[b])) ++b;
  while (e > b && is_space(text[e - 1])) --e;
  return text.substr(b, e - b);
}

}  // namespace dreamsched
