// line_reader.hpp — shared reader for the two "dreamsched-* v1" text formats
// (profile and schedule files, SPEC.md "file format" notes): a magic first
// line, then content lines where blank lines carry no meaning.  Tracks line
// numbers for error locations.  Internal to libdreamsched.
#ifndef DREAMSCHED_LINE_READER_HPP_
#define DREAMSCHED_LINE_READER_HPP_

#include <istream>
#include <string>
#include <string_view>
#include <vector>

#include "dreamsched/errors.hpp"
#include "dreamsched/text_format.hpp"

namespace dreamsched::detail {

class LineReader {
 public:
  LineReader(std::istream& in, std::string_view source) : in_(in), source_(source) {}

  // The magic line must read exactly `magic` (surrounding blanks allowed).
  void expect_magic(std::string_view magic) {
    std::string first;
    const bool got = static_cast<bool>(std::getline(in_, first));
    number_ = 1;
    if (!got || trim(first) != magic) {
      throw ParseError(source_ + ": first line must be '" + std::string(magic) + "'");
    }
  }

  // Next line verbatim (false at end of input).
  bool next_raw(std::string* line) {
    if (!std::getline(in_, *line)) return false;
    ++number_;
    return true;
  }

  // Next line that is not blank (false at end of input).
  bool next_content(std::string* line) {
    while (next_raw(line)) {
      if (!trim(*line).empty()) return true;
    }
    return false;
  }

  // "<source>:<line>" of the line last returned.
  std::string here() const { return source_ + ":" + std::to_string(number_); }
  const std::string& source() const { return source_; }

 private:
  std::istream& in_;
  std::string source_;
  int number_ = 0;
};

// Whitespace-separated words of a line.
inline std::vector<std::string_view> words(std::string_view line) {
  std::vector<std::string_view> out;
  std::size_t i = 0;
  while (i < line.size()) {
    while (i < line.size() && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r' || line[i] == '\n' ||
                               line[i] == '\v' || line[i] == '\f'))
      ++i;
    std::size_t j = i;
    while (j < line.size() && !(line[j] == ' ' || line[j] == '\t' || line[j] == '\r' || line[j] == '\n' ||
                                line[j] == '\v' || line[j] == '\f'))
      ++j;
    if (j > i) out.push_back(line.substr(i, j - i));
    i = j;
  }
  return out;
}

// `word` starts with `key`; returns the rest.
inline bool strip_prefix(std::string_view word, std::string_view key, std::string_view* rest) {
  if (word.substr(0, key.size()) != key) return false;
  *rest = word.substr(key.size());
  return true;
}

}  // namespace dreamsched::detail

#endif  // DREAMSCHED_LINE_READER_HPP_
