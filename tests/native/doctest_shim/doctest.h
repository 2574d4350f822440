// doctest.h — a minimal doctest-compatible test shim (test infrastructure).
//
// The reference's unit suite (/root/reference/proj/tests/unit/*.cpp) is
// written against doctest, which is not vendored there (proj/vendor/ is
// missing) and cannot be fetched here.  This header implements exactly the
// subset those files use — TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, FAIL, doctest::Approx(...).epsilon/scale and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the suite compiles unchanged
// against both the reference library (oracle/_ref, pins the shim) and this
// repository's libdreamsched (the drop-in claim).
//
// Runner flags (doctest's spelling): -tc=/-tce= test-case name include /
// exclude, -sf=/-sfe= source-file include / exclude (comma-separated globs
// with '*'), -ltc lists the test cases.  Exit status 0 iff every case passed.
#ifndef DREAMDDP_DOCTEST_SHIM_H_
#define DREAMDDP_DOCTEST_SHIM_H_

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double value) : value_(value) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  // |lhs - value| < epsilon * (scale + max(|lhs|, |value|)): doctest's rule
  bool matches(double lhs) const {
    return std::fabs(lhs - value_) < epsilon_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
  }
  friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }
  friend bool operator!=(const Approx& a, double rhs) { return !a.matches(rhs); }
  friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || a.matches(lhs); }
  friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || a.matches(lhs); }
  friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && !a.matches(lhs); }
  friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && !a.matches(lhs); }

 private:
  double value_;
  double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
  double scale_ = 1.0;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> cases;
  return cases;
}

struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct AbortCase {};  // thrown by REQUIRE / FAIL to end the current case

struct Counters {
  long long asserts = 0, failed_asserts = 0;
  bool case_failed = false;
  const TestCase* current = nullptr;
};

inline Counters& counters() {
  static Counters c;
  return c;
}

inline void record(bool ok, const char* file, int line, const char* what) {
  Counters& c = counters();
  ++c.asserts;
  if (ok) return;
  ++c.failed_asserts;
  c.case_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\"): %s\n", file, line,
               c.current ? c.current->name : "?", what);
}

// '*' globs, comma-separated alternatives
inline bool glob(const char* p, const char* s) {
  if (*p == '\0') return *s == '\0';
  if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
  return *s && *p == *s && glob(p + 1, s + 1);
}

inline bool any_glob(const std::string& list, const char* s) {
  size_t start = 0;
  while (start <= list.size()) {
    const size_t end = std::min(list.find(',', start), list.size());
    if (glob(list.substr(start, end - start).c_str(), s)) return true;
    start = end + 1;
  }
  return false;
}

inline int run(int argc, char** argv) {
  std::string tc, tce, sf, sfe;
  bool list = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&](const char* key) { return a.rfind(key, 0) == 0 ? a.substr(std::strlen(key)) : std::string(); };
    if (a == "-ltc" || a == "--list-test-cases") list = true;
    else if (a.rfind("-tc=", 0) == 0) tc = val("-tc=");
    else if (a.rfind("-tce=", 0) == 0) tce = val("-tce=");
    else if (a.rfind("-sf=", 0) == 0) sf = val("-sf=");
    else if (a.rfind("-sfe=", 0) == 0) sfe = val("-sfe=");
  }
  int run_n = 0, failed = 0, skipped = 0;
  for (const TestCase& t : registry()) {
    if ((!tc.empty() && !any_glob(tc, t.name)) || (!tce.empty() && any_glob(tce, t.name)) ||
        (!sf.empty() && !any_glob(sf, t.file)) || (!sfe.empty() && any_glob(sfe, t.file))) {
      ++skipped;
      continue;
    }
    if (list) {
      std::printf("%s\t%s:%d\n", t.name, t.file, t.line);
      continue;
    }
    Counters& c = counters();
    c.case_failed = false;
    c.current = &t;
    try {
      t.fn();
    } catch (const AbortCase&) {
      c.case_failed = true;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\"): uncaught exception: %s\n", t.file, t.line,
                   t.name, e.what());
      c.case_failed = true;
    } catch (...) {
      std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\"): uncaught non-std exception\n", t.file, t.line,
                   t.name);
      c.case_failed = true;
    }
    ++run_n;
    if (c.case_failed) ++failed;
  }
  if (list) return 0;
  const Counters& c = counters();
  std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n", run_n, run_n - failed,
              failed, skipped);
  std::printf("[doctest-shim] assertions: %lld | %lld passed | %lld failed\n", c.asserts,
              c.asserts - c.failed_asserts, c.failed_asserts);
  return failed == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                              \
  static void fn();                                                                              \
  static const ::doctest::detail::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                                       &fn);                     \
  static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define DOCTEST_SHIM_ASSERT(abort, text, ...)                                 \
  do {                                                                        \
    bool doctest_ok_ = false;                                                 \
    try {                                                                     \
      doctest_ok_ = static_cast<bool>(__VA_ARGS__);                           \
    } catch (...) {                                                           \
      doctest_ok_ = false;                                                    \
    }                                                                         \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, text);         \
    if (!doctest_ok_ && (abort)) throw ::doctest::detail::AbortCase{};        \
  } while (0)

#define CHECK(...) DOCTEST_SHIM_ASSERT(false, "CHECK(" #__VA_ARGS__ ")", __VA_ARGS__)
#define REQUIRE(...) DOCTEST_SHIM_ASSERT(true, "REQUIRE(" #__VA_ARGS__ ")", __VA_ARGS__)

#define CHECK_THROWS_AS(expr, ...)                                                                   \
  do {                                                                                               \
    bool doctest_ok_ = false;                                                                        \
    try {                                                                                            \
      static_cast<void>(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                                   \
      doctest_ok_ = true;                                                                            \
    } catch (...) {                                                                                  \
    }                                                                                                \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")"); \
  } while (0)

#define CHECK_NOTHROW(...)                                                                  \
  do {                                                                                      \
    bool doctest_ok_ = true;                                                                \
    try {                                                                                   \
      static_cast<void>(__VA_ARGS__);                                                       \
    } catch (...) {                                                                         \
      doctest_ok_ = false;                                                                  \
    }                                                                                       \
    ::doctest::detail::record(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW(" #__VA_ARGS__ ")"); \
  } while (0)

#define FAIL(msg)                                                                   \
  do {                                                                              \
    ::doctest::detail::record(false, __FILE__, __LINE__, "FAIL: " msg);             \
    throw ::doctest::detail::AbortCase{};                                           \
  } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run(argc, argv); }
#endif

#endif  // DREAMDDP_DOCTEST_SHIM_H_
