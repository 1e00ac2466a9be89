// oracle/shim/catch2/catch.hpp — the Catch2 v2 subset the reference's unit
// tests use (/root/reference/proj/tests/*.cpp), for the oracle/_ref build
// only: TEST_CASE, SECTION (each leaf section runs in its own pass of the
// test case, as Catch does), REQUIRE / REQUIRE_FALSE / REQUIRE_THROWS /
// REQUIRE_NOTHROW, CAPTURE, and Approx with margin()/epsilon()/scale()
// (Catch2 v2 semantics: default epsilon = 100 * FLT_EPSILON).
// A failed assertion aborts the current test case and is reported with its
// source location, expression text and captured values; the process exits
// non-zero when any test case failed.  Command line: optional test-name
// substrings or "[tag]" filters, like Catch's.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace Catch {

struct TestCase {
  std::string name, tags;
  std::function<void()> fn;
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, const char* tags, void (*fn)(), const char* file, int line) {
    registry().push_back({name, tags ? tags : "", fn, file, line});
  }
};

struct AssertionFailed {};

struct RunState {
  long long assertions = 0;
  // section scheduling: the run executes the target-th leaf section seen
  int section_seen = 0;
  int section_target = 0;
  bool section_ran = false;
  std::vector<std::string> captures;
};
inline RunState& state() {
  static RunState s;
  return s;
}

class Approx {
  double value_, epsilon_, margin_ = 0.0, scale_ = 0.0;

  static bool margin_cmp(double lhs, double rhs, double margin) {
    return (lhs + margin >= rhs) && (rhs + margin >= lhs);
  }

 public:
  explicit Approx(double v)
      : value_(v), epsilon_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool equals(double other) const {
    return margin_cmp(value_, other, margin_) ||
           margin_cmp(value_, other, epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
  }
  double value() const { return value_; }
  friend bool operator==(double a, const Approx& b) { return b.equals(a); }
  friend bool operator==(const Approx& a, double b) { return a.equals(b); }
  friend bool operator!=(double a, const Approx& b) { return !b.equals(a); }
  friend bool operator!=(const Approx& a, double b) { return !a.equals(b); }
  friend bool operator<=(double a, const Approx& b) { return a < b.value_ || b.equals(a); }
  friend bool operator>=(double a, const Approx& b) { return a > b.value_ || b.equals(a); }
  friend bool operator<=(const Approx& a, double b) { return a.value_ < b || a.equals(b); }
  friend bool operator>=(const Approx& a, double b) { return a.value_ > b || a.equals(b); }
};

inline void fail(const char* macro, const char* expr, const char* file, int line, const char* extra = "") {
  std::fprintf(stderr, "%s:%d: FAILED:\n  %s( %s )%s\n", file, line, macro, expr, extra);
  for (const auto& c : state().captures) std::fprintf(stderr, "  with: %s\n", c.c_str());
  throw AssertionFailed{};
}

struct CaptureGuard {
  std::size_t n;
  template <typename... T>
  CaptureGuard(const char* names, const T&... vals) {
    std::ostringstream os;
    os.precision(17);
    os << names << " :=";
    ((os << ' ' << vals), ...);
    state().captures.push_back(os.str());
    n = state().captures.size();
  }
  ~CaptureGuard() {
    if (state().captures.size() >= n) state().captures.resize(n - 1);
  }
};

// A SECTION body runs only in its scheduled pass.
struct SectionGuard {
  bool active;
  explicit SectionGuard(const char*) {
    RunState& s = state();
    active = (s.section_seen == s.section_target);
    ++s.section_seen;
    if (active) s.section_ran = true;
  }
  explicit operator bool() const { return active; }
};

inline bool tag_match(const TestCase& t, const std::vector<std::string>& filters) {
  if (filters.empty()) return true;
  for (const auto& f : filters) {
    if (!f.empty() && f[0] == '[') {
      if (t.tags.find(f) != std::string::npos) return true;
    } else if (t.name.find(f) != std::string::npos) {
      return true;
    }
  }
  return false;
}

inline int run_all(int argc, char** argv) {
  std::vector<std::string> filters;
  for (int i = 1; i < argc; ++i) filters.emplace_back(argv[i]);
  int ran = 0, failed = 0;
  for (const auto& t : registry()) {
    if (!tag_match(t, filters)) continue;
    ++ran;
    bool ok = true;
    for (int target = 0;; ++target) {
      RunState& s = state();
      s.section_seen = 0;
      s.section_target = target;
      s.section_ran = false;
      s.captures.clear();
      try {
        t.fn();
      } catch (const AssertionFailed&) {
        ok = false;
      } catch (const std::exception& e) {
        std::fprintf(stderr, "%s:%d: FAILED: unexpected exception: %s\n", t.file, t.line, e.what());
        ok = false;
      } catch (...) {
        std::fprintf(stderr, "%s:%d: FAILED: unexpected unknown exception\n", t.file, t.line);
        ok = false;
      }
      if (!ok) break;
      if (target + 1 >= s.section_seen) break;  // every section has had its pass
    }
    if (!ok) {
      ++failed;
      std::fprintf(stderr, "  in test case \"%s\"\n", t.name.c_str());
    }
  }
  if (failed == 0)
    std::printf("All tests passed (%lld assertions in %d test cases)\n", state().assertions, ran);
  else
    std::printf("test cases: %d | %d passed | %d failed (%lld assertions)\n", ran, ran - failed, failed,
                state().assertions);
  return failed == 0 ? 0 : 1;
}

}  // namespace Catch

#define CATCH_INTERNAL_CAT2(a, b) a##b
#define CATCH_INTERNAL_CAT(a, b) CATCH_INTERNAL_CAT2(a, b)
#define CATCH_INTERNAL_UNIQUE(n) CATCH_INTERNAL_CAT(n, __LINE__)

#define CATCH_TEST_CASE_IMPL(fn, ...)                                                         \
  static void fn();                                                                          \
  namespace {                                                                                \
  const Catch::Registrar CATCH_INTERNAL_CAT(fn, _reg)(CATCH_TC_NAME(__VA_ARGS__, ""),        \
                                                      CATCH_TC_TAGS(__VA_ARGS__, "", ""),    \
                                                      &fn, __FILE__, __LINE__);              \
  }                                                                                          \
  static void fn()
#define CATCH_TC_NAME(name, ...) name
#define CATCH_TC_TAGS(name, tags, ...) tags
#define TEST_CASE(...) CATCH_TEST_CASE_IMPL(CATCH_INTERNAL_UNIQUE(catch_tc_), __VA_ARGS__)

#define SECTION(name) if (const Catch::SectionGuard CATCH_INTERNAL_UNIQUE(catch_sec_){name})

#define REQUIRE(...)                                                           \
  do {                                                                         \
    ++Catch::state().assertions;                                               \
    if (!static_cast<bool>(__VA_ARGS__))                                       \
      Catch::fail("REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);                \
  } while (0)
#define REQUIRE_FALSE(...)                                                     \
  do {                                                                         \
    ++Catch::state().assertions;                                               \
    if (static_cast<bool>(__VA_ARGS__))                                        \
      Catch::fail("REQUIRE_FALSE", #__VA_ARGS__, __FILE__, __LINE__);          \
  } while (0)
#define REQUIRE_THROWS(...)                                                    \
  do {                                                                         \
    ++Catch::state().assertions;                                               \
    bool catch_threw_ = false;                                                 \
    try {                                                                      \
      static_cast<void>(__VA_ARGS__);                                          \
    } catch (...) {                                                            \
      catch_threw_ = true;                                                     \
    }                                                                          \
    if (!catch_threw_)                                                         \
      Catch::fail("REQUIRE_THROWS", #__VA_ARGS__, __FILE__, __LINE__,          \
                  " (no exception)");                                          \
  } while (0)
#define REQUIRE_NOTHROW(...)                                                   \
  do {                                                                         \
    ++Catch::state().assertions;                                               \
    try {                                                                      \
      static_cast<void>(__VA_ARGS__);                                          \
    } catch (const std::exception& catch_e_) {                                 \
      Catch::fail("REQUIRE_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__,         \
                  (std::string(" threw: ") + catch_e_.what()).c_str());        \
    } catch (...) {                                                            \
      Catch::fail("REQUIRE_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__,         \
                  " threw");                                                   \
    }                                                                          \
  } while (0)
#define CAPTURE(...) \
  const Catch::CaptureGuard CATCH_INTERNAL_UNIQUE(catch_cap_)(#__VA_ARGS__, __VA_ARGS__)

using Catch::Approx;

#ifdef CATCH_CONFIG_MAIN
int main(int argc, char** argv) { return Catch::run_all(argc, argv); }
#endif
