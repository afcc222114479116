// TEST-ONLY Catch2-subset shim (oracle infrastructure).
//
// The reference tests use Catch2 v3 amalgamated (/root/reference/proj/tests/CMakeLists.txt:1-2),
// which is absent from this image. This header implements the subset those tests use:
// TEST_CASE, SECTION (Catch's re-run-per-leaf-section semantics), CHECK, CHECK_FALSE,
// REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, INFO, FAIL, SUCCEED and
// Catch::Approx (epsilon/margin/scale). Define CATCH_SHIM_MAIN in exactly one TU
// (oracle/shim/catch2/catch_main.cpp) to get main().
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace catchshim {

struct AbortTest {};

struct TestCase {
  std::string name;
  void (*fn)();
  const char* file;
  int line;
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}

struct Registrar {
  Registrar(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({name, fn, file, line});
  }
};

struct State {
  std::string current_test;
  long assertions = 0;
  long failures = 0;
  bool test_failed = false;
  // section tracking
  std::set<std::string> done;
  std::vector<std::string> stack;       // entered section paths
  std::vector<bool> level_entered;      // per depth: a section was entered in this run
  std::vector<bool> child_pending;      // per depth: an unfinished child was skipped
  bool pending = false;
  std::vector<std::string> infos;
};

inline State& state() {
  static State s;
  return s;
}

inline void report_failure(const char* kind, const char* expr, const char* file, int line,
                           const std::string& extra = "") {
  State& s = state();
  ++s.failures;
  s.test_failed = true;
  std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in test \"%s\"%s%s\n", file, line, kind, expr,
               s.current_test.c_str(), extra.empty() ? "" : " : ", extra.c_str());
  for (const std::string& i : s.infos) std::fprintf(stderr, "    with: %s\n", i.c_str());
}

class Section {
 public:
  Section(const char* name, const char* /*file*/, int /*line*/) {
    State& s = state();
    const std::size_t depth = s.stack.size();
    if (s.level_entered.size() <= depth) s.level_entered.resize(depth + 1, false);
    if (s.child_pending.size() <= depth + 1) s.child_pending.resize(depth + 2, false);
    path_ = (s.stack.empty() ? std::string() : s.stack.back() + "/") + name;
    if (s.done.count(path_)) {
      entered_ = false;
    } else if (s.level_entered[depth]) {
      entered_ = false;
      s.pending = true;
      s.child_pending[depth] = true;
    } else {
      entered_ = true;
      s.level_entered[depth] = true;
      s.stack.push_back(path_);
      if (s.level_entered.size() <= depth + 1) s.level_entered.resize(depth + 2, false);
      s.level_entered[depth + 1] = false;
      s.child_pending[depth + 1] = false;
    }
  }
  ~Section() {
    if (!entered_) return;
    State& s = state();
    const std::size_t depth = s.stack.size();  // depth of children of this section
    const bool child_left = depth < s.child_pending.size() && s.child_pending[depth];
    s.stack.pop_back();
    if (!child_left) s.done.insert(path_);
  }
  explicit operator bool() const { return entered_; }

 private:
  std::string path_;
  bool entered_ = false;
};

class ScopedInfo {
 public:
  ScopedInfo() = default;
  ~ScopedInfo() {
    if (pushed_) state().infos.pop_back();
  }
  template <class T>
  ScopedInfo& operator<<(const T& v) {
    os_ << v;
    if (pushed_) state().infos.back() = os_.str();
    else {
      state().infos.push_back(os_.str());
      pushed_ = true;
    }
    return *this;
  }

 private:
  std::ostringstream os_;
  bool pushed_ = false;
};

inline int run_all(int argc, char** argv) {
  std::vector<std::string> filters;
  for (int i = 1; i < argc; ++i) filters.emplace_back(argv[i]);
  State& s = state();
  int tests = 0, failed_tests = 0;
  for (const TestCase& tc : registry()) {
    if (!filters.empty()) {
      bool hit = false;
      for (const auto& f : filters) hit = hit || tc.name.find(f) != std::string::npos;
      if (!hit) continue;
    }
    ++tests;
    s.current_test = tc.name;
    s.test_failed = false;
    s.done.clear();
    int runs = 0;
    do {
      s.stack.clear();
      s.level_entered.assign(1, false);
      s.child_pending.assign(2, false);
      s.pending = false;
      s.infos.clear();
      try {
        tc.fn();
      } catch (const AbortTest&) {
      } catch (const std::exception& e) {
        report_failure("unexpected exception", e.what(), tc.file, tc.line);
      } catch (...) {
        report_failure("unexpected exception", "(unknown)", tc.file, tc.line);
      }
      ++runs;
    } while (s.pending && runs < 10000);
    if (s.test_failed) ++failed_tests;
  }
  std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", tests,
              tests - failed_tests, failed_tests, s.assertions, s.failures);
  return failed_tests == 0 ? 0 : 1;
}

}  // namespace catchshim

namespace Catch {

class Approx {
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
    const double diff = std::fabs(value_ - other);
    if (diff <= margin_) return true;
    return diff <= epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_));
  }
  friend bool operator==(double lhs, const Approx& rhs) { return rhs.equals(lhs); }
  friend bool operator==(const Approx& lhs, double rhs) { return lhs.equals(rhs); }
  friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.equals(lhs); }
  friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.equals(rhs); }

 private:
  double value_;
  double epsilon_;
  double margin_ = 0.0;
  double scale_ = 0.0;
};

inline unsigned rngSeed() { return 0; }

}  // namespace Catch

#define CATCHSHIM_CAT2(a, b) a##b
#define CATCHSHIM_CAT(a, b) CATCHSHIM_CAT2(a, b)
#define CATCHSHIM_UNIQ(p) CATCHSHIM_CAT(p, __LINE__)

#define TEST_CASE(name, ...)                                                          \
  static void CATCHSHIM_UNIQ(catchshim_tc_)();                                        \
  static ::catchshim::Registrar CATCHSHIM_UNIQ(catchshim_reg_)(                       \
      name, &CATCHSHIM_UNIQ(catchshim_tc_), __FILE__, __LINE__);                      \
  static void CATCHSHIM_UNIQ(catchshim_tc_)()

#define SECTION(name, ...) \
  if (::catchshim::Section CATCHSHIM_UNIQ(catchshim_sec_){name, __FILE__, __LINE__})

#define CATCHSHIM_ASSERT(kind, abort, cond, text)                                 \
  do {                                                                            \
    ++::catchshim::state().assertions;                                            \
    bool catchshim_ok_ = false;                                                   \
    try {                                                                         \
      catchshim_ok_ = static_cast<bool>(cond);                                    \
    } catch (const std::exception& e) {                                           \
      ::catchshim::report_failure(kind, text, __FILE__, __LINE__, e.what());      \
      if (abort) throw ::catchshim::AbortTest{};                                  \
      break;                                                                      \
    }                                                                             \
    if (!catchshim_ok_) {                                                         \
      ::catchshim::report_failure(kind, text, __FILE__, __LINE__);                \
      if (abort) throw ::catchshim::AbortTest{};                                  \
    }                                                                             \
  } while (0)

#define CHECK(...) CATCHSHIM_ASSERT("CHECK", false, (__VA_ARGS__), #__VA_ARGS__)
#define CHECK_FALSE(...) CATCHSHIM_ASSERT("CHECK_FALSE", false, !(__VA_ARGS__), #__VA_ARGS__)
#define REQUIRE(...) CATCHSHIM_ASSERT("REQUIRE", true, (__VA_ARGS__), #__VA_ARGS__)
#define REQUIRE_FALSE(...) CATCHSHIM_ASSERT("REQUIRE_FALSE", true, !(__VA_ARGS__), #__VA_ARGS__)

#define CATCHSHIM_THROWS_AS(kind, abort, expr, type)                              \
  do {                                                                            \
    ++::catchshim::state().assertions;                                            \
    bool catchshim_ok_ = false;                                                   \
    try {                                                                         \
      static_cast<void>(expr);                                                    \
    } catch (const type&) {                                                       \
      catchshim_ok_ = true;                                                       \
    } catch (...) {                                                               \
    }                                                                             \
    if (!catchshim_ok_) {                                                         \
      ::catchshim::report_failure(kind, #expr ", " #type, __FILE__, __LINE__);    \
      if (abort) throw ::catchshim::AbortTest{};                                  \
    }                                                                             \
  } while (0)

#define CHECK_THROWS_AS(expr, type) CATCHSHIM_THROWS_AS("CHECK_THROWS_AS", false, expr, type)
#define REQUIRE_THROWS_AS(expr, type) CATCHSHIM_THROWS_AS("REQUIRE_THROWS_AS", true, expr, type)
#define CHECK_NOTHROW(...) \
  CATCHSHIM_ASSERT("CHECK_NOTHROW", false, ((void)(__VA_ARGS__), true), #__VA_ARGS__)

#define INFO(msg)                                              \
  ::catchshim::ScopedInfo CATCHSHIM_UNIQ(catchshim_info_);     \
  CATCHSHIM_UNIQ(catchshim_info_) << msg
#define CAPTURE(x) INFO(#x " := " << (x))

#define FAIL(msg)                                                                   \
  do {                                                                              \
    std::ostringstream catchshim_os_;                                               \
    catchshim_os_ << msg;                                                           \
    ::catchshim::report_failure("FAIL", catchshim_os_.str().c_str(), __FILE__, __LINE__); \
    throw ::catchshim::AbortTest{};                                                 \
  } while (0)
#define SUCCEED(...) ((void)0)

#ifdef CATCH_SHIM_MAIN
int main(int argc, char** argv) { return ::catchshim::run_all(argc, argv); }
#endif
