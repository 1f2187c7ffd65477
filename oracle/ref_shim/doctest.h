// ORACLE — test infrastructure only. The subset of doctest (vendored by the
// reference under proj/vendor/, which is not in the repository) that the
// reference's own test suites use: TEST_CASE, SUBCASE (re-running the test
// case once per subcase, as doctest does), CHECK / CHECK_FALSE (record and
// continue), REQUIRE (record and leave the test case), CHECK_THROWS_AS, and
// doctest::Approx with doctest's default epsilon and scale. The suites under
// /root/reference/proj/tests then build unmodified against oracle/_ref.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || lhs == rhs; }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || lhs == rhs; }
    friend bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value_ && lhs != rhs; }
    friend bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value_ && lhs != rhs; }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
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
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct RequireFailed {};
struct State {
    long checks = 0, failures = 0;
    int subcase_target = 0, subcase_seen = 0;
    bool current_failed = false;
};
inline State& state() {
    static State s;
    return s;
}
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s FAILED: %s\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
// SUBCASE: run k of a test case enters only the k-th subcase it meets.
struct Subcase {
    bool enter;
    explicit Subcase(const char*) {
        State& s = state();
        enter = s.subcase_seen++ == s.subcase_target;
    }
    explicit operator bool() const { return enter; }
};
}  // namespace detail

inline int run_all() {
    using namespace detail;
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        State& s = state();
        s.current_failed = false;
        for (s.subcase_target = 0;; ++s.subcase_target) {
            s.subcase_seen = 0;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                s.current_failed = true;
                std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            }
            if (s.subcase_seen <= s.subcase_target + 1) break;  // no further subcase to enter
        }
        if (s.current_failed) {
            ++failed_cases;
            std::fprintf(stderr, "[doctest-shim] FAILED test case: %s\n", tc.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                registry().size(), registry().size() - size_t(failed_cases), failed_cases, state().checks,
                state().failures);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                     \
    static void fn();                                                                             \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);     \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) ::doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define REQUIRE_FALSE(...) ::doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        bool doctest_ok_ = false;                                                                 \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_ok_ = true;                                                                   \
        } catch (...) {                                                                           \
        }                                                                                         \
        ::doctest::detail::check(doctest_ok_, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                       \
    do {                                                                                          \
        bool doctest_ok_ = true;                                                                  \
        try {                                                                                     \
            static_cast<void>(expr);                                                              \
        } catch (...) {                                                                           \
            doctest_ok_ = false;                                                                  \
        }                                                                                         \
        ::doctest::detail::check(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
