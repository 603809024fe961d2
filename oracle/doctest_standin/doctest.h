// doctest.h — a minimal stand-in for the doctest unit-test framework, enough
// to compile the reference's own unit tests (proj/tests/test_*.cpp and
// doctest_main.cpp) unmodified.
//
// TEST INFRASTRUCTURE.  The reference's tests include "doctest.h" from its
// vendored third-party tree, which is not shipped, so they cannot be built
// as delivered.  This header implements only the surface those tests use —
// TEST_SUITE blocks, TEST_CASE, CHECK / CHECK_FALSE / REQUIRE / FAIL /
// CHECK_THROWS_AS, doctest::Approx with epsilon(), and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so oracle/Makefile can build the
// suite against the pure reference and against the B200 binding
// (ref_binding/) and the GPU tests can compare the two runs.  Output: one
// line per failed check, then "[doctest] test cases: T | P passed | F failed"
// and "[doctest] assertions: A | ... failed"; the exit code is 1 when any
// check failed.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
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
    // doctest's rule: |lhs - value| < epsilon * (scale + max(|lhs|, |value|))
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) < epsilon_ * (scale_ + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_;
    double epsilon_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

inline bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
inline bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
inline bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
inline bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
inline bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value() || rhs.matches(lhs); }
inline bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value() || rhs.matches(lhs); }
inline bool operator<(double lhs, const Approx& rhs) { return lhs < rhs.value() && !rhs.matches(lhs); }
inline bool operator>(double lhs, const Approx& rhs) { return lhs > rhs.value() && !rhs.matches(lhs); }

namespace detail {

struct TestCase {
    void (*fn)();
    const char* name;
    const char* suite;
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    long long assertions = 0, failed_assertions = 0;
    bool current_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};  // a failed REQUIRE ends its test case

struct Registrar {
    Registrar(void (*fn)(), const char* name, const char* suite, const char* file, int line) {
        registry().push_back(TestCase{fn, name, suite, file, line});
    }
};

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.assertions;
    if (ok) return;
    ++s.failed_assertions;
    s.current_failed = true;
    std::printf("%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}

inline int run_all() {
    State& s = state();
    int passed = 0, failed = 0;
    for (const TestCase& t : registry()) {
        s.current_failed = false;
        try {
            t.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw: %s\n", t.file, t.line, t.name, e.what());
            s.current_failed = true;
        } catch (...) {
            std::printf("%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", t.file, t.line, t.name);
            s.current_failed = true;
        }
        if (s.current_failed) {
            ++failed;
            std::printf("[doctest] FAILED: %s / %s\n", t.suite, t.name);
        } else {
            ++passed;
        }
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", passed + failed, passed, failed);
    std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", s.assertions,
                s.assertions - s.failed_assertions, s.failed_assertions);
    return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

// the enclosing TEST_SUITE's name for the registrations inside it
namespace doctest_suite {
inline const char* name() { return ""; }
}  // namespace doctest_suite

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)

#define TEST_SUITE(suite_name)                                                     \
    namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__) {                           \
    namespace doctest_suite {                                                      \
    inline const char* name() { return suite_name; }                               \
    }                                                                              \
    }                                                                              \
    namespace DOCTEST_CAT(doctest_suite_ns_, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, test_name)                                                  \
    static void fn();                                                                               \
    static const ::doctest::detail::Registrar reg(fn, test_name, doctest_suite::name(), __FILE__, __LINE__); \
    static void fn()

#define TEST_CASE(test_name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_fn_, __LINE__), DOCTEST_CAT(doctest_test_reg_, __LINE__), test_name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                 \
    do {                                                                                             \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                     \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);         \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                   \
    } while (0)
#define FAIL(msg)                                                                                    \
    do {                                                                                             \
        ::doctest::detail::report(false, "FAIL", msg, __FILE__, __LINE__);                           \
        throw ::doctest::detail::RequireAbort{};                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                   \
    do {                                                                                             \
        bool doctest_threw_ = false;                                                                 \
        try {                                                                                        \
            static_cast<void>(expr);                                                                 \
        } catch (const __VA_ARGS__&) {                                                               \
            doctest_threw_ = true;                                                                   \
        } catch (...) {                                                                              \
        }                                                                                            \
        ::doctest::detail::report(doctest_threw_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, \
                                  __LINE__);                                                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
