// doctest.h -- the subset of the doctest unit-test framework (2.4 API) that
// the reference's unit tests use (proj/tests/*.cpp: TEST_CASE, CHECK,
// CHECK_FALSE, CHECK_THROWS_AS, REQUIRE, REQUIRE_FALSE, FAIL,
// doctest::Approx).  The reference vendors doctest under proj/vendor/, which
// is absent from this image; this header lets those test files
// compile unmodified against the B200 host layer.  Failures print
// file:line and the expression; the process exits nonzero on any failure
// and prints doctest's summary line.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double v) : value_(v) {}
    Approx &epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx &scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    friend bool operator==(double lhs, const Approx &a) {
        return std::fabs(lhs - a.value_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx &a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx &a) { return !(lhs == a); }
    friend bool operator!=(const Approx &a, double rhs) { return !(rhs == a); }

  private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {

struct TestCase {
    const char *name;
    const char *file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase> &registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    long long asserts = 0, failed_asserts = 0;
    bool case_failed = false;
};
inline State &state() {
    static State s;
    return s;
}

struct RequireAbort {};  // ends the current test case after a failed REQUIRE / FAIL

struct Reg {
    Reg(const char *name, const char *file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

inline void report(bool ok, const char *kind, const char *expr, const char *file, int line) {
    State &s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}

inline int run_all() {
    int passed = 0, failed = 0;
    for (const TestCase &tc : registry()) {
        state().case_failed = false;
        try {
            tc.fn();
        } catch (const RequireAbort &) {
        } catch (const std::exception &e) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", tc.file, tc.line,
                         tc.name);
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed;
            std::fprintf(stderr, "  in TEST_CASE(\"%s\")\n", tc.name);
        } else {
            ++passed;
        }
    }
    const State &s = state();
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", passed + failed, passed, failed);
    std::printf("[doctest] assertions: %lld | %lld passed | %lld failed\n", s.asserts, s.asserts - s.failed_asserts,
                s.failed_asserts);
    std::printf("[doctest] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
    return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                   \
    static void fn();                                                                     \
    static const ::doctest::detail::Reg DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...) ::doctest::detail::report(static_cast<bool>(__VA_ARGS__), "CHECK", #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) \
    ::doctest::detail::report(!static_cast<bool>(__VA_ARGS__), "CHECK_FALSE", #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                                  \
    do {                                                                                              \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                      \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);           \
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                                    \
    } while (0)
#define REQUIRE_FALSE(...) REQUIRE(!(__VA_ARGS__))
#define FAIL(msg)                                                                                     \
    do {                                                                                              \
        ::doctest::detail::report(false, "FAIL", #msg, __FILE__, __LINE__);                            \
        throw ::doctest::detail::RequireAbort{};                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                    \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (const __VA_ARGS__ &) {                                                               \
            doctest_ok_ = true;                                                                       \
        } catch (...) {                                                                               \
        }                                                                                             \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS(expr)                                                                            \
    do {                                                                                              \
        bool doctest_ok_ = false;                                                                     \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (...) {                                                                               \
            doctest_ok_ = true;                                                                       \
        }                                                                                             \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS", #expr, __FILE__, __LINE__);             \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                           \
    do {                                                                                              \
        bool doctest_ok_ = true;                                                                      \
        try {                                                                                         \
            static_cast<void>(expr);                                                                  \
        } catch (...) {                                                                               \
            doctest_ok_ = false;                                                                      \
        }                                                                                             \
        ::doctest::detail::report(doctest_ok_, "CHECK_NOTHROW", #expr, __FILE__, __LINE__);            \
    } while (0)
#define CHECK_EQ(a, b) CHECK((a) == (b))
#define CHECK_NE(a, b) CHECK((a) != (b))
#define CHECK_LT(a, b) CHECK((a) < (b))
#define CHECK_LE(a, b) CHECK((a) <= (b))
#define CHECK_GT(a, b) CHECK((a) > (b))
#define CHECK_GE(a, b) CHECK((a) >= (b))
#define MESSAGE(msg) static_cast<void>(0)
#define INFO(...) static_cast<void>(0)
#define CAPTURE(...) static_cast<void>(0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
