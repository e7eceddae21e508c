// doctest.h -- a minimal stand-in for the doctest framework (TEST INFRASTRUCTURE ONLY).
//
// The reference's unit tests (/root/reference/proj/tests/unit/*.cpp) are written against doctest,
// which is not installed here.  This header implements the subset they use -- TEST_CASE, CHECK,
// CHECK_FALSE, REQUIRE, REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW, doctest::Approx and
// DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN -- so those files compile unmodified against the B200 drop-in
// (include/zinpaint_b200.hpp) and run on the GPU (tests/test_dropin.py).
//
// Semantics kept: a failing CHECK records the failure and continues, a failing REQUIRE ends the
// test case; every test case runs even after failures; the process exits non-zero iff anything
// failed.  The summary line reports test cases and assertions like doctest's.
#ifndef ZI_DOCTEST_SHIM_H
#define ZI_DOCTEST_SHIM_H

#include <cmath>
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.eps_ * (rhs.scale_ + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: FLT_EPSILON * 100
    double scale_ = 1.0;
};

namespace detail {

struct test_case {
    void (*fn)();
    const char* name;
    const char* file;
    int line;
};

struct require_failed {};

inline std::vector<test_case>& registry() {
    static std::vector<test_case> r;
    return r;
}

struct counters {
    long asserts = 0, failed_asserts = 0;
    bool current_failed = false;
};

inline counters& stats() {
    static counters c;
    return c;
}

inline int reg(void (*fn)(), const char* name, const char* file, int line) {
    registry().push_back({fn, name, file, line});
    return 0;
}

inline void check(bool ok, const char* kind, const char* expr, const char* file, int line, bool fatal) {
    ++stats().asserts;
    if (ok) return;
    ++stats().failed_asserts;
    stats().current_failed = true;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
    if (fatal) throw require_failed{};
}

inline int run_all() {
    long passed = 0, failed = 0;
    for (const auto& tc : registry()) {
        stats().current_failed = false;
        try {
            tc.fn();
        } catch (const require_failed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw: %s\n", tc.file, tc.line, tc.name, e.what());
            stats().current_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: ERROR: test case \"%s\" threw an unknown exception\n", tc.file, tc.line,
                         tc.name);
            stats().current_failed = true;
        }
        if (stats().current_failed) {
            ++failed;
            std::fprintf(stderr, "FAILED: %s\n", tc.name);
        } else {
            ++passed;
        }
    }
    std::printf("[doctest] test cases: %ld | %ld passed | %ld failed\n", passed + failed, passed, failed);
    std::printf("[doctest] assertions: %ld | %ld passed | %ld failed\n", stats().asserts,
                stats().asserts - stats().failed_asserts, stats().failed_asserts);
    return failed == 0 && stats().failed_asserts == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                     \
    static void fn();                                                                                 \
    [[maybe_unused]] static const int DOCTEST_CAT(fn, _reg) = ::doctest::detail::reg(&fn, name, __FILE__, __LINE__); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __COUNTER__), name)

#define DOCTEST_ASSERT(kind, fatal, ...) \
    ::doctest::detail::check(static_cast<bool>(__VA_ARGS__), kind, #__VA_ARGS__, __FILE__, __LINE__, fatal)
#define CHECK(...) DOCTEST_ASSERT("CHECK", false, __VA_ARGS__)
#define REQUIRE(...) DOCTEST_ASSERT("REQUIRE", true, __VA_ARGS__)
#define CHECK_FALSE(...) DOCTEST_ASSERT("CHECK_FALSE", false, !(__VA_ARGS__))
#define REQUIRE_FALSE(...) DOCTEST_ASSERT("REQUIRE_FALSE", true, !(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, ...)                                                         \
    do {                                                                                   \
        bool doctest_ok_ = false;                                                          \
        try {                                                                              \
            expr;                                                                          \
        } catch (const __VA_ARGS__&) {                                                     \
            doctest_ok_ = true;                                                            \
        } catch (...) {                                                                    \
        }                                                                                  \
        ::doctest::detail::check(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)
#define CHECK_NOTHROW(...)                                                                 \
    do {                                                                                   \
        bool doctest_ok_ = true;                                                           \
        try {                                                                              \
            __VA_ARGS__;                                                                   \
        } catch (...) {                                                                    \
            doctest_ok_ = false;                                                           \
        }                                                                                  \
        ::doctest::detail::check(doctest_ok_, "CHECK_NOTHROW", #__VA_ARGS__, __FILE__, __LINE__, false); \
    } while (0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif

#endif  // ZI_DOCTEST_SHIM_H
