// Minimal doctest-compatible harness (TEST INFRASTRUCTURE ONLY) for building the reference's unmodified
// test sources (/root/reference/proj/tests/test_*.cpp), whose `vendor/doctest` is not vendored
// (proj/CMakeLists.txt:7).  It implements exactly what those sources use: TEST_CASE, flat SUBCASEs (one
// subcase per run of the test case, as doctest does), CHECK, REQUIRE, CHECK_THROWS_AS, FAIL and
// doctest::Approx(x).epsilon(e).  main() runs every test case and prints one summary line:
//   [reftest] <binary>: <cases> test cases, <failed cases> failed, <checks> checks, <failed checks> failed
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = 1.1920928955078125e-07 * 100, sc = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        sc = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.value) < b.eps * (b.sc + std::max(std::fabs(a), std::fabs(b.value)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    friend bool operator!=(const Approx& b, double a) { return !(a == b); }
};

namespace detail {
struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Register {
    Register(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct State {
    long checks = 0, failed = 0;
    bool case_failed = false;
    std::set<std::string> done;
    const char* entered = nullptr;
    const char* current = "";
};
inline State& state() {
    static State s;
    return s;
}
struct RequireFailed {};
inline bool enter_subcase(const char* name) {
    State& s = state();
    if (s.entered || s.done.count(name)) return false;
    s.entered = name;
    return true;
}
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    s.checks++;
    if (ok) return;
    s.failed++;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: FAILED: %s  [test case \"%s\"%s%s%s]\n", file, line, expr, s.current,
                 s.entered ? ", subcase \"" : "", s.entered ? s.entered : "", s.entered ? "\"" : "");
    if (require) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                      \
    static void fn();                                                                                  \
    static doctest::detail::Register DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);             \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (doctest::detail::enter_subcase(name))
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, ...)                                                                     \
    do {                                                                                               \
        bool doctest_caught = false;                                                                   \
        try {                                                                                          \
            (void)(expr);                                                                              \
        } catch (const __VA_ARGS__&) {                                                                 \
            doctest_caught = true;                                                                     \
        } catch (...) {                                                                                \
        }                                                                                              \
        doctest::detail::check(doctest_caught, "CHECK_THROWS_AS(" #expr ", " #__VA_ARGS__ ")", __FILE__, \
                               __LINE__, false);                                                       \
    } while (0)
#define FAIL(msg) doctest::detail::check(false, "FAIL(" #msg ")", __FILE__, __LINE__, true)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int, char** argv) {
    using namespace doctest::detail;
    State& s = state();
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        cases++;
        s.done.clear();
        s.current = tc.name;
        s.case_failed = false;
        for (;;) {
            s.entered = nullptr;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                s.failed++;
                s.case_failed = true;
                std::fprintf(stderr, "%s:%d: FAILED: unexpected exception: %s  [test case \"%s\"]\n", tc.file, tc.line,
                             e.what(), tc.name);
            }
            if (!s.entered) break;
            s.done.insert(s.entered);
        }
        if (s.case_failed) {
            failed_cases++;
            std::fprintf(stderr, "[case failed] %s\n", tc.name);
        }
    }
    std::printf("[reftest] %s: %d test cases, %d failed, %ld checks, %ld failed\n", argv[0], cases, failed_cases,
                s.checks, s.failed);
    return failed_cases ? 1 : 0;
}
#endif
