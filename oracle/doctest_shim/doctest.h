// Minimal doctest-compatible test harness (test infrastructure, NOT product code).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are written
// against doctest, which the reference tree does not vendor. This header provides
// the subset they use — TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, CHECK_NOTHROW,
// INFO, FAIL, doctest::Approx and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN — so the
// reference's own suites compile unmodified against this repo's kvrail headers and
// libkvrail.so (oracle/Makefile target `suites`, tests/test_ref_suites.py).
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx &epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx &scale(double s) {
        scl = s;
        return *this;
    }
    bool matches(double other) const {
        return std::fabs(other - value) < eps * (scl + std::max(std::fabs(other), std::fabs(value)));
    }
    double value;
    double eps = double(std::numeric_limits<float>::epsilon()) * 100;
    double scl = 1.0;
};
inline bool operator==(double a, const Approx &b) { return b.matches(a); }
inline bool operator==(const Approx &a, double b) { return a.matches(b); }
inline bool operator!=(double a, const Approx &b) { return !b.matches(a); }
inline bool operator!=(const Approx &a, double b) { return !a.matches(b); }

namespace detail {

struct Case {
    const char *name, *file;
    int line;
    void (*fn)();
};
inline std::vector<Case> &registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char *name, const char *file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};
struct Abort {}; // REQUIRE / FAIL end the current test case
struct State {
    int failures = 0;
    std::string info;
    const char *current = "";
};
inline State &state() {
    static State s;
    return s;
}
inline void fail(const char *file, int line, const std::string &what) {
    State &s = state();
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s%s%s\n", file, line, s.current, what.c_str(),
                 s.info.empty() ? "" : "  [info: ", s.info.empty() ? "" : (s.info + "]").c_str());
}
template <typename... A> std::string cat(const A &...a) {
    std::ostringstream o;
    (o << ... << a);
    return o.str();
}

inline int run_all() {
    int failed_cases = 0, n = 0;
    for (const Case &c : registry()) {
        ++n;
        State &s = state();
        const int before = s.failures;
        s.current = c.name;
        s.info.clear();
        try {
            c.fn();
        } catch (const Abort &) {
        } catch (const std::exception &e) {
            fail(c.file, c.line, std::string("unexpected exception: ") + e.what());
        } catch (...) {
            fail(c.file, c.line, "unexpected exception");
        }
        failed_cases += s.failures != before;
    }
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | assertions failed: %d\n", n,
                n - failed_cases, failed_cases, state().failures);
    return failed_cases ? 1 : 0;
}

} // namespace detail
} // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC(fn, name)                                                                                  \
    static void fn();                                                                                          \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);                    \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define CHECK(...)                                                                                             \
    do {                                                                                                       \
        if (!(__VA_ARGS__))                                                                                    \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK( " #__VA_ARGS__ " )");                            \
    } while (0)
#define REQUIRE(...)                                                                                           \
    do {                                                                                                       \
        if (!(__VA_ARGS__)) {                                                                                  \
            doctest::detail::fail(__FILE__, __LINE__, "REQUIRE( " #__VA_ARGS__ " )");                          \
            throw doctest::detail::Abort{};                                                                    \
        }                                                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, ...)                                                                             \
    do {                                                                                                       \
        bool doctest_threw_ = false;                                                                           \
        try {                                                                                                  \
            (void)(expr);                                                                                      \
        } catch (const __VA_ARGS__ &) {                                                                        \
            doctest_threw_ = true;                                                                             \
        } catch (...) {                                                                                        \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): wrong exception type");   \
            doctest_threw_ = true;                                                                             \
        }                                                                                                      \
        if (!doctest_threw_)                                                                                   \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr " ): did not throw");          \
    } while (0)
#define CHECK_NOTHROW(...)                                                                                     \
    do {                                                                                                       \
        try {                                                                                                  \
            (void)(__VA_ARGS__);                                                                               \
        } catch (...) {                                                                                        \
            doctest::detail::fail(__FILE__, __LINE__, "CHECK_NOTHROW( " #__VA_ARGS__ " ) threw");              \
        }                                                                                                      \
    } while (0)
#define INFO(...) (doctest::detail::state().info = doctest::detail::cat(__VA_ARGS__))
#define FAIL(...)                                                                                              \
    do {                                                                                                       \
        doctest::detail::fail(__FILE__, __LINE__, doctest::detail::cat("FAIL: ", __VA_ARGS__));                \
        throw doctest::detail::Abort{};                                                                        \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
