// Minimal stand-in for the doctest single header, written for this repo.
// The reference keeps doctest in a git-ignored vendor/ directory
// (/root/reference/proj/.gitignore:2) that is absent, so its unit tests
// (tests/test_{quant,gemm,ssm,tensor}.cpp) cannot be compiled as shipped.
// This shim implements exactly the macro subset those files use
// (TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, FAIL, doctest::Approx with
// .epsilon) so the reference's own tests can gate the oracle build.
// Test infrastructure only.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

namespace doctest {
struct Approx {
    double value, eps = 1.1920928955078125e-05;  // doctest default: float eps * 100
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) { eps = e; return *this; }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) <
               a.eps * (1.0 + std::max(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};
namespace shim {
struct Case { const char* name; void (*fn)(); };
inline std::vector<Case>& registry() { static std::vector<Case> r; return r; }
inline long& failures() { static long f = 0; return f; }
inline long& checks() { static long c = 0; return c; }
struct Abort {};
struct Reg { Reg(const char* n, void (*f)()) { registry().push_back({n, f}); } };
inline void fail(const char* file, int line, const char* expr, bool fatal) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw Abort{};
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define TEST_CASE_IMPL(fn, name)                                                  \
    static void fn();                                                             \
    static ::doctest::shim::Reg DOCTEST_CAT(fn, _reg)(name, &fn);                 \
    static void fn()
#define TEST_CASE(name) TEST_CASE_IMPL(DOCTEST_CAT(doctest_case_, __LINE__), name)
#define DOCTEST_CHECK_IMPL(expr, fatal)                                           \
    do {                                                                          \
        ++::doctest::shim::checks();                                              \
        if (!(expr)) ::doctest::shim::fail(__FILE__, __LINE__, #expr, fatal);     \
    } while (0)
#define CHECK(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL((__VA_ARGS__), true)
#define FAIL(msg) ::doctest::shim::fail(__FILE__, __LINE__, msg, true)
#define CHECK_THROWS_AS(expr, exc)                                                \
    do {                                                                          \
        ++::doctest::shim::checks();                                              \
        bool doctest_caught = false;                                              \
        try { (void)(expr); } catch (const exc&) { doctest_caught = true; }       \
        catch (...) {}                                                            \
        if (!doctest_caught)                                                      \
            ::doctest::shim::fail(__FILE__, __LINE__, #expr " throws " #exc, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    long cases_failed = 0;
    for (auto& c : ::doctest::shim::registry()) {
        long before = ::doctest::shim::failures();
        try { c.fn(); } catch (const ::doctest::shim::Abort&) {
        } catch (const std::exception& e) {
            ++::doctest::shim::failures();
            std::fprintf(stderr, "case '%s' threw: %s\n", c.name, e.what());
        }
        if (::doctest::shim::failures() != before) {
            ++cases_failed;
            std::fprintf(stderr, "[case failed] %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] cases: %zu | failed: %ld | checks: %ld | failed checks: %ld\n",
                ::doctest::shim::registry().size(), cases_failed, ::doctest::shim::checks(),
                ::doctest::shim::failures());
    return cases_failed == 0 ? 0 : 1;
}
#endif
