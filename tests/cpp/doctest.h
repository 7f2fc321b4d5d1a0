// doctest.h — minimal doctest-compatible test shim (the real doctest is not
// vendored in this image).  Implements exactly the subset the reference's unit
// suites use — TEST_CASE, CHECK/REQUIRE(+_FALSE), CHECK_NOTHROW,
// CHECK_THROWS_AS, doctest::Approx(+epsilon) — so /root/reference/proj/tests/
// test_lora.cpp, test_batch_select.cpp and test_workload.cpp compile unchanged
// against the B200 façade headers (include/fusim/).  Runner: tests/cpp/main.cpp.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100;
    double scale_ = 1.0;
};

namespace detail {
struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};
struct RequireFailed {};
inline long& failures() { static long f = 0; return f; }
inline long& assertions() { static long a = 0; return a; }
inline void fail(const char* kind, const char* expr, const char* file, int line) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED %s( %s )\n", file, line, kind, expr);
}
}  // namespace detail

inline int run_all() {
    long cases_failed = 0;
    for (const auto& c : detail::registry()) {
        const long before = detail::failures();
        try {
            c.fn();
        } catch (const detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++detail::failures();
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
        }
        if (detail::failures() != before) {
            ++cases_failed;
            std::fprintf(stderr, "  in TEST CASE \"%s\"\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %ld failed | assertions: %ld | failed: %ld\n",
                detail::registry().size(), detail::registry().size() - cases_failed, cases_failed,
                detail::assertions(), detail::failures());
    return cases_failed == 0 ? 0 : 1;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                 \
    static void fn();                                                                         \
    static ::doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)

#define DOCTEST_ASSERT_(kind, cond, expr_str, is_require)                             \
    do {                                                                              \
        ++::doctest::detail::assertions();                                            \
        if (!(cond)) {                                                                \
            ::doctest::detail::fail(kind, expr_str, __FILE__, __LINE__);              \
            if (is_require) throw ::doctest::detail::RequireFailed{};                 \
        }                                                                             \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_NOTHROW(...)                                                            \
    do {                                                                              \
        bool ok_ = true;                                                              \
        try { (void)(__VA_ARGS__); } catch (...) { ok_ = false; }                     \
        DOCTEST_ASSERT_("CHECK_NOTHROW", ok_, #__VA_ARGS__, false);                   \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                    \
    do {                                                                              \
        bool ok_ = false;                                                             \
        try { (void)(expr); } catch (const __VA_ARGS__&) { ok_ = true; } catch (...) {} \
        DOCTEST_ASSERT_("CHECK_THROWS_AS", ok_, #expr " throws " #__VA_ARGS__, false); \
    } while (0)
