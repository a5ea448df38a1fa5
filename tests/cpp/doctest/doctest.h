// Minimal doctest-compatible harness (doctest itself is not vendored in this image).
// Enough of the API for the reference's tests/test_render.cpp: TEST_SUITE, TEST_CASE,
// CHECK, REQUIRE, CHECK_THROWS_AS and doctest::Approx (epsilon/scale semantics of
// doctest 2.x: |a - b| < eps * (scale + max(|a|, |b|)), default eps = 100 * FLT_EPSILON).
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    Approx& scale(double s) {
        scl = s;
        return *this;
    }
    double value, eps = (double)FLT_EPSILON * 100, scl = 1.0;
};
inline bool operator==(double lhs, const Approx& a) {
    return std::fabs(lhs - a.value) < a.eps * (a.scl + std::max(std::fabs(lhs), std::fabs(a.value)));
}
inline bool operator==(const Approx& a, double rhs) { return rhs == a; }

struct Registry {
    struct Case {
        const char* name;
        void (*fn)();
    };
    std::vector<Case> cases;
    int checks = 0, failures = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};
struct Reg {
    Reg(const char* name, void (*fn)()) { Registry::get().cases.push_back({name, fn}); }
};
struct RequireFail {};
inline thread_local const char* current_case = "";
inline bool check(bool ok, const char* expr, const char* file, int line) {
    Registry& r = Registry::get();
    ++r.checks;
    if (!ok) {
        ++r.failures;
        std::printf("%s:%d: FAILED in \"%s\": %s\n", file, line, current_case, expr);
    }
    return ok;
}

inline int run_all() {
    Registry& r = Registry::get();
    int failed_cases = 0;
    for (const auto& c : r.cases) {
        current_case = c.name;
        const int before = r.failures;
        try {
            c.fn();
        } catch (const RequireFail&) {
        } catch (const std::exception& e) {
            ++r.failures;
            std::printf("FAILED in \"%s\": unexpected exception: %s\n", c.name, e.what());
        }
        const bool ok = r.failures == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
    }
    std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n[doctest] assertions: %d | %d failed\n",
                r.cases.size(), r.cases.size() - failed_cases, failed_cases, r.checks, r.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_SUITE(name) namespace DOCTEST_CAT(doctest_suite_, __LINE__)
#define TEST_CASE(name)                                                                               \
    static void DOCTEST_CAT(doctest_case_, __LINE__)();                                               \
    static ::doctest::Reg DOCTEST_CAT(doctest_reg_, __LINE__)(name, DOCTEST_CAT(doctest_case_, __LINE__)); \
    static void DOCTEST_CAT(doctest_case_, __LINE__)()
#define CHECK(...) ::doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                              \
    do {                                                                                          \
        if (!::doctest::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)) \
            throw ::doctest::RequireFail();                                                       \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                             \
    do {                                                                     \
        bool doctest_ok = false;                                             \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (const T&) {                                                 \
            doctest_ok = true;                                               \
        } catch (...) {                                                      \
        }                                                                    \
        ::doctest::check(doctest_ok, "throws " #T ": " #expr, __FILE__, __LINE__); \
    } while (0)

#define CHECK_THROWS(expr)                                                   \
    do {                                                                     \
        bool doctest_ok = false;                                             \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (...) {                                                      \
            doctest_ok = true;                                               \
        }                                                                    \
        ::doctest::check(doctest_ok, "throws: " #expr, __FILE__, __LINE__);  \
    } while (0)
#define CHECK_NOTHROW(expr)                                                  \
    do {                                                                     \
        bool doctest_ok = true;                                              \
        try {                                                                \
            (void)(expr);                                                    \
        } catch (...) {                                                      \
            doctest_ok = false;                                              \
        }                                                                    \
        ::doctest::check(doctest_ok, "nothrow: " #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::run_all(); }
#endif
