// doctest.h — TEST INFRASTRUCTURE: a minimal doctest-compatible shim.
//
// The reference's unit tests (/root/reference/proj/tests/*.cpp) include
// <doctest.h>, which is not vendored. This shim implements the subset they
// use (TEST_CASE, single-level SUBCASE, CHECK/CHECK_FALSE/REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains)
// so oracle/Makefile can compile those tests, unmodified, against both the
// reference library and our drop-in libmoesched.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value;
    double eps = 1.1920928955078125e-07 * 100;
    double scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
};
inline bool operator==(double a, const Approx& b) {
    return std::fabs(a - b.value) < b.eps * (b.scale + std::max(std::fabs(a), std::fabs(b.value)));
}
inline bool operator==(const Approx& b, double a) { return a == b; }
inline bool operator!=(double a, const Approx& b) { return !(a == b); }

struct Contains {
    std::string s;
    explicit Contains(const char* x) : s(x) {}
};
inline bool matches(const char* what, const char* want) { return std::strcmp(what, want) == 0; }
inline bool matches(const char* what, const Contains& c) { return std::string(what).find(c.s) != std::string::npos; }

namespace shim {
struct Case {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Reg {
    Reg(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct State {
    int target = 0, seen = 0, failures = 0, checks = 0;
    const char* current = "";
};
inline State& st() {
    static State s;
    return s;
}
struct RequireFailed {};
inline bool enter_subcase() { return st().seen++ == st().target; }
inline void report(bool ok, const char* expr, const char* file, int line) {
    ++st().checks;
    if (!ok) {
        ++st().failures;
        std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, st().current, expr);
    }
}
inline int run_all() {
    int failed_cases = 0;
    for (const Case& c : registry()) {
        st().current = c.name;
        const int before = st().failures;
        for (int pass = 0;; ++pass) {
            st().target = pass;
            st().seen = 0;
            try {
                c.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++st().failures;
                std::fprintf(stderr, "%s:%d: \"%s\" threw: %s\n", c.file, c.line, c.name, e.what());
            }
            if (st().seen <= pass + 1) break;
        }
        if (st().failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %d | %d failed\n", registry().size(),
                failed_cases, st().checks, st().failures);
    return st().failures ? 1 : 0;
}
}  // namespace shim
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                           \
    static void fn();                                                                   \
    static doctest::shim::Reg DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);    \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define SUBCASE(name) if (doctest::shim::enter_subcase())
#define CHECK(...) doctest::shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_FALSE(...) doctest::shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__)
#define REQUIRE(...)                                                                  \
    do {                                                                              \
        const bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                      \
        doctest::shim::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);         \
        if (!doctest_ok_) throw doctest::shim::RequireFailed{};                       \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                   \
    do {                                                                              \
        bool doctest_ok_ = false;                                                     \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type&) {                                                       \
            doctest_ok_ = true;                                                       \
        } catch (...) {                                                               \
        }                                                                             \
        doctest::shim::report(doctest_ok_, "throws " #type ": " #expr, __FILE__, __LINE__); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                     \
    do {                                                                              \
        bool doctest_ok_ = false;                                                     \
        try {                                                                         \
            (void)(expr);                                                             \
        } catch (const type& e) {                                                     \
            doctest_ok_ = doctest::matches(e.what(), matcher);                        \
        } catch (...) {                                                               \
        }                                                                             \
        doctest::shim::report(doctest_ok_, "throws " #type " with " #matcher ": " #expr, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::shim::run_all(); }
#endif
