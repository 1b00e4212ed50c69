// Minimal stand-in for the doctest single header (absent from the reference tree:
// /root/reference/proj/.gitignore:2 ignores vendor/). Supports exactly the macros the
// reference unit tests use: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS, FAIL and
// doctest::Approx(...).epsilon(...). Test infrastructure only (oracle build).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    friend bool operator==(double lhs, const Approx& rhs) {
        const double scale = std::max(std::fabs(lhs), std::fabs(rhs.value_));
        return std::fabs(lhs - rhs.value_) < rhs.eps_ * (1.0 + scale);
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-07 * 100;  // doctest's default: float eps * 100
};

namespace detail {
struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failed_checks() {
    static int n = 0;
    return n;
}
inline int& total_checks() {
    static int n = 0;
    return n;
}
inline void note(bool ok, const char* expr, const char* file, int line, bool fatal) {
    ++total_checks();
    if (ok) return;
    ++failed_checks();
    std::printf("%s:%d: FAILED: %s\n", file, line, expr);
    if (fatal) throw RequireFailed{};
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                         \
    static void fn();                                                                     \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                   \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)
#define CHECK(...) doctest::detail::note(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::note(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define FAIL(msg) doctest::detail::note(false, msg, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                       \
    do {                                                                                  \
        bool caught_ = false;                                                             \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const type&) {                                                           \
            caught_ = true;                                                               \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest::detail::note(caught_, "throws " #type ": " #expr, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& c : doctest::detail::registry()) {
        const int before = doctest::detail::failed_checks();
        try {
            c.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failed_checks();
            std::printf("test case '%s' threw: %s\n", c.name, e.what());
        }
        if (doctest::detail::failed_checks() != before) {
            ++failed_cases;
            std::printf("FAILED test case: %s\n", c.name);
        }
    }
    std::printf("[doctest-shim] test cases: %zu | %d failed | checks: %d | %d failed\n",
                doctest::detail::registry().size(), failed_cases, doctest::detail::total_checks(),
                doctest::detail::failed_checks());
    return failed_cases == 0 ? 0 : 1;
}
#endif
