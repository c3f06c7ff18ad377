// Minimal doctest-compatible test harness (test infrastructure only).
// Written from scratch to run the reference's hot-path test files unmodified
// (SURVEY.md §8c). Supports the subset those files use: TEST_CASE, CHECK,
// REQUIRE, CHECK_THROWS, MESSAGE, INFO and doctest::Approx(v).epsilon(e),
// with doctest's documented Approx rule
//   |a - b| < eps * (scale + max(|a|, |b|)),  eps default = 100*FLT_EPSILON.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.eq(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.eq(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.eq(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.eq(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.eq(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.eq(lhs); }
    double value() const { return value_; }

private:
    bool eq(double v) const {
        return std::fabs(v - value_) <
               eps_ * (scale_ + std::max(std::fabs(v), std::fabs(value_)));
    }
    double value_;
    double eps_ = static_cast<double>(std::numeric_limits<float>::epsilon()) * 100.0;
    double scale_ = 1.0;
};

namespace detail {
struct TestCase {
    const char* name;
    void (*fn)();
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct RequireFailed {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline int& assertions() {
    static int a = 0;
    return a;
}
inline const char*& current() {
    static const char* c = "";
    return c;
}
inline void report(const char* file, int line, const char* expr) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\": %s\n", file, line, current(), expr);
}
template <typename... A>
inline std::string cat(const A&... a) {
    std::ostringstream os;
    (os << ... << a);
    return os.str();
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                       \
    static void fn();                                                                   \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, &fn);                 \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define CHECK(...)                                                                      \
    do {                                                                                \
        ++doctest::detail::assertions();                                                \
        if (!(__VA_ARGS__)) doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);  \
    } while (0)
#define REQUIRE(...)                                                                    \
    do {                                                                                \
        ++doctest::detail::assertions();                                                \
        if (!(__VA_ARGS__)) {                                                           \
            doctest::detail::report(__FILE__, __LINE__, #__VA_ARGS__);                  \
            throw doctest::detail::RequireFailed{};                                     \
        }                                                                               \
    } while (0)
#define CHECK_THROWS(...)                                                               \
    do {                                                                                \
        ++doctest::detail::assertions();                                                \
        bool threw_ = false;                                                            \
        try {                                                                           \
            (void)(__VA_ARGS__);                                                        \
        } catch (...) {                                                                 \
            threw_ = true;                                                              \
        }                                                                               \
        if (!threw_) doctest::detail::report(__FILE__, __LINE__, "throws: " #__VA_ARGS__); \
    } while (0)
#define MESSAGE(...) \
    std::fprintf(stderr, "  [msg] %s\n", doctest::detail::cat(__VA_ARGS__).c_str())
#define INFO(...) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& tc : doctest::detail::registry()) {
        doctest::detail::current() = tc.name;
        const int before = doctest::detail::failures();
        try {
            tc.fn();
        } catch (const doctest::detail::RequireFailed&) {
        } catch (const std::exception& e) {
            ++doctest::detail::failures();
            std::fprintf(stderr, "exception in \"%s\": %s\n", tc.name, e.what());
        }
        if (doctest::detail::failures() != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %d\n",
                doctest::detail::registry().size(),
                doctest::detail::registry().size() - failed_cases, failed_cases,
                doctest::detail::assertions());
    return failed_cases == 0 ? 0 : 1;
}
#endif
