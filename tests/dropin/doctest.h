// TEST INFRASTRUCTURE ONLY -- a minimal stand-in for the doctest header the
// reference's unit tests include (doctest itself is not in this image). It
// implements exactly the subset those files use (TEST_SUITE_BEGIN/END,
// TEST_CASE, CHECK, CHECK_FALSE, REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS,
// CHECK_THROWS_WITH_AS, doctest::Approx, doctest::Contains), so the
// UNMODIFIED reference test sources compile against the B200 drop-in
// headers (tests/dropin/Makefile).
//
//   <binary> [--tc-exclude=substr1,...] [--test-case=substr1,...] [--test-suite=name]
// exit code: number of failed test cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <string>
#include <vector>

namespace doctest {

struct Approx {
    double value, eps = std::numeric_limits<float>::epsilon() * 100, scale = 1.0;
    explicit Approx(double v) : value(v) {}
    Approx& epsilon(double e) {
        eps = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value) < a.eps * (a.scale + std::max(std::fabs(lhs), std::fabs(a.value)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
};

struct Contains {
    std::string needle;
    explicit Contains(const char* s) : needle(s) {}
    bool match(const std::string& s) const { return s.find(needle) != std::string::npos; }
};

namespace detail {
struct Case {
    const char* name;
    const char* suite;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
inline const char*& current_suite() {
    static const char* s = "";
    return s;
}
struct Reg {
    Reg(const char* name, const char* suite, void (*fn)()) { registry().push_back({name, suite, fn}); }
};
struct SuiteSet {
    explicit SuiteSet(const char* s) { current_suite() = s; }
};
struct Abort {};
inline int& failures() {
    static int f = 0;
    return f;
}
inline void fail(const char* file, int line, const char* what) {
    ++failures();
    std::fprintf(stderr, "%s:%d: FAILED: %s\n", file, line, what);
}
inline bool matches(const std::string& what, const char* s) { return what == s; }
inline bool matches(const std::string& what, const Contains& c) { return c.match(what); }
}  // namespace detail
}  // namespace doctest

#define DT_CAT2(a, b) a##b
#define DT_CAT(a, b) DT_CAT2(a, b)
#define TEST_SUITE_BEGIN(name) static doctest::detail::SuiteSet DT_CAT(dt_suite_, __LINE__)(name)
#define TEST_SUITE_END() static_assert(true, "")
#define TEST_CASE(name)                                                                                   \
    static void DT_CAT(dt_case_, __LINE__)();                                                             \
    static doctest::detail::Reg DT_CAT(dt_reg_, __LINE__)(name, doctest::detail::current_suite(),         \
                                                          DT_CAT(dt_case_, __LINE__));                    \
    static void DT_CAT(dt_case_, __LINE__)()

#define CHECK(...)                                                                 \
    do {                                                                           \
        if (!(__VA_ARGS__)) doctest::detail::fail(__FILE__, __LINE__, #__VA_ARGS__); \
    } while (0)
#define CHECK_FALSE(...) CHECK(!(__VA_ARGS__))
#define REQUIRE(...)                                                                   \
    do {                                                                               \
        if (!(__VA_ARGS__)) {                                                          \
            doctest::detail::fail(__FILE__, __LINE__, "REQUIRE " #__VA_ARGS__);        \
            throw doctest::detail::Abort{};                                            \
        }                                                                              \
    } while (0)
#define CHECK_NOTHROW(expr)                                                             \
    do {                                                                                \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const std::exception& e) {                                             \
            doctest::detail::fail(__FILE__, __LINE__, (std::string(#expr " threw: ") + e.what()).c_str()); \
        } catch (...) {                                                                 \
            doctest::detail::fail(__FILE__, __LINE__, #expr " threw");                  \
        }                                                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                     \
    do {                                                                                \
        bool dt_ok = false;                                                             \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type&) {                                                         \
            dt_ok = true;                                                               \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!dt_ok) doctest::detail::fail(__FILE__, __LINE__, #expr " did not throw " #type); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, type)                                       \
    do {                                                                                \
        bool dt_ok = false;                                                             \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const type& e) {                                                       \
            dt_ok = doctest::detail::matches(e.what(), matcher);                        \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!dt_ok) doctest::detail::fail(__FILE__, __LINE__, #expr " did not throw " #type " with " #matcher); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    std::vector<std::string> exclude, include;
    std::string suite;
    auto split = [](std::string rest, std::vector<std::string>& out) {
        size_t p;
        while ((p = rest.find(',')) != std::string::npos) {
            out.push_back(rest.substr(0, p));
            rest = rest.substr(p + 1);
        }
        if (!rest.empty()) out.push_back(rest);
    };
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a.rfind("--tc-exclude=", 0) == 0) {
            split(a.substr(13), exclude);
        } else if (a.rfind("--test-case=", 0) == 0) {
            split(a.substr(12), include);
        } else if (a.rfind("--test-suite=", 0) == 0) {
            suite = a.substr(13);
        }
    }
    int ran = 0, failed = 0, skipped = 0;
    for (const auto& c : doctest::detail::registry()) {
        if (!suite.empty() && suite != c.suite) continue;
        const std::string name = c.name;
        if (!include.empty() &&
            std::none_of(include.begin(), include.end(), [&](const std::string& x) { return name.find(x) != std::string::npos; }))
            continue;
        if (std::any_of(exclude.begin(), exclude.end(), [&](const std::string& x) { return name.find(x) != std::string::npos; })) {
            ++skipped;
            std::printf("[skip] %s\n", c.name);
            continue;
        }
        const int before = doctest::detail::failures();
        ++ran;
        try {
            c.fn();
        } catch (const doctest::detail::Abort&) {
        } catch (const std::exception& e) {
            doctest::detail::fail(c.name, 0, (std::string("unexpected exception: ") + e.what()).c_str());
        } catch (...) {
            doctest::detail::fail(c.name, 0, "unexpected exception");
        }
        const bool ok = doctest::detail::failures() == before;
        failed += !ok;
        std::printf("[%s] %s :: %s\n", ok ? " ok " : "FAIL", c.suite, c.name);
    }
    std::printf("test cases: %d run, %d passed, %d failed, %d excluded\n", ran, ran - failed, failed, skipped);
    return failed;
}
#endif
