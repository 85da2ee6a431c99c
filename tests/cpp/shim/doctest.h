// Minimal doctest-compatible test harness (own code). Implements just the
// macros the reference's unit suites use, so proj/tests/token_tree_test.cpp and
// proj/tests/transformer_test.cpp compile UNCHANGED against this repository's
// drop-in library (doctest itself is absent from the image; the reference's
// vendor/ directory is gitignored, proj/.gitignore:2).
//
// SUBCASE blocks run once, in order, inside a single execution of their test
// case (the reference suites only use independent subcases).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

namespace doctest_shim {

struct TestCase {
    const char* name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Reg {
    Reg(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline int& failures() {
    static int f = 0;
    return f;
}
inline int& checks() {
    static int c = 0;
    return c;
}

struct RequireFailed {};

inline void report(const char* file, int line, const std::string& what) {
    std::printf("  FAILED %s:%d: %s\n", file, line, what.c_str());
    ++failures();
}

inline bool check(bool ok, const char* file, int line, const char* expr) {
    ++checks();
    if (!ok) report(file, line, std::string("CHECK(") + expr + ")");
    return ok;
}

}  // namespace doctest_shim

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        const double m = std::fmax(std::fabs(lhs), std::fabs(a.value_));
        return std::fabs(lhs - a.value_) < a.eps_ * (1.0 + m);
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }

private:
    double value_;
    double eps_ = 1.1920929e-07f * 100;
};

struct Contains {
    explicit Contains(const char* s) : needle(s) {}
    std::string needle;
    bool matches(const std::string& hay) const { return hay.find(needle) != std::string::npos; }
};

}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)

#define TEST_CASE(name)                                                                   \
    static void DS_CAT(ds_test_fn_, __LINE__)();                                          \
    static doctest_shim::Reg DS_CAT(ds_test_reg_, __LINE__)(name, DS_CAT(ds_test_fn_, __LINE__)); \
    static void DS_CAT(ds_test_fn_, __LINE__)()

#define SUBCASE(name) if (true)

#define CHECK(...) doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define REQUIRE(...)                                                                      \
    do {                                                                                  \
        if (!doctest_shim::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)) \
            throw doctest_shim::RequireFailed{};                                          \
    } while (0)
#define FAIL(msg)                                                                         \
    do {                                                                                  \
        std::ostringstream ds_os_;                                                        \
        ds_os_ << msg;                                                                    \
        doctest_shim::report(__FILE__, __LINE__, "FAIL: " + ds_os_.str());               \
        throw doctest_shim::RequireFailed{};                                              \
    } while (0)
#define MESSAGE(msg)                                                                      \
    do {                                                                                  \
        std::ostringstream ds_os_;                                                        \
        ds_os_ << msg;                                                                    \
        std::printf("  MESSAGE %s\n", ds_os_.str().c_str());                              \
    } while (0)
#define CHECK_THROWS_AS(expr, Type)                                                       \
    do {                                                                                  \
        bool ds_ok_ = false;                                                              \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const Type&) {                                                           \
            ds_ok_ = true;                                                                \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest_shim::check(ds_ok_, __FILE__, __LINE__, "THROWS_AS(" #expr ", " #Type ")"); \
    } while (0)
#define CHECK_THROWS_WITH_AS(expr, matcher, Type)                                         \
    do {                                                                                  \
        bool ds_ok_ = false;                                                              \
        try {                                                                             \
            (void)(expr);                                                                 \
        } catch (const Type& ds_e_) {                                                     \
            ds_ok_ = (matcher).matches(ds_e_.what());                                     \
        } catch (...) {                                                                   \
        }                                                                                 \
        doctest_shim::check(ds_ok_, __FILE__, __LINE__, "THROWS_WITH_AS(" #expr ")");      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    int failed_cases = 0;
    for (const auto& tc : doctest_shim::registry()) {
        const int before = doctest_shim::failures();
        try {
            tc.fn();
        } catch (const doctest_shim::RequireFailed&) {
        } catch (const std::exception& e) {
            doctest_shim::report("<exception>", 0, std::string(tc.name) + ": " + e.what());
        } catch (...) {
            doctest_shim::report("<exception>", 0, std::string(tc.name) + ": unknown exception");
        }
        const bool ok = doctest_shim::failures() == before;
        failed_cases += !ok;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
    }
    std::printf("test cases: %zu | passed: %zu | failed: %d | assertions: %d | failed assertions: %d\n",
                doctest_shim::registry().size(), doctest_shim::registry().size() - failed_cases,
                failed_cases, doctest_shim::checks(), doctest_shim::failures());
    return failed_cases == 0 ? 0 : 1;
}
#endif
