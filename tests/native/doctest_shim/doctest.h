// A minimal stand-in for the doctest macros the reference's unit tests use
// (proj/tests/test_*.cpp: TEST_CASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// CHECK_NOTHROW, CAPTURE, doctest::Approx).  The real doctest.h is vendored
// in the reference's gitignored vendor/ and is absent here.
// Written for this repository: a registry of test functions, per-check
// failure reporting, and a main() when DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN is
// defined.  `reference_unit_tests [substring]` runs the cases whose names
// contain the substring; the exit code is the number of failed cases.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
  public:
    explicit Approx(double value) : value_(value) {}
    Approx& epsilon(double e) {
        epsilon_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    // doctest's rule: |lhs - value| < epsilon * (scale + max(|lhs|, |value|))
    friend bool operator==(double lhs, const Approx& rhs) {
        return std::fabs(lhs - rhs.value_) <
               rhs.epsilon_ * (rhs.scale_ + std::max(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

  private:
    double value_;
    double epsilon_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

namespace shim {

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
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireFailed {};

inline int& case_failures() {
    static int n = 0;
    return n;
}

inline void report(const char* file, int line, const char* what, const char* expr) {
    ++case_failures();
    std::printf("    %s:%d: %s failed: %s\n", file, line, what, expr);
}

}  // namespace shim
}  // namespace doctest

#define DOCTEST_SHIM_CAT2(a, b) a##b
#define DOCTEST_SHIM_CAT(a, b) DOCTEST_SHIM_CAT2(a, b)
#define DOCTEST_SHIM_CASE(fn, name)                                                       \
    static void fn();                                                                     \
    static ::doctest::shim::Registrar DOCTEST_SHIM_CAT(fn, _reg)(name, __FILE__, __LINE__, \
                                                                 &fn);                    \
    static void fn()
#define TEST_CASE(name) DOCTEST_SHIM_CASE(DOCTEST_SHIM_CAT(doctest_shim_case_, __COUNTER__), name)

#define CHECK(...)                                                                     \
    do {                                                                               \
        try {                                                                          \
            if (!static_cast<bool>(__VA_ARGS__))                                       \
                ::doctest::shim::report(__FILE__, __LINE__, "CHECK", #__VA_ARGS__);     \
        } catch (const std::exception& e_) {                                           \
            ::doctest::shim::report(__FILE__, __LINE__, "CHECK threw", e_.what());      \
        }                                                                              \
    } while (0)
#define REQUIRE(...)                                                                   \
    do {                                                                               \
        if (!static_cast<bool>(__VA_ARGS__)) {                                         \
            ::doctest::shim::report(__FILE__, __LINE__, "REQUIRE", #__VA_ARGS__);       \
            throw ::doctest::shim::RequireFailed{};                                    \
        }                                                                              \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                                                    \
    do {                                                                               \
        bool caught_ = false;                                                          \
        try {                                                                          \
            (void)(expr);                                                              \
        } catch (const type&) {                                                        \
            caught_ = true;                                                            \
        } catch (...) {                                                                \
        }                                                                              \
        if (!caught_)                                                                  \
            ::doctest::shim::report(__FILE__, __LINE__, "CHECK_THROWS_AS(" #type ")", #expr); \
    } while (0)
#define CHECK_NOTHROW(...)                                                             \
    do {                                                                               \
        try {                                                                          \
            (void)(__VA_ARGS__);                                                       \
        } catch (...) {                                                                \
            ::doctest::shim::report(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__); \
        }                                                                              \
    } while (0)
#define CAPTURE(x) ((void)0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : "";
    int cases = 0, failed = 0;
    for (const auto& c : ::doctest::shim::registry()) {
        if (*filter && !std::strstr(c.name, filter)) continue;
        ++cases;
        ::doctest::shim::case_failures() = 0;
        try {
            c.fn();
        } catch (const ::doctest::shim::RequireFailed&) {
        } catch (const std::exception& e) {
            ::doctest::shim::report(c.file, c.line, "test case threw", e.what());
        } catch (...) {
            ::doctest::shim::report(c.file, c.line, "test case threw", "unknown exception");
        }
        const bool ok = ::doctest::shim::case_failures() == 0;
        failed += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", c.name);
        std::fflush(stdout);
    }
    std::printf("%d test cases: %d passed, %d failed\n", cases, cases - failed, failed);
    return failed;
}
#endif
