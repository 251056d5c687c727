// TEST INFRASTRUCTURE ONLY — the subset of the doctest API the reference's
// unit tests use (TEST_SUITE_BEGIN/END, TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS, doctest::Approx), restated so that
// /root/reference/proj/tests/test_*.cpp compile unmodified against the
// Eigen-API shim into oracle/_ref/ref_unit_tests (doctest itself is absent:
// SURVEY.md §0.1, proj/.gitignore:2). Approx follows doctest 2.4's
// definition: |a - b| < eps * (scale + max(|a|, |b|)), scale 1, default eps
// 100 * FLT_EPSILON.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double a, const Approx& b) {
        return std::fabs(a - b.v_) < b.eps_ * (b.scale_ + std::fmax(std::fabs(a), std::fabs(b.v_)));
    }
    friend bool operator==(const Approx& b, double a) { return a == b; }
    friend bool operator!=(double a, const Approx& b) { return !(a == b); }
    double value() const { return v_; }

private:
    double v_;
    double eps_ = 100.0 * double(FLT_EPSILON);
    double scale_ = 1.0;
};

namespace detail {
struct TestCase {
    const char* suite;
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
inline const char*& current_suite() {
    static const char* s = "";
    return s;
}
inline int set_suite(const char* s) {
    current_suite() = s;
    return 0;
}
inline int add(const char* name, void (*fn)(), const char* file, int line) {
    registry().push_back({current_suite(), name, fn, file, line});
    return 0;
}
struct Counters {
    long checks = 0, failed = 0;
};
inline Counters& counters() {
    static Counters c;
    return c;
}
struct RequireFailure {};
inline bool check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++counters().checks;
    if (!ok) {
        ++counters().failed;
        std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
        if (require) throw RequireFailure{};
    }
    return ok;
}
}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define TEST_SUITE_BEGIN(name) \
    static const int DOCTEST_CAT(doctest_suite_, __LINE__) = doctest::detail::set_suite(name)
#define TEST_SUITE_END() static const int DOCTEST_CAT(doctest_suite_end_, __LINE__) = doctest::detail::set_suite("")
#define DOCTEST_TEST_CASE_IMPL(f, name)                                                                  \
    static void f();                                                                                     \
    static const int DOCTEST_CAT(f, _reg) = doctest::detail::add(name, &f, __FILE__, __LINE__); \
    static void f()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_test_, __COUNTER__), name)
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) doctest::detail::check(!(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                                      \
    do {                                                                                                 \
        bool doctest_ok_ = false;                                                                        \
        try {                                                                                            \
            expr;                                                                                        \
        } catch (const type&) {                                                                          \
            doctest_ok_ = true;                                                                          \
        } catch (...) {                                                                                  \
        }                                                                                                \
        doctest::detail::check(doctest_ok_, #expr " throws " #type, __FILE__, __LINE__, false);          \
    } while (0)
#define CHECK_NOTHROW(expr)                                                                              \
    do {                                                                                                 \
        bool doctest_ok_ = true;                                                                         \
        try {                                                                                            \
            expr;                                                                                        \
        } catch (...) {                                                                                  \
            doctest_ok_ = false;                                                                         \
        }                                                                                                \
        doctest::detail::check(doctest_ok_, #expr " does not throw", __FILE__, __LINE__, false);         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
/// Runs every registered case (optionally only those whose "suite/name"
/// contains argv[1]); prints one line per case and a summary; exit code 1 on
/// any failure.
int main(int argc, char** argv) {
    using namespace doctest::detail;
    const char* filt = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    for (const TestCase& tc : registry()) {
        std::string full = std::string(tc.suite) + "/" + tc.name;
        if (filt && full.find(filt) == std::string::npos) continue;
        ++cases;
        const long before = counters().failed;
        bool threw = false;
        try {
            tc.fn();
        } catch (const RequireFailure&) {
        } catch (const std::exception& e) {
            threw = true;
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
        }
        const bool ok = !threw && counters().failed == before;
        if (!ok) ++failed_cases;
        std::printf("[%s] %s\n", ok ? "pass" : "FAIL", full.c_str());
    }
    std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", cases,
                cases - failed_cases, failed_cases, counters().checks, counters().failed);
    return failed_cases ? 1 : 0;
}
#endif
