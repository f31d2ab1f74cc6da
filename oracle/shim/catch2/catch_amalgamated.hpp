// ORACLE TEST INFRASTRUCTURE — not product code.
// Minimal Catch2-v3-compatible surface so the reference's own unit tests
// (proj/tests/*.cpp, which `#include <catch2/catch_amalgamated.hpp>` per
// proj/tests/CMakeLists.txt:1-3) build and run unmodified in this container.
// Supported: TEST_CASE, SECTION (flat and nested, re-run-per-leaf semantics),
// CHECK, REQUIRE, CHECK_THROWS_AS, CAPTURE, FAIL, Catch::Approx (epsilon/margin).
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace qps_catch {

struct TestCase {
    std::string name;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct State {
    int checks = 0, failures = 0;
    std::string current;
    std::set<std::string> sections_done;
    bool entered = false, skipped = false;
    std::vector<std::string> captured;
};
inline State& st() {
    static State s;
    return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
    auto& s = st();
    ++s.checks;
    if (ok) return;
    ++s.failures;
    std::fprintf(stderr, "%s:%d: FAILED %s( %s ) in \"%s\"\n", file, line, fatal ? "REQUIRE" : "CHECK", expr,
                 s.current.c_str());
    for (const auto& c : s.captured) std::fprintf(stderr, "    with %s\n", c.c_str());
    if (fatal) throw RequireFailed{};
}

inline bool section_enter(const std::string& name) {
    auto& s = st();
    if (s.entered) {
        if (!s.sections_done.count(name)) s.skipped = true;
        return false;
    }
    if (s.sections_done.count(name)) return false;
    s.sections_done.insert(name);
    s.entered = true;
    return true;
}

struct SectionGuard {
    bool active;
    explicit SectionGuard(const char* name) : active(section_enter(name)) {}
    explicit operator bool() const { return active; }
};

template <class... T>
inline void capture(const char* names, const T&... v) {
    std::ostringstream os;
    os << names << " := ";
    int i = 0;
    ((os << (i++ ? ", " : "") << v), ...);
    st().captured.push_back(os.str());
}

inline int run_all() {
    auto& s = st();
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        s.current = tc.name;
        s.sections_done.clear();
        const int before = s.failures;
        for (int pass = 0; pass < 64; ++pass) {
            s.entered = false;
            s.skipped = false;
            s.captured.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "FAILED: unexpected exception in \"%s\": %s\n", tc.name.c_str(), e.what());
            } catch (...) {
                ++s.failures;
                std::fprintf(stderr, "FAILED: unknown exception in \"%s\"\n", tc.name.c_str());
            }
            if (!s.skipped) break;
        }
        if (s.failures != before) ++failed_cases;
        std::fprintf(stderr, "[%s] %s\n", s.failures == before ? "PASS" : "FAIL", tc.name.c_str());
    }
    std::fprintf(stderr, "%zu test cases, %d failed; %d checks, %d failed\n", registry().size(), failed_cases,
                 s.checks, s.failures);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace qps_catch

namespace Catch {
class Approx {
public:
    explicit Approx(double v)
        : value_(v), eps_(std::numeric_limits<float>::epsilon() * 100.0), margin_(0.0), scale_(0.0) {}
    Approx& epsilon(double e) { eps_ = e; return *this; }
    Approx& margin(double m) { margin_ = m; return *this; }
    Approx& scale(double s) { scale_ = s; return *this; }
    bool matches(double other) const {
        auto mc = [](double a, double b, double m) { return (a + m >= b) && (b + m >= a); };
        return mc(value_, other, margin_) ||
               mc(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    friend bool operator==(double o, const Approx& a) { return a.matches(o); }
    friend bool operator==(const Approx& a, double o) { return a.matches(o); }
    friend bool operator!=(double o, const Approx& a) { return !a.matches(o); }
    friend bool operator!=(const Approx& a, double o) { return !a.matches(o); }

private:
    double value_, eps_, margin_, scale_;
};
}  // namespace Catch

#define QPS_CAT2(a, b) a##b
#define QPS_CAT(a, b) QPS_CAT2(a, b)
#define QPS_TEST_CASE_IMPL(fn, name)                                     \
    static void fn();                                                    \
    static qps_catch::Registrar QPS_CAT(fn, _reg)(name, &fn);            \
    static void fn()
#define TEST_CASE(name, ...) QPS_TEST_CASE_IMPL(QPS_CAT(qps_test_fn_, __LINE__), name)
#define SECTION(name) if (qps_catch::SectionGuard QPS_CAT(qps_sec_, __LINE__){name})
#define CHECK(...) qps_catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) qps_catch::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                        \
    do {                                                                                   \
        bool qps_ok = false;                                                               \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const type&) {                                                            \
            qps_ok = true;                                                                 \
        } catch (...) {                                                                    \
        }                                                                                  \
        qps_catch::report(qps_ok, #expr " throws " #type, __FILE__, __LINE__, false);      \
    } while (0)
#define CAPTURE(...) qps_catch::capture(#__VA_ARGS__, __VA_ARGS__)
#define FAIL(msg) qps_catch::report(false, msg, __FILE__, __LINE__, true)

#ifndef QPS_CATCH_NO_MAIN
int main() { return qps_catch::run_all(); }
#endif
