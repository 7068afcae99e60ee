// Minimal Catch2-API shim (test infrastructure). Catch2 is absent from this
// image (reference: tests/CMakeLists.txt:1-2). The reference's unit tests use
// only TEST_CASE, single-level SECTION, CHECK/REQUIRE(_FALSE),
// CHECK_THROWS_AS, FAIL and Catch::Approx(x).epsilon(e).margin(m)
// (SURVEY §4); this header implements exactly that surface so the UNMODIFIED
// test sources compile against the drop-in headers (and against the oracle).
// A TEST_CASE body is re-run once per SECTION, each run executing one section.
#ifndef CATCH_SHIM_AMALGAMATED_HPP
#define CATCH_SHIM_AMALGAMATED_HPP

#include <cmath>
#include <cstdio>
#include <exception>
#include <limits>
#include <string>
#include <vector>

namespace Catch {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& margin(double m) {
        margin_ = m;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double other) const {
        auto within = [](double a, double b, double m) { return a + m >= b && b + m >= a; };
        return within(value_, other, margin_) ||
               within(value_, other, eps_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_)));
    }
    friend bool operator==(double lhs, const Approx& rhs) { return rhs.matches(lhs); }
    friend bool operator==(const Approx& lhs, double rhs) { return lhs.matches(rhs); }
    friend bool operator!=(double lhs, const Approx& rhs) { return !rhs.matches(lhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !lhs.matches(rhs); }
    friend bool operator<=(double lhs, const Approx& rhs) { return lhs < rhs.value_ || rhs.matches(lhs); }
    friend bool operator>=(double lhs, const Approx& rhs) { return lhs > rhs.value_ || rhs.matches(lhs); }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double margin_ = 0.0;
    double scale_ = 0.0;
};

}  // namespace Catch

namespace catchshim {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};
inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, void (*f)(), const char* file, int line) { registry().push_back({n, f, file, line}); }
};
struct State {
    int target = 0, seen = 0;
    long checks = 0, failed_checks = 0;
    bool test_failed = false;
    std::string section;
};
inline State& state() {
    static State s;
    return s;
}
struct RequireAbort {};

inline bool enter_section(const char* name) {
    State& s = state();
    const int id = s.seen++;
    if (id != s.target) return false;
    s.section = name;
    return true;
}
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    State& s = state();
    ++s.checks;
    if (ok) return;
    ++s.failed_checks;
    s.test_failed = true;
    std::printf("    FAILED %s:%d%s%s: %s\n", file, line, s.section.empty() ? "" : " in section ",
                s.section.c_str(), expr);
    if (require) throw RequireAbort{};
}

inline int run_all() {
    int failed = 0, passed = 0;
    for (const TestCase& t : registry()) {
        State& s = state();
        s.target = 0;
        s.test_failed = false;
        for (;;) {
            s.seen = 0;
            s.section.clear();
            try {
                t.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                s.test_failed = true;
                std::printf("    FAILED %s: unexpected exception in section '%s': %s\n", t.name, s.section.c_str(),
                            e.what());
            } catch (...) {
                s.test_failed = true;
                std::printf("    FAILED %s: unknown exception\n", t.name);
            }
            if (s.seen == 0 || ++s.target >= s.seen) break;
        }
        std::printf("[%s] %s\n", s.test_failed ? "FAIL" : "PASS", t.name);
        (s.test_failed ? failed : passed)++;
    }
    std::printf("test cases: %d passed, %d failed; checks: %ld, failed checks: %ld\n", passed, failed,
                state().checks, state().failed_checks);
    return failed;
}

}  // namespace catchshim

#define CATCHSHIM_CAT2(a, b) a##b
#define CATCHSHIM_CAT(a, b) CATCHSHIM_CAT2(a, b)
#define CATCHSHIM_TC(fn, reg, name)                                     \
    static void fn();                                                   \
    static catchshim::Registrar reg(name, &fn, __FILE__, __LINE__);     \
    static void fn()
#define TEST_CASE(name, ...) \
    CATCHSHIM_TC(CATCHSHIM_CAT(catchshim_fn_, __LINE__), CATCHSHIM_CAT(catchshim_reg_, __LINE__), name)
#define SECTION(name, ...) if (catchshim::enter_section(name))
#define CHECK(...) catchshim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) catchshim::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_FALSE(...) catchshim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE_FALSE(...) catchshim::check(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, true)
#define CATCHSHIM_THROWS(expr, type, req)                                                   \
    do {                                                                                    \
        bool catchshim_ok_ = false;                                                         \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const type&) {                                                             \
            catchshim_ok_ = true;                                                           \
        } catch (...) {                                                                     \
        }                                                                                   \
        catchshim::check(catchshim_ok_, #expr " throws " #type, __FILE__, __LINE__, req);   \
    } while (0)
#define CHECK_THROWS_AS(expr, type) CATCHSHIM_THROWS(expr, type, false)
#define REQUIRE_THROWS_AS(expr, type) CATCHSHIM_THROWS(expr, type, true)
#define FAIL(msg) catchshim::check(false, msg, __FILE__, __LINE__, true)

#endif
