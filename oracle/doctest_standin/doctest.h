// Minimal stand-in for doctest (absent from /root/reference/proj/vendor) —
// TEST INFRASTRUCTURE ONLY. Enough of its macro surface to build the
// reference's own unit suites unchanged (oracle/Makefile `ref-suites`):
// TEST_SUITE, TEST_CASE, SUBCASE (run in sequence), CHECK, REQUIRE,
// CHECK_MESSAGE, CHECK_THROWS_AS, FAIL.
#pragma once

#include <cstdio>
#include <exception>
#include <vector>

namespace doctest_standin {

struct Case {
    const char* name;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Register {
    Register(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};
struct Stats {
    long checks = 0, failed = 0;
};
inline Stats& stats() {
    static Stats s;
    return s;
}
struct RequireFailed {};
inline void check(bool ok, const char* expr, const char* file, int line, bool require) {
    ++stats().checks;
    if (ok) return;
    ++stats().failed;
    std::fprintf(stderr, "%s:%d: %s(%s) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireFailed{};
}
inline int run_all() {
    int bad_cases = 0;
    for (const Case& c : registry()) {
        const long before = stats().failed;
        try {
            c.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            ++stats().failed;
            std::fprintf(stderr, "test case \"%s\": exception: %s\n", c.name, e.what());
        }
        if (stats().failed != before) {
            ++bad_cases;
            std::fprintf(stderr, "FAILED test case: %s\n", c.name);
        }
    }
    std::printf("[doctest stand-in] test cases: %zu | %zu passed | %d failed; checks: %ld | %ld failed\n",
                registry().size(), registry().size() - static_cast<std::size_t>(bad_cases), bad_cases, stats().checks,
                stats().failed);
    return bad_cases ? 1 : 0;
}

}  // namespace doctest_standin

namespace doctest {
/// Approximate floating-point comparison (relative epsilon, as doctest's default).
class Approx {
public:
    explicit Approx(double v) : v_(v) {}
    friend bool operator==(double x, const Approx& a) {
        const double scale = (x < 0 ? -x : x) > (a.v_ < 0 ? -a.v_ : a.v_) ? (x < 0 ? -x : x) : (a.v_ < 0 ? -a.v_ : a.v_);
        const double d = x - a.v_;
        return (d < 0 ? -d : d) <= 1.1920929e-7f * 100 * (scale + 1.0);
    }
    friend bool operator==(const Approx& a, double x) { return x == a; }

private:
    double v_;
};
}  // namespace doctest

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_SUITE(name) namespace
#define DS_CASE(fn, name)                                                      \
    static void fn();                                                          \
    static const doctest_standin::Register DS_CAT(fn, _reg)(name, &fn);        \
    static void fn()
#define TEST_CASE(name) DS_CASE(DS_CAT(ds_case_, __COUNTER__), name)
#define SUBCASE(name) if (true)
#define CHECK(...) doctest_standin::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_standin::check(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_MESSAGE(cond, msg) CHECK(cond)
#define FAIL(msg) doctest_standin::check(false, "FAIL", __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                            \
    do {                                                                       \
        bool ds_thrown = false;                                                \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const type&) {                                                \
            ds_thrown = true;                                                  \
        } catch (...) {                                                        \
        }                                                                      \
        doctest_standin::check(ds_thrown, #expr " throws " #type, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_standin::run_all(); }
#endif
