// TEST INFRASTRUCTURE — a minimal stand-in for the doctest header (doctest
// is not installed in this image and there is no network). It implements
// only what the reference's suites use: TEST_CASE, CHECK, REQUIRE,
// CHECK_THROWS_AS (P/tests/{column,relation,kernels,engine}_test.cpp), so
// those files compile UNMODIFIED against the drop-in library
// (integration/colog_fvlog) and run their own assertions against the GPU.
//
// Semantics follow doctest's: a failed CHECK records the failure and goes
// on, a failed REQUIRE ends the test case, an exception escaping a test case
// fails it. The process exit code is the number of failed test cases
// (capped at 255), and one summary line is printed:
//   [doctest] test cases: N | N passed | 0 failed | assertions: A | A passed | 0 failed
#pragma once

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

namespace doctest_mini {

struct TestCase {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};

inline std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}

struct State {
    long asserts = 0, failed_asserts = 0;
    bool case_failed = false;
};

inline State& state() {
    static State s;
    return s;
}

struct RequireAbort {};

inline int add(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
    return 0;
}

inline void report(bool ok, bool require, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    s.case_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED\n", file, line, require ? "REQUIRE" : "CHECK", expr);
    if (require) throw RequireAbort{};
}

inline int run_all() {
    long passed = 0, failed = 0;
    for (const TestCase& t : registry()) {
        state().case_failed = false;
        try {
            t.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw: %s\n", t.file, t.line, t.name, e.what());
            state().case_failed = true;
        } catch (...) {
            std::fprintf(stderr, "%s:%d: TEST CASE \"%s\" threw an unknown exception\n", t.file, t.line, t.name);
            state().case_failed = true;
        }
        if (state().case_failed) {
            ++failed;
            std::fprintf(stderr, "  in TEST CASE \"%s\"\n", t.name);
        } else {
            ++passed;
        }
    }
    const State& s = state();
    std::printf("[doctest] test cases: %ld | %ld passed | %ld failed | assertions: %ld | %ld passed | %ld failed\n",
                passed + failed, passed, failed, s.asserts, s.asserts - s.failed_asserts, s.failed_asserts);
    return failed > 255 ? 255 : static_cast<int>(failed);
}

}  // namespace doctest_mini

#define DOCTEST_MINI_CAT2(a, b) a##b
#define DOCTEST_MINI_CAT(a, b) DOCTEST_MINI_CAT2(a, b)
#define DOCTEST_MINI_TC(fn, name)                                                                     \
    static void fn();                                                                                 \
    static const int DOCTEST_MINI_CAT(fn, _reg) = doctest_mini::add(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_MINI_TC(DOCTEST_MINI_CAT(doctest_mini_case_, __COUNTER__), name)

#define CHECK(...) doctest_mini::report(static_cast<bool>(__VA_ARGS__), false, #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...) doctest_mini::report(static_cast<bool>(__VA_ARGS__), true, #__VA_ARGS__, __FILE__, __LINE__)
#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        bool doctest_mini_ok = false;                                                              \
        try {                                                                                      \
            expr;                                                                                  \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_mini_ok = true;                                                                \
        } catch (...) {                                                                            \
        }                                                                                          \
        doctest_mini::report(doctest_mini_ok, false, #expr " throws " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest_mini::run_all(); }
#endif
