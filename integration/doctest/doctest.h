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

#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <execinfo.h>
#include <sys/wait.h>
#include <unistd.h>
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

// Verbose runs print a raw backtrace on a crash (addresses resolve with
// addr2line against the -g build).
inline void crash_handler(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    const char msg[] = "[doctest] fatal signal, backtrace:\n";
    (void)!write(2, msg, sizeof msg - 1);
    backtrace_symbols_fd(frames, n, 2);
    std::signal(sig, SIG_DFL);
    std::raise(sig);
}

// Runs one test case in this process; returns true when it passed.
inline bool run_case(const TestCase& t) {
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
    return !state().case_failed;
}

// DOCTEST_MINI_FORK=1: every test case runs in a child process, so a crash
// inside one case (the reference's random-program generator indexes an
// empty vector on this toolchain's RNG stream, P/tests/engine_test.cpp:83)
// is reported as that case's failure and the others still run. Each case
// prints one "[doctest] case: <status> <assertions> <name>" line (status ok /
// failed / crashed(signal)). The child's assertion counts come back through a pipe.
inline int run_all() {
    long passed = 0, failed = 0;
    const bool verbose = std::getenv("DOCTEST_MINI_VERBOSE") != nullptr;
    const bool fork_each = std::getenv("DOCTEST_MINI_FORK") != nullptr;
    if (verbose) {
        std::signal(SIGSEGV, crash_handler);
        std::signal(SIGABRT, crash_handler);
    }
    for (const TestCase& t : registry()) {
        if (verbose) std::fprintf(stderr, "[doctest] running \"%s\"\n", t.name);
        std::string status;
        const long before = state().asserts, failed_before = state().failed_asserts;
        if (fork_each) {
            std::fflush(stdout);
            std::fflush(stderr);
            int fd[2];
            if (pipe(fd) != 0) return 255;
            const pid_t pid = fork();
            if (pid == 0) {
                close(fd[0]);
                const bool ok = run_case(t);
                long counts[2] = {state().asserts - before, state().failed_asserts - failed_before};
                (void)!write(fd[1], counts, sizeof counts);
                std::fflush(stdout);
                std::fflush(stderr);
                _exit(ok ? 0 : 1);
            }
            close(fd[1]);
            long counts[2] = {0, 0};
            const bool got = read(fd[0], counts, sizeof counts) == static_cast<ssize_t>(sizeof counts);
            close(fd[0]);
            int ws = 0;
            waitpid(pid, &ws, 0);
            state().asserts += counts[0];
            state().failed_asserts += counts[1];
            if (WIFSIGNALED(ws) || !got) status = "crashed(" + std::to_string(WIFSIGNALED(ws) ? WTERMSIG(ws) : 0) + ")";
            else status = WEXITSTATUS(ws) == 0 ? "ok" : "failed";
        } else {
            status = run_case(t) ? "ok" : "failed";
        }
        std::printf("[doctest] case: %s %ld %s\n", status.c_str(), state().asserts - before, t.name);
        if (status == "ok") {
            ++passed;
        } else {
            ++failed;
            std::fprintf(stderr, "  in TEST CASE \"%s\"\n", t.name);
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
