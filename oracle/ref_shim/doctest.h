// Minimal stand-in for the doctest single header, written for this repo.
//
// TEST INFRASTRUCTURE ONLY. The reference's unit test
// (/root/reference/proj/tests/test_ordering.cpp) includes <doctest.h> from a
// gitignored vendor/ directory that is absent (proj/.gitignore:2). This shim
// implements just the macros that test uses (TEST_CASE, CHECK, CHECK_MESSAGE,
// CHECK_THROWS_AS, REQUIRE) so the reference test can be compiled in place and
// run against the reference's own ordering.cpp, pinning oracle/_ref.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

namespace shim {

struct Case {
    const char* name;
    void (*fn)();
};

inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}

struct Counters {
    long asserts = 0;
    long failures = 0;
    int failed_cases = 0;
};

inline Counters& counters() {
    static Counters c;
    return c;
}

struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal, const std::string& msg = "") {
    ++counters().asserts;
    if (ok) return;
    ++counters().failures;
    std::fprintf(stderr, "%s:%d: FAILED: %s %s\n", file, line, expr, msg.c_str());
    if (fatal) throw RequireFailed{};
}

template <typename... Ts>
std::string concat(const Ts&... parts) {
    std::ostringstream os;
    ((os << parts), ...);
    return os.str();
}

}  // namespace shim

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)
#define TEST_CASE(name)                                                                     \
    static void SHIM_CAT(shim_case_, __LINE__)();                                           \
    static shim::Registrar SHIM_CAT(shim_reg_, __LINE__)(name, &SHIM_CAT(shim_case_, __LINE__)); \
    static void SHIM_CAT(shim_case_, __LINE__)()

#define CHECK(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_MESSAGE(expr, ...) \
    shim::report(static_cast<bool>(expr), #expr, __FILE__, __LINE__, false, shim::concat(__VA_ARGS__))
#define CHECK_THROWS_AS(expr, exc)                                          \
    do {                                                                    \
        bool shim_thrown = false;                                           \
        try {                                                               \
            (void)(expr);                                                   \
        } catch (const exc&) {                                              \
            shim_thrown = true;                                             \
        } catch (...) {                                                     \
        }                                                                   \
        shim::report(shim_thrown, #expr " throws " #exc, __FILE__, __LINE__, false); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() {
    for (const auto& c : shim::registry()) {
        long before = shim::counters().failures;
        try {
            c.fn();
        } catch (const shim::RequireFailed&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "test case '%s' threw: %s\n", c.name, e.what());
            ++shim::counters().failures;
        }
        if (shim::counters().failures != before) ++shim::counters().failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed | assertions: %ld | %ld failed\n",
                shim::registry().size(), shim::registry().size() - shim::counters().failed_cases,
                shim::counters().failed_cases, shim::counters().asserts, shim::counters().failures);
    return shim::counters().failures == 0 ? 0 : 1;
}
#endif
