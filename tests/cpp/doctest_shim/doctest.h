// Minimal doctest-compatible test shim (TEST INFRASTRUCTURE).
//
// The reference's unit tests (/root/reference/proj/tests/test_*.cpp) are
// written against doctest, which is not in this image.  This header provides
// the subset they use — TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS_AS,
// doctest::Approx with .epsilon()/.scale(), DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN —
// with doctest's semantics, so those files compile UNCHANGED against
// include/rank1/ and run on the B200 library (tests/test_reference_unit_cpp.py).
//
// Semantics kept from doctest:
//  * Approx(v): |lhs - v| < eps * (scale + max(|lhs|, |v|)), eps defaults to
//    100 * FLT_EPSILON, scale to 1.
//  * CHECK records a failure and continues; REQUIRE aborts the test case.
//  * SUBCASE: the test case body is re-run once per leaf subcase; each run
//    enters exactly one subcase not yet run (code outside subcases runs each time).
//  * An exception escaping a test case fails it.
//  * Command line: -tc=<globs> / --test-case=<globs> (comma separated, '*'
//    wildcard) selects test cases, -tce= / --test-case-exclude= excludes;
//    -ltc lists them.  Exit status 0 iff every selected case passed.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

    template <typename T>
    friend bool operator==(const T& lhs, const Approx& r) { return r.matches(static_cast<double>(lhs)); }
    template <typename T>
    friend bool operator==(const Approx& l, const T& rhs) { return l.matches(static_cast<double>(rhs)); }
    template <typename T>
    friend bool operator!=(const T& lhs, const Approx& r) { return !r.matches(static_cast<double>(lhs)); }
    template <typename T>
    friend bool operator!=(const Approx& l, const T& rhs) { return !l.matches(static_cast<double>(rhs)); }
    template <typename T>
    friend bool operator<=(const T& lhs, const Approx& r) { return static_cast<double>(lhs) < r.value_ || r.matches(static_cast<double>(lhs)); }
    template <typename T>
    friend bool operator>=(const T& lhs, const Approx& r) { return static_cast<double>(lhs) > r.value_ || r.matches(static_cast<double>(lhs)); }
    template <typename T>
    friend bool operator<(const T& lhs, const Approx& r) { return static_cast<double>(lhs) < r.value_ && !r.matches(static_cast<double>(lhs)); }
    template <typename T>
    friend bool operator>(const T& lhs, const Approx& r) { return static_cast<double>(lhs) > r.value_ && !r.matches(static_cast<double>(lhs)); }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};

namespace detail {

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

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

struct RequireAbort {};

struct RunState {
    int failed_asserts = 0;
    int asserts = 0;
    // SUBCASE bookkeeping for the current test case
    std::set<int> done;       // subcase lines already run
    bool entered = false;     // a subcase was entered in this run
    bool pending = false;     // an unrun subcase was skipped in this run
};

inline RunState& state() {
    static RunState s;
    return s;
}

inline void report(bool ok, const char* kind, const char* expr, const char* file, int line) {
    RunState& s = state();
    ++s.asserts;
    if (ok) return;
    ++s.failed_asserts;
    std::fprintf(stderr, "%s:%d: ERROR: %s( %s ) is NOT correct!\n", file, line, kind, expr);
}

struct Subcase {
    bool enter = false;
    Subcase(const char* /*name*/, int line) {
        RunState& s = state();
        if (s.done.count(line)) return;
        if (s.entered) {
            s.pending = true;
            return;
        }
        s.entered = true;
        s.done.insert(line);
        enter = true;
    }
};

inline bool glob(const char* p, const char* s) {
    if (!*p) return !*s;
    if (*p == '*') return glob(p + 1, s) || (*s && glob(p, s + 1));
    return *s && (*p == *s) && glob(p + 1, s + 1);
}

inline bool any_glob(const std::string& list, const char* name) {
    size_t b = 0;
    while (b <= list.size()) {
        size_t e = list.find(',', b);
        if (e == std::string::npos) e = list.size();
        if (glob(list.substr(b, e - b).c_str(), name)) return true;
        b = e + 1;
    }
    return false;
}

inline int run_all(int argc, char** argv) {
    std::string inc, exc;
    bool list = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto val = [&](const char* pre) -> bool {
            if (a.rfind(pre, 0) == 0) return true;
            return false;
        };
        if (val("-tc=")) inc = a.substr(4);
        else if (val("--test-case=")) inc = a.substr(12);
        else if (val("-tce=")) exc = a.substr(5);
        else if (val("--test-case-exclude=")) exc = a.substr(20);
        else if (a == "-ltc" || a == "--list-test-cases") list = true;
    }
    int ran = 0, failed = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        if ((!inc.empty() && !any_glob(inc, tc.name)) || (!exc.empty() && any_glob(exc, tc.name))) {
            ++skipped;
            continue;
        }
        if (list) {
            std::printf("%s\n", tc.name);
            continue;
        }
        RunState& s = state();
        s.done.clear();
        const int before = s.failed_asserts;
        bool threw = false;
        do {
            s.entered = false;
            s.pending = false;
            try {
                tc.fn();
            } catch (const RequireAbort&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s:%d: ERROR: test case THREW exception: %s\n", tc.file,
                             tc.line, e.what());
                threw = true;
            } catch (...) {
                std::fprintf(stderr, "%s:%d: ERROR: test case THREW an unknown exception\n",
                             tc.file, tc.line);
                threw = true;
            }
        } while (s.pending && !threw);
        ++ran;
        const bool ok = !threw && s.failed_asserts == before;
        if (!ok) {
            ++failed;
            std::fprintf(stderr, "TEST CASE FAILED: %s (%s:%d)\n", tc.name, tc.file, tc.line);
        }
    }
    if (list) return 0;
    std::printf("[doctest-shim] test cases: %d | %d passed | %d failed | %d skipped\n", ran,
                ran - failed, failed, skipped);
    std::printf("[doctest-shim] assertions: %d | %d passed | %d failed |\n", state().asserts,
                state().asserts - state().failed_asserts, state().failed_asserts);
    std::printf("[doctest-shim] Status: %s!\n", failed ? "FAILURE" : "SUCCESS");
    return failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __COUNTER__)

#define DOCTEST_TEST_CASE_IMPL(fn, reg, name)                                               \
    static void fn();                                                                       \
    static ::doctest::detail::Registrar reg(name, __FILE__, __LINE__, &fn);                 \
    static void fn()
#define DOCTEST_TEST_CASE_IMPL2(id, name) \
    DOCTEST_TEST_CASE_IMPL(DOCTEST_CAT(doctest_fn_, id), DOCTEST_CAT(doctest_reg_, id), name)
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL2(__COUNTER__, name)

#define SUBCASE(name) \
    for (::doctest::detail::Subcase doctest_sc_(name, __LINE__); doctest_sc_.enter; doctest_sc_.enter = false)

#define CHECK(...)                                                                          \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                   \
        } catch (...) {                                                                     \
            doctest_ok_ = false;                                                            \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK", #__VA_ARGS__, __FILE__, __LINE__);  \
    } while (0)

#define REQUIRE(...)                                                                        \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            doctest_ok_ = static_cast<bool>(__VA_ARGS__);                                   \
        } catch (...) {                                                                     \
            doctest_ok_ = false;                                                            \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "REQUIRE", #__VA_ARGS__, __FILE__, __LINE__);\
        if (!doctest_ok_) throw ::doctest::detail::RequireAbort{};                          \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                          \
    do {                                                                                    \
        bool doctest_ok_ = false;                                                           \
        try {                                                                               \
            static_cast<void>(expr);                                                        \
        } catch (const __VA_ARGS__&) {                                                      \
            doctest_ok_ = true;                                                             \
        } catch (...) {                                                                     \
        }                                                                                   \
        ::doctest::detail::report(doctest_ok_, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__,  \
                                  __FILE__, __LINE__);                                      \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return ::doctest::detail::run_all(argc, argv); }
#endif
