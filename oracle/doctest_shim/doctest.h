// Minimal doctest-compatible test harness so the reference's own unit tests
// (/root/reference/proj/tests/test_*.cpp, doctest is not vendored there:
// proj/.gitignore:2) compile unmodified against the shim-built oracle.
// TEST INFRASTRUCTURE ONLY. Supports the subset the reference uses:
// TEST_CASE, SUBCASE (Catch/doctest re-run semantics), CHECK, CHECK_FALSE,
// REQUIRE, CHECK_NOTHROW, CHECK_THROWS_AS, FAIL, doctest::Approx.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <iostream>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v) : value_(v), eps_(1.1920928955078125e-07 * 100), scale_(1.0) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    Approx& scale(double s) {
        scale_ = s;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
    friend bool operator<=(const Approx& a, double rhs) { return a.value_ < rhs || rhs == a; }
    friend bool operator>=(const Approx& a, double rhs) { return a.value_ > rhs || rhs == a; }

private:
    double value_, eps_, scale_;
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

struct AbortTest {};

struct State {
    int failed_asserts = 0;
    int passed_asserts = 0;
    bool current_failed = false;
    const char* current = "";
    // Subcase tracking (re-run semantics).
    std::set<std::string> done;
    std::vector<std::string> stack;
    std::vector<bool> taken;     // a subcase was entered at this depth this run
    std::vector<bool> pending;   // a not-done subcase was skipped inside this depth
    bool any_pending = false;
};

inline State& state() {
    static State s;
    return s;
}

inline void report_fail(const char* file, int line, const char* what, const char* expr) {
    State& s = state();
    ++s.failed_asserts;
    s.current_failed = true;
    std::fprintf(stderr, "%s:%d: %s( %s ) FAILED in test case \"%s\"\n", file, line, what, expr,
                 s.current);
}

inline void report_pass() { ++state().passed_asserts; }

class Subcase {
public:
    Subcase(const char* name, const char* file, int line) {
        State& s = state();
        const std::size_t depth = s.stack.size();
        std::string key = (depth ? s.stack.back() : std::string(s.current)) + "/" + name + "@" +
                          file + ":" + std::to_string(line);
        if (s.taken.size() <= depth)
            s.taken.resize(depth + 1, false);
        if (s.done.count(key)) {
            entered_ = false;
            return;
        }
        if (s.taken[depth]) {
            entered_ = false;
            s.any_pending = true;
            for (std::size_t d = 0; d < s.pending.size() && d < depth; ++d)
                s.pending[d] = true;
            return;
        }
        s.taken[depth] = true;
        entered_ = true;
        key_ = key;
        s.stack.push_back(key);
        if (s.taken.size() <= depth + 1)
            s.taken.resize(depth + 2, false);
        s.taken[depth + 1] = false;
        if (s.pending.size() <= depth)
            s.pending.resize(depth + 1, false);
        s.pending[depth] = false;
    }
    ~Subcase() {
        if (!entered_)
            return;
        State& s = state();
        const std::size_t depth = s.stack.size() - 1;
        if (!s.pending[depth])
            s.done.insert(key_);
        s.stack.pop_back();
    }
    explicit operator bool() const { return entered_; }

private:
    bool entered_ = false;
    std::string key_;
};

inline int run_all() {
    State& s = state();
    int failed_cases = 0;
    for (const TestCase& tc : registry()) {
        s.current = tc.name;
        s.current_failed = false;
        s.done.clear();
        int runs = 0;
        do {
            s.any_pending = false;
            s.stack.clear();
            s.taken.assign(1, false);
            s.pending.clear();
            try {
                tc.fn();
            } catch (const AbortTest&) {
            } catch (const std::exception& e) {
                std::fprintf(stderr, "%s:%d: test case \"%s\" threw: %s\n", tc.file, tc.line,
                             tc.name, e.what());
                s.current_failed = true;
                ++s.failed_asserts;
            }
            ++runs;
        } while (s.any_pending && runs < 1000);
        if (s.current_failed)
            ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %zu | %zu passed | %d failed\n", registry().size(),
                registry().size() - failed_cases, failed_cases);
    std::printf("[doctest-shim] assertions: %d passed | %d failed\n", s.passed_asserts,
                s.failed_asserts);
    return failed_cases == 0 ? 0 : 1;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_IMPL(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_IMPL(a, b)
#define DOCTEST_UNIQUE(prefix) DOCTEST_CAT(prefix, __LINE__)

#define TEST_CASE(name)                                                                    \
    static void DOCTEST_UNIQUE(doctest_fn_)();                                             \
    static ::doctest::detail::Registrar DOCTEST_UNIQUE(doctest_reg_)(                      \
        name, __FILE__, __LINE__, &DOCTEST_UNIQUE(doctest_fn_));                           \
    static void DOCTEST_UNIQUE(doctest_fn_)()

#define SUBCASE(name) \
    if (const ::doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sc_){name, __FILE__, __LINE__})

#define DOCTEST_ASSERT_IMPL(kind, cond, expr_text, abort)                        \
    do {                                                                          \
        bool doctest_ok_ = false;                                                 \
        try {                                                                     \
            doctest_ok_ = static_cast<bool>(cond);                                \
        } catch (...) {                                                           \
            doctest_ok_ = false;                                                  \
        }                                                                         \
        if (doctest_ok_) {                                                        \
            ::doctest::detail::report_pass();                                     \
        } else {                                                                  \
            ::doctest::detail::report_fail(__FILE__, __LINE__, kind, expr_text);  \
            if (abort)                                                            \
                throw ::doctest::detail::AbortTest{};                             \
        }                                                                         \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_NOTHROW(...)                                                               \
    do {                                                                                 \
        try {                                                                            \
            (void)(__VA_ARGS__);                                                         \
            ::doctest::detail::report_pass();                                            \
        } catch (...) {                                                                  \
            ::doctest::detail::report_fail(__FILE__, __LINE__, "CHECK_NOTHROW",          \
                                           #__VA_ARGS__);                                \
        }                                                                                \
    } while (0)

#define CHECK_THROWS_AS(expr, ...)                                                       \
    do {                                                                                 \
        bool doctest_ok_ = false;                                                        \
        try {                                                                            \
            (void)(expr);                                                                \
        } catch (const __VA_ARGS__&) {                                                   \
            doctest_ok_ = true;                                                          \
        } catch (...) {                                                                  \
        }                                                                                \
        if (doctest_ok_)                                                                 \
            ::doctest::detail::report_pass();                                            \
        else                                                                             \
            ::doctest::detail::report_fail(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr); \
    } while (0)

#define FAIL(msg)                                                                        \
    do {                                                                                 \
        ::doctest::detail::report_fail(__FILE__, __LINE__, "FAIL", "");                  \
        std::cerr << "  " << msg << std::endl;                                           \
        throw ::doctest::detail::AbortTest{};                                            \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
