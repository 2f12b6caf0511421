// doctest.h — a from-scratch stand-in for the subset of the doctest test
// framework the reference's suites use (proj/tests/*.cpp: TEST_CASE,
// SUBCASE, CHECK, CHECK_FALSE, CHECK_NOTHROW, CHECK_THROWS_AS, REQUIRE,
// FAIL, doctest::Approx).  TEST INFRASTRUCTURE: it lets the reference's own
// test files compile unchanged here, against the reference and against the
// drop-in (tests/cpp/Makefile).  doctest itself is not vendored in the
// reference tree (its CMake fetches it), so this follows doctest's
// documented semantics:
//   - a TEST_CASE with SUBCASEs is run once per leaf subcase, re-entering
//     the body from the top each time;
//   - CHECK* record a failure and continue, REQUIRE/FAIL end the test case;
//   - Approx(x) == y  iff  |x - y| < eps * (scale + max(|x|, |y|)), default
//     eps = 100 * FLT_EPSILON, scale = 1.
//   - the runner prints every failed assertion and exits non-zero if any
//     test case failed; DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN (or
//     WG_DOCTEST_MAIN) in one translation unit provides main().
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.v_) < a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.v_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.v_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.v_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.v_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.v_ && lhs != a; }

  private:
    double v_;
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

// Subcase bookkeeping of the running test case: one leaf path per pass.
struct Runner {
    std::set<std::string> done;   // finished subcase paths
    std::vector<std::string> path;
    std::vector<bool> entered;    // per depth: a subcase was entered this pass
    bool skipped_undone = false;  // an unfinished subcase was skipped this pass
    unsigned failed_asserts = 0;
    unsigned asserts = 0;
    const char* current = "";
    std::vector<bool> child_skipped;  // per open subcase: an unfinished child was skipped
};

inline Runner& runner() {
    static Runner r;
    return r;
}

struct RequireFailed {};

class Subcase {
  public:
    Subcase(const char* name) {
        Runner& r = runner();
        const std::size_t depth = r.path.size();
        if (r.entered.size() <= depth) r.entered.resize(depth + 1, false);
        std::string full;
        for (const auto& p : r.path) full += p + "/";
        full += name;
        key_ = full;
        if (r.done.count(full)) return;
        if (r.entered[depth]) {  // a sibling runs this pass; come back later
            r.skipped_undone = true;
            if (!r.child_skipped.empty()) r.child_skipped.back() = true;
            return;
        }
        r.entered[depth] = true;
        r.path.push_back(name);
        r.child_skipped.push_back(false);
        active_ = true;
    }
    ~Subcase() {
        if (!active_) return;
        Runner& r = runner();
        const bool pending_children = r.child_skipped.back();
        r.child_skipped.pop_back();
        r.path.pop_back();
        if (r.entered.size() > r.path.size() + 1) r.entered.resize(r.path.size() + 1);
        if (!pending_children) r.done.insert(key_);
    }
    explicit operator bool() const { return active_; }

  private:
    std::string key_;
    bool active_ = false;
};

inline void report_failure(const char* file, int line, const char* what, const std::string& expr) {
    Runner& r = runner();
    ++r.failed_asserts;
    std::string sub;
    for (const auto& p : r.path) sub += " / " + p;
    std::fprintf(stderr, "%s:%d: FAILED in \"%s\"%s: %s( %s )\n", file, line, r.current, sub.c_str(), what,
                 expr.c_str());
}

inline void check(bool ok, const char* file, int line, const char* what, const char* expr, bool require) {
    ++runner().asserts;
    if (ok) return;
    report_failure(file, line, what, expr);
    if (require) throw RequireFailed{};
}

inline int run_all() {
    unsigned cases_failed = 0, cases = 0, asserts = 0, failed_asserts = 0;
    for (const TestCase& tc : registry()) {
        ++cases;
        Runner& r = runner();
        r = Runner{};
        r.current = tc.name;
        bool case_failed = false;
        for (;;) {
            r.path.clear();
            r.entered.assign(1, false);
            r.child_skipped.clear();
            r.skipped_undone = false;
            const unsigned before = r.failed_asserts;
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report_failure(tc.file, tc.line, "unexpected exception", e.what());
            } catch (...) {
                report_failure(tc.file, tc.line, "unexpected exception", "unknown type");
            }
            if (r.failed_asserts != before) case_failed = true;
            // a subcase left early by REQUIRE / an exception counts as done
            if (!r.path.empty()) {
                std::string full;
                for (std::size_t k = 0; k < r.path.size(); ++k) full += (k ? "/" : "") + r.path[k];
                r.done.insert(full);
            }
            if (!r.skipped_undone) break;
        }
        asserts += r.asserts;
        failed_asserts += r.failed_asserts;
        if (case_failed) ++cases_failed;
    }
    std::printf("[doctest-shim] test cases: %u | %u passed | %u failed\n", cases, cases - cases_failed,
                cases_failed);
    std::printf("[doctest-shim] assertions: %u | %u passed | %u failed\n", asserts, asserts - failed_asserts,
                failed_asserts);
    return cases_failed ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                            \
    static void DOCTEST_ANON(doctest_fn_)();                                                       \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,       \
                                                                   &DOCTEST_ANON(doctest_fn_));    \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define DOCTEST_ASSERT_(what, cond, require) \
    ::doctest::detail::check(static_cast<bool>(cond), __FILE__, __LINE__, what, #cond, require)

#define CHECK(...) DOCTEST_ASSERT_("CHECK", (__VA_ARGS__), false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_("REQUIRE", (__VA_ARGS__), true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_("REQUIRE_FALSE", !(__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                              \
    do {                                                                                        \
        bool doctest_ok_ = false;                                                               \
        try {                                                                                   \
            static_cast<void>(expr);                                                            \
        } catch (const __VA_ARGS__&) {                                                          \
            doctest_ok_ = true;                                                                 \
        } catch (...) {                                                                         \
        }                                                                                       \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__, \
                                 false);                                                        \
    } while (0)

#define CHECK_NOTHROW(...)                                                                       \
    do {                                                                                         \
        bool doctest_ok_ = true;                                                                 \
        try {                                                                                    \
            static_cast<void>(__VA_ARGS__);                                                      \
        } catch (...) {                                                                          \
            doctest_ok_ = false;                                                                 \
        }                                                                                        \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, false); \
    } while (0)

#define FAIL(msg)                                                                      \
    do {                                                                               \
        std::ostringstream doctest_os_;                                                \
        doctest_os_ << msg;                                                            \
        ::doctest::detail::report_failure(__FILE__, __LINE__, "FAIL", doctest_os_.str()); \
        throw ::doctest::detail::RequireFailed{};                                      \
    } while (0)

#if defined(DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN) || defined(WG_DOCTEST_MAIN)
int main() { return ::doctest::detail::run_all(); }
#endif
