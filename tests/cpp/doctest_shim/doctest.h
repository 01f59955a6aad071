// doctest.h — a minimal stand-in for the doctest unit-test framework (no
// network here to fetch the real one), covering exactly what the reference's
// unit tests use (proj/tests/test_*.cpp): TEST_CASE, SUBCASE (doctest's
// re-run-per-leaf semantics), CHECK, CHECK_THROWS_AS, FAIL, doctest::Approx
// with epsilon(), and DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN.  Test
// infrastructure only: tests/cpp/Makefile compiles the reference's test
// sources, unmodified where they lie under /root/reference, against the B200
// drop-in (include/hydro + libh2d.so) and against the reference library.
#pragma once

#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
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
    // doctest's rule: |lhs - v| < eps * (scale + max(|lhs|, |v|))
    bool matches(double lhs) const {
        return std::fabs(lhs - v_) < eps_ * (scale_ + std::fmax(std::fabs(lhs), std::fabs(v_)));
    }

private:
    double v_;
    double eps_ = static_cast<double>(1.19209290e-07F) * 100;  // FLT_EPSILON * 100
    double scale_ = 1.0;
};
inline bool operator==(double l, const Approx& r) { return r.matches(l); }
inline bool operator==(const Approx& l, double r) { return l.matches(r); }
inline bool operator!=(double l, const Approx& r) { return !r.matches(l); }
inline bool operator!=(const Approx& l, double r) { return !l.matches(r); }

namespace detail {

struct Case {
    const char* name;
    const char* file;
    int line;
    void (*fn)();
};
inline std::vector<Case>& registry() {
    static std::vector<Case> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) { registry().push_back({name, file, line, fn}); }
};

// SUBCASE bookkeeping: every run of a test case enters at most one not yet
// finished subcase per nesting depth; the case re-runs until every leaf path
// has run (doctest's semantics)
struct Subcases {
    std::set<std::string> done;
    std::vector<std::string> stack;
    std::vector<char> entered;     // per depth: a subcase was entered this run
    std::vector<char> unfinished;  // per depth: a child subcase is still pending
    bool pending = false;
    void reset_run() {
        stack.clear();
        entered.assign(64, 0);
        unfinished.assign(65, 0);
        pending = false;
    }
};
inline Subcases& subcases() {
    static Subcases s;
    return s;
}

struct Stats {
    int checks = 0, failed_checks = 0;
    bool case_failed = false;
};
inline Stats& stats() {
    static Stats s;
    return s;
}

inline void report(const char* file, int line, const std::string& what) {
    std::printf("%s:%d: ERROR: %s\n", file, line, what.c_str());
    stats().failed_checks++;
    stats().case_failed = true;
}

inline void check(bool ok, const char* file, int line, const char* expr) {
    stats().checks++;
    if (!ok) report(file, line, std::string("CHECK( ") + expr + " ) is NOT correct!");
}

struct FailNow {};

class Subcase {
public:
    Subcase(const char* name, const char* file, int line) {
        Subcases& s = subcases();
        depth_ = static_cast<int>(s.stack.size());
        key_ = (depth_ ? s.stack.back() : std::string()) + "/" + file + ":" + std::to_string(line) + ":" + name;
        if (s.done.count(key_)) return;
        if (s.entered[depth_]) {  // a sibling ran this time: come back next run
            s.pending = true;
            s.unfinished[depth_] = 1;
            return;
        }
        s.entered[depth_] = 1;
        s.unfinished[depth_ + 1] = 0;
        s.stack.push_back(key_);
        active_ = true;
    }
    ~Subcase() {
        if (!active_) return;
        Subcases& s = subcases();
        s.stack.pop_back();
        if (s.unfinished[depth_ + 1])
            s.unfinished[depth_] = 1;  // a child is pending: this path is not finished
        else
            s.done.insert(key_);
    }
    explicit operator bool() const { return active_; }

private:
    std::string key_;
    int depth_ = 0;
    bool active_ = false;
};

inline int run_all() {
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        ++cases;
        stats().case_failed = false;
        Subcases& s = subcases();
        s.done.clear();
        do {
            s.reset_run();
            try {
                c.fn();
            } catch (const FailNow&) {
            } catch (const std::exception& e) {
                report(c.file, c.line, std::string("test case THREW exception: ") + e.what());
            } catch (...) {
                report(c.file, c.line, "test case THREW an unknown exception");
            }
        } while (s.pending);
        if (stats().case_failed) {
            ++failed_cases;
            std::printf("[doctest] FAILED test case: %s\n", c.name);
        }
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed\n", cases, cases - failed_cases, failed_cases);
    std::printf("[doctest] assertions: %d | %d passed | %d failed\n", stats().checks,
                stats().checks - stats().failed_checks, stats().failed_checks);
    std::printf("[doctest] Status: %s!\n", failed_cases ? "FAILURE" : "SUCCESS");
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_(fn, name)                                                                     \
    static void fn();                                                                             \
    static doctest::detail::Registrar DOCTEST_CAT(fn, _reg)(name, __FILE__, __LINE__, &fn);       \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_(DOCTEST_CAT(doctest_case_, __COUNTER__), name)
#define SUBCASE(name) if (const doctest::detail::Subcase DOCTEST_CAT(doctest_sub_, __LINE__){name, __FILE__, __LINE__})
#define CHECK(...) doctest::detail::check(static_cast<bool>(__VA_ARGS__), __FILE__, __LINE__, #__VA_ARGS__)
#define CHECK_THROWS_AS(expr, ...)                                                                \
    do {                                                                                          \
        doctest::detail::stats().checks++;                                                        \
        bool doctest_threw_ = false;                                                              \
        try {                                                                                     \
            (void)(expr);                                                                         \
        } catch (const __VA_ARGS__&) {                                                            \
            doctest_threw_ = true;                                                                \
        } catch (...) {                                                                           \
        }                                                                                         \
        if (!doctest_threw_)                                                                      \
            doctest::detail::report(__FILE__, __LINE__, "CHECK_THROWS_AS( " #expr ", " #__VA_ARGS__ " ) failed"); \
    } while (0)
#define FAIL(msg)                                                                                 \
    do {                                                                                          \
        doctest::detail::report(__FILE__, __LINE__, std::string("FAIL: ") + (msg));               \
        throw doctest::detail::FailNow{};                                                         \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return doctest::detail::run_all(); }
#endif
