// doctest_min/doctest.h — a small stand-in for the doctest single-header
// framework (doctest 2.x; not in this image), implementing only what the
// reference's unit suites (proj/tests/*_test.cpp) use: TEST_CASE, SUBCASE,
// CHECK, REQUIRE, CHECK_THROWS_AS, FAIL and doctest::Approx.  It lets those
// suites compile UNMODIFIED against the B200 drop-in headers (include/tucker)
// and libtucker_b200.so, which is the point: the reference's own tests run
// against the GPU engine.
//
// Semantics restated from doctest's documentation:
//  * a TEST_CASE body is re-run until every leaf SUBCASE has run once; on each
//    run at most one not-yet-finished subcase per nesting level is entered;
//  * CHECK records a failure and continues; REQUIRE and FAIL abort the case;
//  * Approx(v) == x  iff  |x - v| < eps * (scale + max(|x|, |v|)), with
//    eps = 100 * FLT_EPSILON and scale = 1 unless set.
// Test infrastructure only; nothing in the product links it.
#pragma once

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <exception>
#include <functional>
#include <set>
#include <sstream>
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
    bool matches(double x) const { return std::fabs(x - value_) < eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_))); }
    double value() const { return value_; }

private:
    double value_;
    double eps_ = static_cast<double>(FLT_EPSILON) * 100.0;
    double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }

namespace detail {

struct AbortCase {};  // thrown by REQUIRE / FAIL

struct Registry {
    struct Case {
        const char* name;
        const char* file;
        int line;
        void (*fn)();
    };
    std::vector<Case> cases;
    // subcase bookkeeping for the running case
    std::set<std::string> finished;
    std::vector<std::string> path;
    std::vector<bool> entered_at_level;
    bool skipped = false;
    int failures_in_case = 0;
    long assertions = 0, failed_assertions = 0;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

inline std::string path_key(const std::vector<std::string>& p) {
    std::string k;
    for (const auto& s : p) k += s + "\x1f";
    return k;
}

struct Subcase {
    bool entered = false;
    std::string key;
    bool skipped_before = false;
    Subcase(const char* name, const char* file, int line) {
        Registry& r = Registry::get();
        const std::size_t level = r.path.size();
        if (r.entered_at_level.size() <= level) r.entered_at_level.resize(level + 1, false);
        std::vector<std::string> p = r.path;
        p.push_back(std::string(name) + "@" + file + ":" + std::to_string(line));
        key = path_key(p);
        if (r.finished.count(key)) return;
        if (r.entered_at_level[level]) {  // a sibling already ran on this pass
            r.skipped = true;
            return;
        }
        entered = true;
        r.entered_at_level[level] = true;
        r.path = p;
        if (r.entered_at_level.size() <= level + 1) r.entered_at_level.resize(level + 2, false);
        r.entered_at_level[level + 1] = false;
        skipped_before = r.skipped;
        r.skipped = false;
    }
    ~Subcase() {
        if (!entered) return;
        Registry& r = Registry::get();
        if (!r.skipped) r.finished.insert(key);  // no child left unvisited under this subcase
        r.skipped = r.skipped || skipped_before;
        r.path.pop_back();
    }
    explicit operator bool() const { return entered; }
};

inline void report_failure(const char* file, int line, const std::string& what) {
    Registry& r = Registry::get();
    ++r.failed_assertions;
    ++r.failures_in_case;
    std::string where;
    for (const auto& s : r.path) where += " / " + s.substr(0, s.find('@'));
    std::fprintf(stderr, "%s:%d: FAILED%s: %s\n", file, line, where.c_str(), what.c_str());
}

inline int register_case(const char* name, const char* file, int line, void (*fn)()) {
    Registry::get().cases.push_back({name, file, line, fn});
    return 0;
}

inline int run_all(int argc, char** argv) {
    Registry& r = Registry::get();
    std::string filter = argc > 1 ? argv[1] : "";
    int failed_cases = 0, run_cases = 0;
    for (const auto& c : r.cases) {
        if (!filter.empty() && std::string(c.name).find(filter) == std::string::npos) continue;
        ++run_cases;
        r.finished.clear();
        r.failures_in_case = 0;
        for (int pass = 0; pass < 10000; ++pass) {
            r.path.clear();
            r.entered_at_level.assign(1, false);
            r.skipped = false;
            try {
                c.fn();
            } catch (const AbortCase&) {
            } catch (const std::exception& e) {
                report_failure(c.file, c.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                report_failure(c.file, c.line, "unexpected non-std exception");
            }
            if (!r.skipped) break;
        }
        std::printf("[%s] %s\n", r.failures_in_case ? "FAIL" : " ok ", c.name);
        if (r.failures_in_case) ++failed_cases;
    }
    std::printf("test cases: %d | %d passed | %d failed; assertions: %ld | %ld failed\n", run_cases,
                run_cases - failed_cases, failed_cases, r.assertions, r.failed_assertions);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_UNIQUE(base) DOCTEST_CAT(base, __LINE__)

#define DOCTEST_TEST_CASE_IMPL(fn, name)                                                                     \
    static void fn();                                                                                        \
    static const int DOCTEST_CAT(fn, _reg) = doctest::detail::register_case(name, __FILE__, __LINE__, &fn); \
    static void fn()
#define TEST_CASE(name) DOCTEST_TEST_CASE_IMPL(DOCTEST_UNIQUE(doctest_case_), name)

#define SUBCASE(name) \
    if (const doctest::detail::Subcase DOCTEST_UNIQUE(doctest_sub_){name, __FILE__, __LINE__})

#define DOCTEST_ASSERT_IMPL(expr, abort)                                           \
    do {                                                                           \
        ++doctest::detail::Registry::get().assertions;                             \
        bool doctest_ok_ = false;                                                  \
        try {                                                                      \
            doctest_ok_ = static_cast<bool>(expr);                                 \
        } catch (const std::exception& doctest_e_) {                               \
            doctest::detail::report_failure(__FILE__, __LINE__,                    \
                                            std::string(#expr " threw: ") + doctest_e_.what()); \
            if (abort) throw doctest::detail::AbortCase{};                         \
            break;                                                                 \
        }                                                                          \
        if (!doctest_ok_) {                                                        \
            doctest::detail::report_failure(__FILE__, __LINE__, #expr);            \
            if (abort) throw doctest::detail::AbortCase{};                         \
        }                                                                          \
    } while (0)
#define CHECK(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL((__VA_ARGS__), true)

#define CHECK_THROWS_AS(expr, ...)                                                               \
    do {                                                                                         \
        ++doctest::detail::Registry::get().assertions;                                           \
        try {                                                                                    \
            static_cast<void>(expr);                                                             \
            doctest::detail::report_failure(__FILE__, __LINE__, #expr " did not throw " #__VA_ARGS__); \
        } catch (const __VA_ARGS__&) {                                                           \
        } catch (const std::exception& doctest_e_) {                                             \
            doctest::detail::report_failure(__FILE__, __LINE__,                                  \
                                            std::string(#expr " threw another type: ") + doctest_e_.what()); \
        } catch (...) {                                                                          \
            doctest::detail::report_failure(__FILE__, __LINE__, #expr " threw a non-std type");  \
        }                                                                                        \
    } while (0)

#define FAIL(...)                                                              \
    do {                                                                       \
        std::ostringstream doctest_msg_;                                       \
        doctest_msg_ << __VA_ARGS__;                                           \
        doctest::detail::report_failure(__FILE__, __LINE__, doctest_msg_.str()); \
        throw doctest::detail::AbortCase{};                                    \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
