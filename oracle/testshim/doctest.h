// Minimal doctest-compatible harness -- TEST INFRASTRUCTURE ONLY (oracle/).
//
// The reference's unit tests (proj/tests/test_*.cpp) are written against
// doctest, which is gitignored in the reference (proj/.gitignore:2 vendor/)
// and absent from this image.  This header implements only the macros those
// files use (TEST_CASE, SUBCASE, CHECK, REQUIRE, CHECK_THROWS, doctest::Approx
// with .epsilon()) so the reference tests compile and run VERBATIM against the
// oracle build in oracle/_ref.  SUBCASE follows doctest's re-entry model: a
// test case is re-run until every leaf subcase has been entered once.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <set>
#include <string>
#include <vector>

namespace doctest {

class Approx {
public:
    explicit Approx(double v)
        : value_(v), eps_(static_cast<double>(std::numeric_limits<float>::epsilon()) * 100) {}
    Approx& epsilon(double e) {
        eps_ = e;
        return *this;
    }
    bool matches(double lhs) const {
        return std::fabs(lhs - value_) <
               eps_ * (1.0 + std::max(std::fabs(lhs), std::fabs(value_)));
    }
    double value() const { return value_; }

private:
    double value_, eps_;
};
inline bool operator==(double l, const Approx& r) { return r.matches(l); }
inline bool operator==(const Approx& l, double r) { return l.matches(r); }
inline bool operator!=(double l, const Approx& r) { return !r.matches(l); }
inline bool operator<=(double l, const Approx& r) { return l < r.value() || r.matches(l); }
inline bool operator>=(double l, const Approx& r) { return l > r.value() || r.matches(l); }

namespace detail {

struct RequireFailed {};

struct State {
    std::set<std::vector<std::string>> done;
    std::set<std::vector<std::string>> entered_under;  // parents with a child entered this run
    std::vector<std::string> cur, deepest;
    long checks = 0, failures = 0;
    const char* test_name = "";
};
inline State& state() {
    static State s;
    return s;
}

struct TestEntry {
    const char* name;
    void (*fn)();
};
inline std::vector<TestEntry>& registry() {
    static std::vector<TestEntry> r;
    return r;
}
struct Registrar {
    Registrar(const char* name, void (*fn)()) { registry().push_back({name, fn}); }
};

inline void report(bool ok, const char* expr, const char* file, int line) {
    State& s = state();
    ++s.checks;
    if (!ok) {
        ++s.failures;
        std::string path;
        for (auto& p : s.cur) path += " / " + p;
        std::fprintf(stderr, "%s:%d: FAILED in [%s%s]: %s\n", file, line, s.test_name,
                     path.c_str(), expr);
    }
}

class Subcase {
public:
    explicit Subcase(const char* name) {
        State& s = state();
        std::vector<std::string> path = s.cur;
        path.push_back(name);
        if (s.done.count(path) || s.entered_under.count(s.cur)) {
            active_ = false;
            return;
        }
        s.entered_under.insert(s.cur);
        s.cur = path;
        s.deepest = path;
        active_ = true;
    }
    ~Subcase() {
        if (active_) state().cur.pop_back();
    }
    explicit operator bool() const { return active_; }

private:
    bool active_ = false;
};

inline int run_all(int argc, char** argv) {
    State& s = state();
    int cases = 0, failed_cases = 0;
    for (const auto& t : registry()) {
        if (argc > 1 && std::strstr(t.name, argv[1]) == nullptr) continue;
        ++cases;
        long before = s.failures;
        s.done.clear();
        s.test_name = t.name;
        for (int run = 0; run < 10000 && !s.done.count({}); ++run) {
            s.cur.clear();
            s.deepest.clear();
            s.entered_under.clear();
            try {
                t.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                ++s.failures;
                std::fprintf(stderr, "exception in [%s]: %s\n", t.name, e.what());
            }
            s.done.insert(s.deepest);
        }
        if (s.failures != before) ++failed_cases;
    }
    std::printf("[doctest-shim] test cases: %d | passed: %d | failed: %d | checks: %ld | failed checks: %ld\n",
                cases, cases - failed_cases, failed_cases, s.checks, s.failures);
    return failed_cases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(name, id)                                                        \
    static void DOCTEST_CAT(doctest_tc_, id)();                                          \
    static doctest::detail::Registrar DOCTEST_CAT(doctest_reg_, id)(name,                \
                                                                    &DOCTEST_CAT(doctest_tc_, id)); \
    static void DOCTEST_CAT(doctest_tc_, id)()
#define TEST_CASE(name) DOCTEST_TC_IMPL(name, __COUNTER__)
#define SUBCASE(name) if (doctest::detail::Subcase DOCTEST_CAT(doctest_sc_, __LINE__){name})
#define CHECK(...) doctest::detail::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__)
#define REQUIRE(...)                                                                     \
    do {                                                                                 \
        bool doctest_ok_ = static_cast<bool>(__VA_ARGS__);                               \
        doctest::detail::report(doctest_ok_, #__VA_ARGS__, __FILE__, __LINE__);          \
        if (!doctest_ok_) throw doctest::detail::RequireFailed{};                        \
    } while (0)
#define CHECK_THROWS(...)                                                                \
    do {                                                                                 \
        bool doctest_threw_ = false;                                                     \
        try {                                                                            \
            (void)(__VA_ARGS__);                                                         \
        } catch (...) {                                                                  \
            doctest_threw_ = true;                                                       \
        }                                                                                \
        doctest::detail::report(doctest_threw_, "THROWS: " #__VA_ARGS__, __FILE__, __LINE__); \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::detail::run_all(argc, argv); }
#endif
