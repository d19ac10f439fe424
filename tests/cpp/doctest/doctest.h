// doctest.h — a small, self-written stand-in for the doctest macros the
// reference's unit tests use (TEST_CASE, SUBCASE, CHECK*, REQUIRE*,
// CHECK_THROWS_AS / _WITH_AS, CAPTURE, FAIL, doctest::Approx / Contains), so
// /root/reference/proj/tests/unit/test_*.cpp compile UNCHANGED against the
// drop-in headers include/synscale/*.hpp (tests/cpp/Makefile).  doctest itself
// is not in this image.  TEST INFRASTRUCTURE ONLY.
//
// Subcases follow doctest's model: a test case body runs once per leaf
// subcase; each run enters the first unfinished subcase at every nesting level.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
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
    friend bool operator==(double lhs, const Approx& a) {
        return std::fabs(lhs - a.value_) <
               a.eps_ * (a.scale_ + std::max(std::fabs(lhs), std::fabs(a.value_)));
    }
    friend bool operator==(const Approx& a, double rhs) { return rhs == a; }
    friend bool operator!=(double lhs, const Approx& a) { return !(lhs == a); }
    friend bool operator!=(const Approx& a, double rhs) { return !(rhs == a); }
    friend bool operator<=(double lhs, const Approx& a) { return lhs < a.value_ || lhs == a; }
    friend bool operator>=(double lhs, const Approx& a) { return lhs > a.value_ || lhs == a; }
    friend bool operator<(double lhs, const Approx& a) { return lhs < a.value_ && lhs != a; }
    friend bool operator>(double lhs, const Approx& a) { return lhs > a.value_ && lhs != a; }

private:
    double value_;
    double eps_ = std::numeric_limits<float>::epsilon() * 100;
    double scale_ = 1.0;
};

struct Contains {
    explicit Contains(std::string s) : text(std::move(s)) {}
    bool matches(const std::string& what) const { return what.find(text) != std::string::npos; }
    std::string text;
};

namespace detail {

struct RequireFailed {};

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
    const TestCase* current = nullptr;
    long checks = 0, failures = 0;
    bool caseFailed = false;
    // subcase bookkeeping
    std::set<std::string> done;         // finished subcase paths
    std::vector<std::string> stack;     // entered subcases (paths) of this run
    std::vector<bool> pendingUnder;     // per stack entry: an unfinished child was skipped
    std::vector<bool> enteredAtLevel;   // per depth: a subcase was entered this run
    bool pending = false;               // some subcase still has to run
    std::vector<std::string> captures;
};

inline State& st() {
    static State s;
    return s;
}

inline void report(const char* file, int line, const std::string& what) {
    State& s = st();
    ++s.failures;
    s.caseFailed = true;
    std::fprintf(stderr, "%s:%d: FAILED in TEST_CASE(\"%s\")", file, line,
                 s.current ? s.current->name : "?");
    for (const auto& p : s.stack) std::fprintf(stderr, " / SUBCASE(\"%s\")", p.c_str());
    std::fprintf(stderr, "\n  %s\n", what.c_str());
    for (const auto& c : s.captures) std::fprintf(stderr, "  with %s\n", c.c_str());
}

inline void check(bool ok, const char* file, int line, const char* macro, const char* expr,
                  bool require) {
    ++st().checks;
    if (ok) return;
    report(file, line, std::string(macro) + "( " + expr + " )");
    if (require) throw RequireFailed{};
}

struct Registrar {
    Registrar(const char* name, const char* file, int line, void (*fn)()) {
        registry().push_back({name, file, line, fn});
    }
};

class Subcase {
public:
    Subcase(const char* name, const char*, int) {
        State& s = st();
        const std::size_t depth = s.stack.size();
        path_ = (s.stack.empty() ? std::string() : s.stack.back() + "/") + name;
        if (s.enteredAtLevel.size() <= depth) s.enteredAtLevel.resize(depth + 1, false);
        if (s.done.count(path_)) return;
        if (s.enteredAtLevel[depth]) {  // a sibling ran this time; come back later
            s.pending = true;
            for (std::size_t i = 0; i < s.pendingUnder.size(); ++i) s.pendingUnder[i] = true;
            return;
        }
        s.enteredAtLevel[depth] = true;
        s.stack.push_back(path_);
        s.pendingUnder.push_back(false);
        entered_ = true;
    }
    ~Subcase() {
        if (!entered_) return;
        State& s = st();
        const bool childPending = s.pendingUnder.back();
        s.stack.pop_back();
        s.pendingUnder.pop_back();
        if (s.enteredAtLevel.size() > s.stack.size() + 1)
            s.enteredAtLevel.resize(s.stack.size() + 1);
        if (!childPending) s.done.insert(path_);
    }
    explicit operator bool() const { return entered_; }

private:
    std::string path_;
    bool entered_ = false;
};

struct Capture {
    template <class T>
    Capture(const char* name, const T& v) {
        std::ostringstream os;
        os << name << " := " << v;
        st().captures.push_back(os.str());
    }
    ~Capture() { st().captures.pop_back(); }
};

inline std::string what_of(const std::exception& e) { return e.what(); }

inline bool matches(const std::string& text, const Contains& c) { return c.matches(text); }
inline bool matches(const std::string& text, const char* exact) { return text == exact; }
inline bool matches(const std::string& text, const std::string& exact) { return text == exact; }

inline int run_all() {
    State& s = st();
    long cases = 0, failedCases = 0;
    for (const TestCase& tc : registry()) {
        ++cases;
        s.current = &tc;
        s.caseFailed = false;
        s.done.clear();
        for (int run = 0; run < 10000; ++run) {
            s.stack.clear();
            s.pendingUnder.clear();
            s.enteredAtLevel.assign(1, false);
            s.pending = false;
            s.captures.clear();
            try {
                tc.fn();
            } catch (const RequireFailed&) {
            } catch (const std::exception& e) {
                report(tc.file, tc.line, std::string("unexpected exception: ") + e.what());
            } catch (...) {
                report(tc.file, tc.line, "unexpected non-std exception");
            }
            if (!s.pending) break;
        }
        if (s.caseFailed) ++failedCases;
    }
    std::printf("[doctest shim] test cases: %ld | %ld passed | %ld failed\n", cases,
                cases - failedCases, failedCases);
    std::printf("[doctest shim] assertions: %ld | %ld failed\n", s.checks, s.failures);
    return failedCases ? 1 : 0;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT2(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT2(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                        \
    static void DOCTEST_ANON(doctest_fn_)();                                                   \
    static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__,   \
                                                                   &DOCTEST_ANON(doctest_fn_)); \
    static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) \
    if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name, __FILE__, __LINE__})

#define DOCTEST_CHECK_IMPL(macro, expr, require)                                               \
    ::doctest::detail::check(static_cast<bool>(expr), __FILE__, __LINE__, macro, #expr, require)

#define CHECK(...) DOCTEST_CHECK_IMPL("CHECK", (__VA_ARGS__), false)
#define REQUIRE(...) DOCTEST_CHECK_IMPL("REQUIRE", (__VA_ARGS__), true)
#define CHECK_FALSE(...) DOCTEST_CHECK_IMPL("CHECK_FALSE", !(__VA_ARGS__), false)
#define REQUIRE_FALSE(...) DOCTEST_CHECK_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), true)
#define CHECK_MESSAGE(cond, msg) DOCTEST_CHECK_IMPL("CHECK_MESSAGE", (cond), false)
#define REQUIRE_MESSAGE(cond, msg) DOCTEST_CHECK_IMPL("REQUIRE_MESSAGE", (cond), true)
#define FAIL(msg)                                                                              \
    do {                                                                                       \
        std::ostringstream doctest_os_;                                                        \
        doctest_os_ << "FAIL: " << msg;                                                        \
        ::doctest::detail::report(__FILE__, __LINE__, doctest_os_.str());                      \
        throw ::doctest::detail::RequireFailed{};                                              \
    } while (0)
#define CAPTURE(x) const ::doctest::detail::Capture DOCTEST_ANON(doctest_cap_)(#x, x)
#define INFO(...) ((void)0)

#define CHECK_NOTHROW(...)                                                                     \
    do {                                                                                       \
        bool doctest_ok_ = true;                                                               \
        try {                                                                                  \
            (void)(__VA_ARGS__);                                                               \
        } catch (...) {                                                                        \
            doctest_ok_ = false;                                                               \
        }                                                                                      \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, \
                                 false);                                                       \
    } while (0)

#define DOCTEST_THROWS_AS(expr, type, require)                                                 \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const type&) {                                                                \
            doctest_ok_ = true;                                                                \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_AS",           \
                                 #expr ", " #type, require);                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, ...) DOCTEST_THROWS_AS(expr, __VA_ARGS__, false)
#define REQUIRE_THROWS_AS(expr, ...) DOCTEST_THROWS_AS(expr, __VA_ARGS__, true)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                               \
    do {                                                                                       \
        bool doctest_ok_ = false;                                                              \
        try {                                                                                  \
            (void)(expr);                                                                      \
        } catch (const __VA_ARGS__& e) {                                                       \
            doctest_ok_ = ::doctest::detail::matches(::doctest::detail::what_of(e), matcher);  \
        } catch (...) {                                                                        \
        }                                                                                      \
        ::doctest::detail::check(doctest_ok_, __FILE__, __LINE__, "CHECK_THROWS_WITH_AS",      \
                                 #expr ", " #matcher ", " #__VA_ARGS__, false);                \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
