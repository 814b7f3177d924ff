// TEST INFRASTRUCTURE ONLY — a minimal stand-in for <doctest.h> (doctest is
// not installed in this image).  It implements exactly the subset the
// reference's unit tests use (proj/tests/test_*.cpp): TEST_CASE, CHECK /
// CHECK_FALSE / REQUIRE / REQUIRE_FALSE, CHECK_THROWS_AS, CHECK_NOTHROW and
// doctest::Approx(..).epsilon(..), so those files compile UNCHANGED against the
// B200 drop-in (include/ccdkit + libccdkit.so).
//
// Runner: every registered case runs in registration order; a failing REQUIRE
// aborts its case; the summary line mirrors doctest's
// ("[doctest] test cases: N | P passed | F failed").  Command line:
//   -tce=<substr>[,<substr>...]   skip test cases whose name contains one
//   -tc=<substr>                  run only cases whose name contains it
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

namespace doctest {

struct TestCase {
    const char* name;
    void (*fn)();
    const char* file;
    int line;
};

inline std::vector<TestCase>& registry()
{
    static std::vector<TestCase> r;
    return r;
}

struct Registrar {
    Registrar(const char* name, void (*fn)(), const char* file, int line)
    {
        registry().push_back({ name, fn, file, line });
    }
};

struct RequireFailed {};

inline int& assert_failures()
{
    static int n = 0;
    return n;
}
inline int& asserts_total()
{
    static int n = 0;
    return n;
}

inline void report_failure(const char* file, int line, const char* macro, const char* expr,
                           const char* what = nullptr)
{
    ++assert_failures();
    std::printf("%s:%d: ERROR: %s( %s ) failed%s%s\n", file, line, macro, expr, what ? ": " : "",
                what ? what : "");
    std::fflush(stdout);
}

class Approx {
public:
    explicit Approx(double v)
        : value_(v)
    {
    }
    Approx& epsilon(double e)
    {
        eps_ = e;
        return *this;
    }
    friend bool operator==(double lhs, const Approx& rhs)
    {
        return std::fabs(lhs - rhs.value_)
            < rhs.eps_ * (1.0 + std::fmax(std::fabs(lhs), std::fabs(rhs.value_)));
    }
    friend bool operator==(const Approx& lhs, double rhs) { return rhs == lhs; }
    friend bool operator!=(double lhs, const Approx& rhs) { return !(lhs == rhs); }
    friend bool operator!=(const Approx& lhs, double rhs) { return !(rhs == lhs); }

private:
    double value_;
    double eps_ = 1.1920928955078125e-05 * 100; // doctest's default: float eps * 100
};

inline bool name_matches(const char* name, const std::string& list)
{
    std::size_t pos = 0;
    while (pos <= list.size()) {
        const std::size_t comma = list.find(',', pos);
        const std::string item = list.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        if (!item.empty() && std::strstr(name, item.c_str()))
            return true;
        if (comma == std::string::npos)
            break;
        pos = comma + 1;
    }
    return false;
}

inline int run(int argc, char** argv)
{
    std::string exclude, include;
    for (int i = 1; i < argc; ++i) {
        if (std::strncmp(argv[i], "-tce=", 5) == 0)
            exclude = argv[i] + 5;
        else if (std::strncmp(argv[i], "-tc=", 4) == 0)
            include = argv[i] + 4;
    }
    int passed = 0, failed = 0, skipped = 0;
    for (const TestCase& tc : registry()) {
        if ((!exclude.empty() && name_matches(tc.name, exclude))
            || (!include.empty() && !name_matches(tc.name, include))) {
            ++skipped;
            std::printf("[doctest] skipped: %s\n", tc.name);
            continue;
        }
        const int before = assert_failures();
        try {
            tc.fn();
        } catch (const RequireFailed&) {
        } catch (const std::exception& e) {
            report_failure(tc.file, tc.line, "TEST_CASE", tc.name, e.what());
        } catch (...) {
            report_failure(tc.file, tc.line, "TEST_CASE", tc.name, "unknown exception");
        }
        if (assert_failures() == before) {
            ++passed;
        } else {
            ++failed;
            std::printf("[doctest] FAILED: %s\n", tc.name);
        }
        std::fflush(stdout);
    }
    std::printf("[doctest] test cases: %d | %d passed | %d failed | %d skipped\n", passed + failed, passed,
                failed, skipped);
    std::printf("[doctest] assertions: %d | %d failed\n", asserts_total(), assert_failures());
    return failed == 0 ? 0 : 1;
}

} // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_TC_IMPL(fn, name)                                                                  \
    static void fn();                                                                              \
    static const doctest::Registrar DOCTEST_CAT(fn, _reg)(name, &fn, __FILE__, __LINE__);          \
    static void fn()
#define TEST_CASE(name) DOCTEST_TC_IMPL(DOCTEST_CAT(doctest_tc_, __LINE__), name)

#define DOCTEST_ASSERT_IMPL(macro, cond, expr, fatal)                                              \
    do {                                                                                           \
        ++doctest::asserts_total();                                                                \
        bool doctest_ok_ = false;                                                                  \
        try {                                                                                      \
            doctest_ok_ = static_cast<bool>(cond);                                                 \
        } catch (const std::exception& e) {                                                        \
            doctest::report_failure(__FILE__, __LINE__, macro, expr, e.what());                    \
            if (fatal)                                                                             \
                throw doctest::RequireFailed {};                                                   \
            break;                                                                                 \
        }                                                                                          \
        if (!doctest_ok_) {                                                                        \
            doctest::report_failure(__FILE__, __LINE__, macro, expr);                              \
            if (fatal)                                                                             \
                throw doctest::RequireFailed {};                                                   \
        }                                                                                          \
    } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), #__VA_ARGS__, false)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !(__VA_ARGS__), #__VA_ARGS__, false)
#define REQUIRE(...) DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), #__VA_ARGS__, true)
#define REQUIRE_FALSE(...) DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), #__VA_ARGS__, true)

#define CHECK_THROWS_AS(expr, ...)                                                                 \
    do {                                                                                           \
        ++doctest::asserts_total();                                                                \
        bool doctest_threw_ = false;                                                               \
        try {                                                                                      \
            static_cast<void>(expr);                                                               \
        } catch (const __VA_ARGS__&) {                                                             \
            doctest_threw_ = true;                                                                 \
        } catch (...) {                                                                            \
        }                                                                                          \
        if (!doctest_threw_)                                                                       \
            doctest::report_failure(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr ", " #__VA_ARGS__); \
    } while (0)

#define CHECK_NOTHROW(...)                                                                         \
    do {                                                                                           \
        ++doctest::asserts_total();                                                                \
        try {                                                                                      \
            static_cast<void>(__VA_ARGS__);                                                        \
        } catch (const std::exception& e) {                                                        \
            doctest::report_failure(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__, e.what());  \
        } catch (...) {                                                                            \
            doctest::report_failure(__FILE__, __LINE__, "CHECK_NOTHROW", #__VA_ARGS__);            \
        }                                                                                          \
    } while (0)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main(int argc, char** argv) { return doctest::run(argc, argv); }
#endif
