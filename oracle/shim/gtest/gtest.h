// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// GTest-subset shim so the reference's own suites (proj/tests/*.cpp) compile
// and run unmodified as the oracle's self-check.  Covers the surface listed
// in SURVEY.md Appendix D: TEST, TEST_F, EXPECT/ASSERT_{EQ,NE,LT,LE,GT,GE,
// TRUE,FALSE,NEAR,THROW}, FAIL(), GTEST_SKIP(), ::testing::Test,
// ::testing::TempDir(), with << message streaming.  Tests run in
// registration order; `--gtest_filter=substr` selects by substring.
#ifndef ORACLE_GTEST_SHIM_H
#define ORACLE_GTEST_SHIM_H

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace testing {

class Test {
public:
    virtual ~Test() = default;
    virtual void SetUp() {}
    virtual void TearDown() {}
    virtual void TestBody() = 0;
};

inline std::string TempDir() {
    const char* t = std::getenv("TEST_TMPDIR");
    std::string d = t ? t : "/tmp";
    if (d.empty() || d.back() != '/') d += '/';
    return d;
}

namespace internal {

struct Registry {
    struct Entry {
        std::string name;
        std::function<Test*()> make;
    };
    std::vector<Entry> tests;
    static Registry& get() {
        static Registry r;
        return r;
    }
};

struct State {
    bool failed = false;
    bool skipped = false;
    static State& cur() {
        static State s;
        return s;
    }
};

struct AbortTest {};
struct SkipTest {};

inline bool Register(const char* suite, const char* name, std::function<Test*()> make) {
    Registry::get().tests.push_back({std::string(suite) + "." + name, std::move(make)});
    return true;
}

/** Collects the streamed message and reports on destruction. */
class Reporter {
public:
    Reporter(const char* file, int line, std::string what, bool fatal)
        : file_(file), line_(line), what_(std::move(what)), fatal_(fatal) {}
    template <class T>
    Reporter& operator<<(const T& v) {
        msg_ << v;
        return *this;
    }
    ~Reporter() noexcept(false) {
        State::cur().failed = true;
        std::fprintf(stderr, "%s:%d: Failure\n%s\n%s\n", file_, line_, what_.c_str(),
                     msg_.str().c_str());
        if (fatal_ && !std::uncaught_exceptions()) throw AbortTest{};
    }

private:
    const char* file_;
    int line_;
    std::string what_;
    bool fatal_;
    std::ostringstream msg_;
};

class Skipper {
public:
    template <class T>
    Skipper& operator<<(const T& v) {
        msg_ << v;
        return *this;
    }
    ~Skipper() noexcept(false) {
        State::cur().skipped = true;
        std::fprintf(stderr, "  skipped: %s\n", msg_.str().c_str());
        if (!std::uncaught_exceptions()) throw SkipTest{};
    }

private:
    std::ostringstream msg_;
};

struct Null {
    template <class T>
    Null& operator<<(const T&) {
        return *this;
    }
};

template <class T>
std::string show(const T& v) {
    if constexpr (requires(std::ostream& o, const T& x) { o << x; }) {
        std::ostringstream s;
        s.precision(17);
        s << v;
        return s.str();
    } else {
        return "<value>";
    }
}

}  // namespace internal

inline int RunAllTests(int argc, char** argv) {
    std::string filter;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        if (a.rfind("--gtest_filter=", 0) == 0) filter = a.substr(15);
    }
    int failed = 0, passed = 0, skipped = 0;
    for (auto& e : internal::Registry::get().tests) {
        if (!filter.empty() && e.name.find(filter) == std::string::npos) continue;
        internal::State::cur() = internal::State{};
        std::fprintf(stderr, "[ RUN      ] %s\n", e.name.c_str());
        Test* t = nullptr;
        try {
            t = e.make();
            t->SetUp();
            t->TestBody();
        } catch (const internal::AbortTest&) {
        } catch (const internal::SkipTest&) {
        } catch (const std::exception& ex) {
            internal::State::cur().failed = true;
            std::fprintf(stderr, "uncaught exception: %s\n", ex.what());
        } catch (...) {
            internal::State::cur().failed = true;
            std::fprintf(stderr, "uncaught non-std exception\n");
        }
        if (t) {
            try {
                t->TearDown();
            } catch (...) {
            }
            delete t;
        }
        if (internal::State::cur().failed) {
            ++failed;
            std::fprintf(stderr, "[  FAILED  ] %s\n", e.name.c_str());
        } else if (internal::State::cur().skipped) {
            ++skipped;
            std::fprintf(stderr, "[  SKIPPED ] %s\n", e.name.c_str());
        } else {
            ++passed;
            std::fprintf(stderr, "[       OK ] %s\n", e.name.c_str());
        }
    }
    std::fprintf(stderr, "[==========] %d passed, %d failed, %d skipped\n", passed, failed,
                 skipped);
    return failed ? 1 : 0;
}

}  // namespace testing

#define GTEST_SHIM_CLASS(suite, name) suite##_##name##_Test

#define TEST(suite, name)                                                               \
    class GTEST_SHIM_CLASS(suite, name) : public ::testing::Test {                       \
    public:                                                                             \
        void TestBody() override;                                                       \
    };                                                                                  \
    static bool gtest_shim_reg_##suite##_##name = ::testing::internal::Register(         \
        #suite, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS(suite, name)); }); \
    void GTEST_SHIM_CLASS(suite, name)::TestBody()

#define TEST_F(fixture, name)                                                           \
    class GTEST_SHIM_CLASS(fixture, name) : public fixture {                             \
    public:                                                                             \
        void TestBody() override;                                                       \
    };                                                                                  \
    static bool gtest_shim_reg_##fixture##_##name = ::testing::internal::Register(       \
        #fixture, #name, [] { return static_cast<::testing::Test*>(new GTEST_SHIM_CLASS(fixture, name)); }); \
    void GTEST_SHIM_CLASS(fixture, name)::TestBody()

#define GTEST_SHIM_CHECK(cond, text, fatal)                                     \
    if (cond)                                                                   \
        ;                                                                       \
    else                                                                        \
        ::testing::internal::Reporter(__FILE__, __LINE__, text, fatal)

#define GTEST_SHIM_CMP(a, b, op, fatal)                                                      \
    if (auto gtest_shim_a = (a); true)                                                      \
        if (auto gtest_shim_b = (b); gtest_shim_a op gtest_shim_b)                           \
            ;                                                                               \
        else                                                                                \
            ::testing::internal::Reporter(__FILE__, __LINE__,                                \
                                          std::string("Expected: (" #a ") " #op " (" #b      \
                                                      "), actual: ") +                       \
                                              ::testing::internal::show(gtest_shim_a) +      \
                                              " vs " + ::testing::internal::show(gtest_shim_b), \
                                          fatal)

#define EXPECT_EQ(a, b) GTEST_SHIM_CMP(a, b, ==, false)
#define EXPECT_NE(a, b) GTEST_SHIM_CMP(a, b, !=, false)
#define EXPECT_LT(a, b) GTEST_SHIM_CMP(a, b, <, false)
#define EXPECT_LE(a, b) GTEST_SHIM_CMP(a, b, <=, false)
#define EXPECT_GT(a, b) GTEST_SHIM_CMP(a, b, >, false)
#define EXPECT_GE(a, b) GTEST_SHIM_CMP(a, b, >=, false)
#define ASSERT_EQ(a, b) GTEST_SHIM_CMP(a, b, ==, true)
#define ASSERT_NE(a, b) GTEST_SHIM_CMP(a, b, !=, true)
#define ASSERT_LT(a, b) GTEST_SHIM_CMP(a, b, <, true)
#define ASSERT_LE(a, b) GTEST_SHIM_CMP(a, b, <=, true)
#define ASSERT_GT(a, b) GTEST_SHIM_CMP(a, b, >, true)
#define ASSERT_GE(a, b) GTEST_SHIM_CMP(a, b, >=, true)
#define EXPECT_TRUE(c) GTEST_SHIM_CHECK(static_cast<bool>(c), "Value of: " #c " expected true", false)
#define EXPECT_FALSE(c) GTEST_SHIM_CHECK(!static_cast<bool>(c), "Value of: " #c " expected false", false)
#define ASSERT_TRUE(c) GTEST_SHIM_CHECK(static_cast<bool>(c), "Value of: " #c " expected true", true)
#define ASSERT_FALSE(c) GTEST_SHIM_CHECK(!static_cast<bool>(c), "Value of: " #c " expected false", true)
#define EXPECT_DOUBLE_EQ(a, b) EXPECT_EQ(a, b)

#define GTEST_SHIM_NEAR(a, b, tol, fatal)                                                 \
    if (double gtest_shim_d = std::abs(double(a) - double(b)); gtest_shim_d <= double(tol)) \
        ;                                                                                  \
    else                                                                                   \
        ::testing::internal::Reporter(__FILE__, __LINE__,                                   \
                                      std::string("|" #a " - " #b "| = ") +                 \
                                          ::testing::internal::show(gtest_shim_d) +        \
                                          " exceeds " #tol,                                 \
                                      fatal)
#define EXPECT_NEAR(a, b, tol) GTEST_SHIM_NEAR(a, b, tol, false)
#define ASSERT_NEAR(a, b, tol) GTEST_SHIM_NEAR(a, b, tol, true)

#define GTEST_SHIM_THROW(stmt, exc, fatal)                                            \
    if (int gtest_shim_r = [&]() -> int {                                            \
            try {                                                                    \
                stmt;                                                                \
            } catch (const exc&) {                                                   \
                return 0;                                                            \
            } catch (...) {                                                          \
                return 2;                                                            \
            }                                                                        \
            return 1;                                                                \
        }();                                                                         \
        gtest_shim_r == 0)                                                           \
        ;                                                                            \
    else                                                                             \
        ::testing::internal::Reporter(__FILE__, __LINE__,                             \
                                      gtest_shim_r == 1 ? "Expected " #stmt " to throw " #exc \
                                                        : #stmt " threw a different type", \
                                      fatal)
#define EXPECT_THROW(stmt, exc) GTEST_SHIM_THROW(stmt, exc, false)
#define ASSERT_THROW(stmt, exc) GTEST_SHIM_THROW(stmt, exc, true)
#define EXPECT_NO_THROW(stmt) GTEST_SHIM_THROW(stmt; throw 0, int, false)

#define FAIL() ::testing::internal::Reporter(__FILE__, __LINE__, "Failed", true)
#define ADD_FAILURE() ::testing::internal::Reporter(__FILE__, __LINE__, "Failed", false)
#define SUCCEED() ::testing::internal::Null()
#define GTEST_SKIP() ::testing::internal::Skipper()

#endif  // ORACLE_GTEST_SHIM_H
