// Minimal stand-in for doctest.h (absent from this image): the
// TEST_CASE / CHECK / REQUIRE subset the reference's own test files use, so
// their cases read the same when compiled against include/ssdlab_b200.hpp.
// TEST INFRASTRUCTURE ONLY.
#pragma once

#include <cstdio>
#include <exception>
#include <functional>
#include <string>
#include <vector>

namespace doctest_shim {
struct Case {
  const char* name;
  std::function<void()> fn;
};
inline std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
inline int& failures() {
  static int f = 0;
  return f;
}
inline int& checks() {
  static int c = 0;
  return c;
}
struct Registrar {
  Registrar(const char* n, void (*f)()) { registry().push_back({n, f}); }
};
struct RequireFailed {};
inline void report(bool ok, const char* expr, const char* file, int line, bool require) {
  ++checks();
  if (ok) return;
  ++failures();
  std::fprintf(stderr, "%s:%d: %s(%s) failed\n", file, line, require ? "REQUIRE" : "CHECK", expr);
  if (require) throw RequireFailed{};
}
}  // namespace doctest_shim

#define DS_CAT2(a, b) a##b
#define DS_CAT(a, b) DS_CAT2(a, b)
#define TEST_CASE(name)                                                                                  \
  static void DS_CAT(ds_case_, __LINE__)();                                                              \
  static doctest_shim::Registrar DS_CAT(ds_reg_, __LINE__)(name, &DS_CAT(ds_case_, __LINE__));           \
  static void DS_CAT(ds_case_, __LINE__)()
#define CHECK(...) doctest_shim::report(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define REQUIRE(...) doctest_shim::report(bool(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define CHECK_THROWS_AS(expr, type)                                                                      \
  do {                                                                                                   \
    bool ds_caught = false;                                                                              \
    try {                                                                                                \
      (void)(expr);                                                                                      \
    } catch (const type&) {                                                                              \
      ds_caught = true;                                                                                  \
    } catch (...) {                                                                                      \
    }                                                                                                    \
    doctest_shim::report(ds_caught, #expr " throws " #type, __FILE__, __LINE__, false);                \
  } while (0)

// main(): run every case (or those whose name contains argv[1]); one JSON
// summary line on stdout.
#define DOCTEST_SHIM_MAIN                                                                                \
  int main(int argc, char** argv) {                                                                      \
    int ran = 0, failed_cases = 0;                                                                       \
    for (const auto& c : doctest_shim::registry()) {                                                     \
      if (argc > 1 && std::string(c.name).find(argv[1]) == std::string::npos) continue;                 \
      const int before = doctest_shim::failures();                                                       \
      try {                                                                                              \
        c.fn();                                                                                          \
      } catch (const doctest_shim::RequireFailed&) {                                                     \
      } catch (const std::exception& e) {                                                                \
        ++doctest_shim::failures();                                                                      \
        std::fprintf(stderr, "%s: exception %s\n", c.name, e.what());                                    \
      }                                                                                                  \
      ++ran;                                                                                             \
      if (doctest_shim::failures() != before) {                                                          \
        ++failed_cases;                                                                                  \
        std::fprintf(stderr, "FAILED: %s\n", c.name);                                                    \
      }                                                                                                  \
    }                                                                                                    \
    std::printf("{\"cases\": %d, \"failed\": %d, \"checks\": %d}\n", ran, failed_cases,                 \
                doctest_shim::checks());                                                                 \
    return failed_cases ? 1 : 0;                                                                         \
  }
