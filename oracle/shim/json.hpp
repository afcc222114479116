// TEST INFRASTRUCTURE ONLY. Compile-only stand-in for nlohmann/json (an un-vendored
// dependency of the reference's io.hpp, used there only for the volume / projection JSON
// sidecars). The oracle build exercises io.hpp's binary formats (the FGSC compressed model,
// io.hpp:319-425), never the sidecars; every json operation here throws at run time.
#pragma once
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <string>

namespace nlohmann {

class json {
 public:
  struct exception : std::runtime_error {
    using std::runtime_error::runtime_error;
  };
  json() = default;
  json(const json&) = default;
  json& operator=(const json&) = default;
  template <class T>
  json(const T&) {}
  json(std::initializer_list<json>) {}
  json& operator[](const char*) { return *this; }
  const json& at(const char*) const { fail(); }
  const json& at(std::size_t) const { fail(); }
  const json& at(int) const { fail(); }
  template <class T>
  operator T() const { fail(); }
  template <class T>
  T get() const { fail(); }
  std::string dump(int = -1) const { fail(); }
  static json parse(const std::string&) { fail(); }
  friend bool operator==(const json&, const char*) { fail(); }

 private:
  [[noreturn]] static void fail() { throw exception("json: not available in the oracle build (test-only shim)"); }
};

}  // namespace nlohmann
