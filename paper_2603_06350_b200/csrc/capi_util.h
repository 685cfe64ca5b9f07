// capi_util.h — status codes, the thread-local last error and the
// exception -> status boundary shared by the C-ABI translation units.
// No exception crosses the C-ABI: guarded() maps them to MOE_* codes with the
// reference's exception classes (std::invalid_argument -> MOE_EINVAL,
// std::runtime_error -> MOE_EINFEASIBLE).
#pragma once
#include <cstddef>
#include <stdexcept>
#include <string>

#include "moe_b200.h"

namespace moe {

extern thread_local std::string g_last_error;

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MOE_OK;
  } catch (const Status& s) {
    g_last_error = s.what();
    return s.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MOE_EINVAL;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return MOE_EINFEASIBLE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MOE_ESTATE;
  }
}

inline void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}

constexpr size_t pad16(size_t b) { return (b + 15) & ~size_t(15); }

}  // namespace moe
