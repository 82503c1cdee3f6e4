// Maps C-ABI statuses (include/lpmc_b200.h) back onto the exception types the
// reference throws, with the reference's what() text.
#pragma once

#include <stdexcept>
#include <string>

#include "../lpmc_b200.h"

namespace lpmc {

// Device / driver failure; the reference has no counterpart (it never runs
// on a GPU) and the library never falls back to the CPU.
class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {

inline void throw_status(lpmc_status st, const lpmc_error& err) {
  const std::string msg(err.message);
  switch (st) {
    case LPMC_OK: return;
    case LPMC_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LPMC_DOMAIN_ERROR: throw std::domain_error(msg);
    case LPMC_RUNTIME_ERROR: throw std::runtime_error(msg);
    default: throw device_error(msg);
  }
}

}  // namespace detail
}  // namespace lpmc
