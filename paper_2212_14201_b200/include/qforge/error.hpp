// qforge drop-in (B200 backend): exception types.
// Same hierarchy and names as the reference (error.hpp:10-86), so callers'
// catch clauses keep working; libqsb status codes are mapped onto them.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "qsb.h"

namespace qforge {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ValidationError : public Error {
 public:
  using Error::Error;
};
class FlatCircuitRequired : public Error {
 public:
  using Error::Error;
};
class UnsupportedError : public Error {
 public:
  using Error::Error;
};
class NonTerminationGuard : public Error {
 public:
  using Error::Error;
};

namespace detail {
// Converts a libqsb status into the matching qforge exception.
inline void qs_check(int rc) {
  if (rc == QS_OK) return;
  const std::string msg = qs_last_error();
  switch (rc) {
    case QS_ERR_VALIDATION: throw ValidationError(msg);
    case QS_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    case QS_ERR_MEMORY: throw Error("out of device memory: " + msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

}  // namespace qforge
