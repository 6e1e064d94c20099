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

// Text-format failures (noise configs here; same kinds as error.hpp:50-86).
enum class ParseErrorKind { Syntax, UnknownMnemonic, ArityError, RangeError, UnterminatedBlock };

inline const char* parse_error_kind_name(ParseErrorKind k) {
  constexpr const char* names[] = {"Syntax", "UnknownMnemonic", "ArityError", "RangeError", "UnterminatedBlock"};
  const auto i = static_cast<unsigned>(k);
  return i < 5 ? names[i] : "?";
}

// line / column are 1-based; column 0 = the whole line.
class ParseError : public Error {
 public:
  ParseError(ParseErrorKind k, std::uint32_t ln, std::uint32_t col, const std::string& msg)
      : Error(std::string(parse_error_kind_name(k)) + " at line " + std::to_string(ln) +
              (col ? ":" + std::to_string(col) : std::string()) + ": " + msg),
        kind(k),
        line(ln),
        column(col) {}
  ParseErrorKind kind;
  std::uint32_t line;
  std::uint32_t column;
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
