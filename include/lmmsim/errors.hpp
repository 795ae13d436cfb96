// rserve-b200 — error taxonomy of the intra-request pipeline host API.
//
// Mirrors the reference's exception hierarchy class-for-class
// (reference: proj/include/lmmsim/errors.hpp:23-80) so code written against
// the reference (its unit tests included) catches the same types. The C-ABI
// (include/rserve.h) maps each class to one rs_status value and back.
#pragma once

#include <stdexcept>
#include <string>

namespace lmmsim {

/// Root of every error raised by the pipeline host code.
class SimError : public std::runtime_error {
 public:
  explicit SimError(const std::string& what) : std::runtime_error(what) {}
  explicit SimError(const char* what) : std::runtime_error(what) {}
};

#define LMMSIM_ERROR_CLASS(Name)                                 \
  class Name : public SimError {                                 \
   public:                                                       \
    explicit Name(const std::string& what) : SimError(what) {}   \
    explicit Name(const char* what) : SimError(what) {}          \
  }

LMMSIM_ERROR_CLASS(ConfigError);          // bad knob; message names the field
LMMSIM_ERROR_CLASS(RegistryError);        // duplicate / unknown request id
LMMSIM_ERROR_CLASS(DoubleEncodeError);    // an item's embeddings marked twice
LMMSIM_ERROR_CLASS(AlignmentError);       // encode range != one MM item
LMMSIM_ERROR_CLASS(DependencyViolation);  // prefill past the ready frontier
LMMSIM_ERROR_CLASS(InputError);           // malformed input (layout, numbers)
LMMSIM_ERROR_CLASS(DataError);            // report lacks required cells
LMMSIM_ERROR_CLASS(IoError);              // file open / write failures
LMMSIM_ERROR_CLASS(InternalError);        // broken invariant: always a bug

#undef LMMSIM_ERROR_CLASS

}  // namespace lmmsim
