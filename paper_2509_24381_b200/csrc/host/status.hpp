// rserve-b200 — exception <-> rs_status translation for the C-ABI.
//
// Every extern "C" entry point runs its body inside rserve::guarded(); the
// thrown lmmsim exception class becomes the status code (one per class of
// reference errors.hpp:23-80) and its what() text the thread-local
// rs_last_error() string, so a caller can rethrow the identical error.
#pragma once

#include <cstdlib>
#include <cstring>
#include <string>

#include "lmmsim/errors.hpp"
#include "rserve.h"

namespace rserve {

/// CUDA / NCCL failures raised inside the product.
class DeviceError : public std::runtime_error {
 public:
  DeviceError(rs_status code, const std::string& what)
      : std::runtime_error(what), code_(code) {}
  rs_status code() const { return code_; }

 private:
  rs_status code_;
};

std::string& last_error_slot();

template <typename F>
rs_status guarded(F&& body) {
  try {
    body();
    return RS_OK;
  } catch (const DeviceError& e) {
    last_error_slot() = e.what();
    return e.code();
  } catch (const lmmsim::ConfigError& e) {
    last_error_slot() = e.what();
    return RS_ERR_CONFIG;
  } catch (const lmmsim::RegistryError& e) {
    last_error_slot() = e.what();
    return RS_ERR_REGISTRY;
  } catch (const lmmsim::DoubleEncodeError& e) {
    last_error_slot() = e.what();
    return RS_ERR_DOUBLE_ENCODE;
  } catch (const lmmsim::AlignmentError& e) {
    last_error_slot() = e.what();
    return RS_ERR_ALIGNMENT;
  } catch (const lmmsim::DependencyViolation& e) {
    last_error_slot() = e.what();
    return RS_ERR_DEPENDENCY_VIOLATION;
  } catch (const lmmsim::InputError& e) {
    last_error_slot() = e.what();
    return RS_ERR_INPUT;
  } catch (const lmmsim::DataError& e) {
    last_error_slot() = e.what();
    return RS_ERR_DATA;
  } catch (const lmmsim::IoError& e) {
    last_error_slot() = e.what();
    return RS_ERR_IO;
  } catch (const lmmsim::InternalError& e) {
    last_error_slot() = e.what();
    return RS_ERR_INTERNAL;
  } catch (const lmmsim::SimError& e) {
    last_error_slot() = e.what();
    return RS_ERR_SIM;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return RS_ERR_UNKNOWN;
  }
}

inline char* c_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  return p;
}

}  // namespace rserve
