// Error plumbing: internal code throws hp::Error carrying the C ABI status
// code that corresponds to the reference's exception type
// (include/hpsim/errors.hpp:22-44); the C ABI catches and records it.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "hpsim_b200.h"

namespace hp {

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

[[noreturn]] inline void config_error(const std::string& m) { throw Error(HP_ERR_CONFIG, m); }
[[noreturn]] inline void dimension_error(const std::string& m) { throw Error(HP_ERR_DIMENSION, m); }
[[noreturn]] inline void domain_error(const std::string& m) { throw Error(HP_ERR_DOMAIN, m); }
[[noreturn]] inline void usage_error(const std::string& m) { throw Error(HP_ERR_USAGE, m); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(HP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

}  // namespace hp

#define HP_CUDA(x) ::hp::cuda_check((x), #x)
