// Status codes + thread-local last-error text for the C-ABI. No exception
// crosses the ABI (SURVEY.md §8b "Errors"); the Python/C++ wrappers map the
// codes back to the reference's exception types.
#pragma once
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "bs_exec.h"

namespace bs200 {

inline std::string& last_error_text() {
  thread_local std::string text;
  return text;
}

inline int bs_fail(int code, const std::string& what) {
  last_error_text() = what;
  return code;
}

inline int bs_fail_cuda(cudaError_t e, const char* where) {
  last_error_text() = std::string(where) + ": " + cudaGetErrorString(e);
  return BS_ECUDA;
}

}  // namespace bs200
