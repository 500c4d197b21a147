// common.h — error plumbing shared by the host-side translation units of libslip.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/slip.h"

namespace slip {

void set_error(const std::string& msg);

// Record a CUDA error (if any) and return SLIP_ECUDA.
inline slip_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return SLIP_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return SLIP_ECUDA;
}

}  // namespace slip

#define SLIP_TRY(expr)                   \
  do {                                   \
    slip_status _st = (expr);            \
    if (_st != SLIP_OK) return _st;      \
  } while (0)

#define SLIP_CUDA(expr)                                             \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) return ::slip::cuda_status(_e, #expr);   \
  } while (0)

#define SLIP_CHECK(cond, code, msg)       \
  do {                                    \
    if (!(cond)) {                        \
      ::slip::set_error(msg);             \
      return code;                        \
    }                                     \
  } while (0)
