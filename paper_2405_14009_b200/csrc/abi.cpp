// abi.cpp — error state and small C-ABI entry points of libslip.
#include <string>

#include "common.h"

namespace slip {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace slip

extern "C" {

int32_t slip_version(void) { return 1; }

const char* slip_last_error(void) { return slip::g_last_error.c_str(); }

const char* slip_status_str(slip_status s) {
  switch (s) {
    case SLIP_OK: return "SLIP_OK";
    case SLIP_EINVAL: return "SLIP_EINVAL";
    case SLIP_EUNRECOVERABLE: return "SLIP_EUNRECOVERABLE";
    case SLIP_EINFEASIBLE_MEMORY: return "SLIP_EINFEASIBLE_MEMORY";
    case SLIP_ESTATE: return "SLIP_ESTATE";
    case SLIP_ECUDA: return "SLIP_ECUDA";
    case SLIP_ENCCL: return "SLIP_ENCCL";
    case SLIP_ENONFINITE: return "SLIP_ENONFINITE";
    case SLIP_EUNSUPPORTED: return "SLIP_EUNSUPPORTED";
  }
  return "SLIP_E?";
}

}  // extern "C"
