// Thread-local error text behind rp_last_error(); status codes mirror
// ref:proj/core/include/revprop/errors.hpp:9-48.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "kernels.h"

static thread_local std::string g_last_error;

int rp_fail(int code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}

int rp_check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return RP_OK;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  // device memory exhausted is the reference's BudgetError (errors.hpp), not a fault
  return e == cudaErrorMemoryAllocation ? RP_ERR_BUDGET : RP_ERR_CUDA;
}

extern "C" const char* rp_last_error(void) { return g_last_error.c_str(); }

namespace rp {
static bool g_pdl = false;  // measured: no gain for this step (see profiles/)
bool pdl_enabled() { return g_pdl; }
}  // namespace rp

// Programmatic dependent launch on (1, default) or off (0) for all kernels of the library.
extern "C" int rp_set_pdl(int on) {
  rp::g_pdl = on != 0;
  return RP_OK;
}

extern "C" int rp_version(char* buf, int len) {
  const char* v = "revprop_b200 0.1 (sm_100a: tcgen05/TMEM/TMA GEMM, fused LN, attention)";
  if (buf && len > 0) {
    std::strncpy(buf, v, static_cast<size_t>(len) - 1);
    buf[len - 1] = '\0';
  }
  return RP_OK;
}
