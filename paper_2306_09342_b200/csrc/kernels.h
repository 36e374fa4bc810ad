// Host-side helpers shared by the launchers: error reporting that maps onto the
// reference's exception classes (ref:proj/core/include/revprop/errors.hpp:9-48).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/revprop_b200.h"

// Record `msg` as the thread-local last error and return `code`.
int rp_fail(int code, const char* msg);
// cudaGetLastError() -> RP_OK or RP_ERR_CUDA with the CUDA error string.
int rp_check_launch(const char* what);
// attention forward kernel variant (attention.cu, rp_set_attention_fwd_variant)
int rp_attn_fwd_variant();
unsigned long long* rp_attn_trace_buffer();
