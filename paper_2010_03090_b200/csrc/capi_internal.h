// capi_internal.h -- helpers shared by the C-ABI translation units (capi.cu,
// comm.cu): the per-thread last-error text and launch counter, and the
// status mapping.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/utf8v_cuda.h"

namespace u8v_capi {

extern thread_local std::string t_err;
extern thread_local int t_launches;

// Records `what` (and the CUDA error text) as this thread's last error and
// returns `code`.
int fail(int code, const std::string& what, cudaError_t e = cudaSuccess);

// Restores the caller's current device on scope exit (entry points that
// switch to a session's or a communicator's device).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() { cudaGetDevice(&prev); }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace u8v_capi

#define CK(call)                                                             \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) return u8v_capi::fail(UTF8V_ERR_CUDA, #call, _e); \
  } while (0)
