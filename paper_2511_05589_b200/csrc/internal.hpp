// internal.hpp — context layout and error helpers shared by the C-ABI units.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: no-ops unless a profiler attaches

#include <string>

#include "kernels.cuh"

struct copris_ctx {
  int device;
  int num_sms;
  uint32_t* d_err;   // device error word (kernels.cuh ERR_*)
  unsigned long long* d_rowctr;  // row-claim counter of the fused kernels (one launch at a time)
  void* d_scratch;   // reduction scratch
  copris_b200::LaunchInfo last;  // what the last loss launch did (introspection)
  long long* d_trace;  // phase tracing buffer (COPRIS_TRACE=1 at context creation)
  copris_b200::Tuning tuning;  // kernel selection, read from COPRIS_* once at creation
};


namespace copris_b200 {

// Records `msg` as this thread's last error and returns `code`.
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

// NVTX range over a host scope (visible in Nsight Systems timelines).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Makes `dev` current for the scope of a call and restores the caller's device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

}  // namespace copris_b200
