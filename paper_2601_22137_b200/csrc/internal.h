// Host-side hooks shared by the translation units of libprism.so (defined in prism.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/prism.h"

namespace prism {
// NVTX range for the lifetime of the object (phases of a call on the host timeline).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Record `msg` as the calling thread's last error (prism_last_error) and return `s`.
prism_status fail_ext(prism_status s, const std::string& msg);
// The handle's auxiliary (communication) stream on the current device, created on first use.
cudaStream_t handle_aux_stream(prism_handle h);
// Reusable event `idx` (< 16) of the handle on the current device (timing disabled).
cudaEvent_t handle_event(prism_handle h, int idx);
}  // namespace prism
