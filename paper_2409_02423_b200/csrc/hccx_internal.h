// hccx_internal.h -- host helpers shared by capi.cu and comm.cu.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a tool (nsys, ncu) is attached

#include "hccx.h"
#include "hccx_kernels.h"

namespace hccx {

hccx_status_t cuda_status(cudaError_t e);
// HCCX_ERR_CUDA, reporting the pending CUDA error and the failing site on
// stderr when HCCX_VERBOSE is set (diagnostics for multi-device failures).
hccx_status_t cuda_fail(const char* file, int line);
#define HCCX_CUDA_FAIL ::hccx::cuda_fail(__FILE__, __LINE__)
hccx_status_t cuda_status_at(cudaError_t e, const char* file, int line);
#define HCCX_STATUS(e) ::hccx::cuda_status_at((e), __FILE__, __LINE__)
hccx_status_t check_codec(hccx_codec_t c);
CodecSel sel_of(hccx_codec_t c);
void finalize_params(StepParams& p, CodecSel c, int op);
void set_divisor(StepParams& p, int mode, int nranks);
hccx_status_t run_step(CodecSel c, int op, StepParams& p, cudaStream_t s);
hccx_status_t read_flag(uint32_t* d_err, cudaStream_t s);

// NVTX range around one C-ABI entry point (the host side of a collective or
// codec call: enqueue, or the whole call for the synchronous variants).
class NvtxRange {
 public:
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define HCCX_NVTX(name) ::hccx::NvtxRange hccx_nvtx_range_(name)

// RAII: make `dev` current for the scope (no-op when dev < 0).
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = 0;
};

}  // namespace hccx
