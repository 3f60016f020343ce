// step_launch.cuh -- host-side launch of step_kernel<Codec, Op>; included by
// the per-rate-range translation units so the 31 fixed-rate instantiations
// compile in parallel.
#pragma once
#include "step_kernel.cuh"

namespace hccx {

template <class Codec>
cudaError_t launch_codec_step(int op, const StepParams& p, cudaStream_t stream) {
  const void* k = nullptr;
  switch (op) {
    case kOpEncode: k = reinterpret_cast<const void*>(&step_kernel<Codec, kOpEncode>); break;
    case kOpDecode: k = reinterpret_cast<const void*>(&step_kernel<Codec, kOpDecode>); break;
    case kOpDAR: k = reinterpret_cast<const void*>(&step_kernel<Codec, kOpDAR>); break;
    case kOpDecodeAdd: k = reinterpret_cast<const void*>(&step_kernel<Codec, kOpDecodeAdd>); break;
    default: return cudaErrorInvalidValue;
  }
  const uint64_t groups = (p.n + kGroupVals - 1) / kGroupVals;
  if (groups == 0 || p.njobs == 0) return cudaSuccess;
  const int grid = stream_grid(k, groups);
  void* args[] = {const_cast<StepParams*>(&p)};
  count_launch();
  return cudaLaunchKernel(k, dim3(grid), dim3(kStepThreads), args, 0, stream);
}

}  // namespace hccx
