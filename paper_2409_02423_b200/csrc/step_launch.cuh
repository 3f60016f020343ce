// step_launch.cuh -- host-side launch of step_kernel<Codec, Op>; included by
// the per-rate-range translation units so the 31 fixed-rate instantiations
// compile in parallel.
#pragma once
#include <atomic>

#include "step_kernel.cuh"

namespace hccx {

// Launch with programmatic stream serialization, so a kernel's launch and
// prologue overlap the previous kernel's tail (the kernels call
// pdl_wait_and_release() before touching global memory).
inline cudaError_t launch_pdl(const void* k, int grid, int threads, void** args, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, k, args);
}

template <class Codec, int kOp>
cudaError_t launch_tma(const StepParams& p, cudaStream_t stream) {
  using L = TmaLayout<Codec, kOp>;
  const void* k = reinterpret_cast<const void*>(&step_tma_kernel<Codec, kOp>);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L::kSmem));
    configured.fetch_or(bit);
  }
  const uint64_t groups = (p.n + kGroupVals - 1) / kGroupVals;
  const uint64_t tiles = (p.n / kGroupVals / kTileGroups) * static_cast<uint64_t>(p.njobs);
  const int grid = tma_grid(k, kTmaThreads, L::kSmem, tiles > 0 ? tiles : groups * p.njobs);
  void* args[] = {const_cast<StepParams*>(&p)};
  count_launch();
  return launch_pdl(k, grid, kTmaThreads, args, L::kSmem, stream);
}

template <class Codec, int kOp>
cudaError_t launch_op(const StepParams& p, cudaStream_t stream) {
  const uint64_t groups = (p.n + kGroupVals - 1) / kGroupVals;
  if (groups == 0 || p.njobs == 0) return cudaSuccess;
  if constexpr (Codec::kFastPath) {
    if (p.vec_ok && p.fast_ok && p.tma_ok) return launch_tma<Codec, kOp>(p, stream);
  }
  const void* k = reinterpret_cast<const void*>(&step_kernel<Codec, kOp>);
  const int grid = stream_grid(k, groups);
  void* args[] = {const_cast<StepParams*>(&p)};
  count_launch();
  return launch_pdl(k, grid, kStepThreads, args, 0, stream);
}

template <class Codec>
cudaError_t launch_codec_step(int op, const StepParams& p, cudaStream_t stream) {
  switch (op) {
    case kOpEncode: return launch_op<Codec, kOpEncode>(p, stream);
    case kOpDecode: return launch_op<Codec, kOpDecode>(p, stream);
    case kOpDAR: return launch_op<Codec, kOpDAR>(p, stream);
    case kOpDecodeAdd: return launch_op<Codec, kOpDecodeAdd>(p, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx
