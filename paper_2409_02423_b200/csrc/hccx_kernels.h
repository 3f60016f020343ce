// hccx_kernels.h -- internal interface between the C ABI (capi.cpp, comm.cpp)
// and the CUDA kernels.  Not installed; the public surface is include/hccx.h.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hccx {

enum : uint32_t { kErrNonFinite = 1u, kErrTimeout = 2u, kErrPeer = 4u, kErrCorrupt = 8u };

enum StepOp : int { kOpEncode = 0, kOpDecode = 1, kOpDAR = 2, kOpDecodeAdd = 3 };

constexpr int kMaxJobs = 16;
constexpr int kMaxOuts = 16;

struct StepJob {
  const void* src;        // floats (Encode) or payload (Decode/DAR/DecodeAdd)
  const float* local;     // DAR / DecodeAdd: the local chunk added on the right
  void* dst;              // payload (Encode/DAR) or floats (DecodeAdd)
  float* outs[kMaxOuts];  // Decode: destinations; DAR: optional decoded copy
  int nouts;
};

struct StepParams {
  StepJob jobs[kMaxJobs];
  int njobs;
  uint64_t n;       // values per job
  int vec_ok;       // every float pointer 32-byte aligned
  int fast_ok;      // every payload pointer aligned for the codec's word path
  int tma_ok;       // every source pointer 16-byte aligned (bulk-copy path)
  int div_mode;     // 0 none, 1 multiply by recip (p power of two), 2 IEEE divide
  float recip;
  float divisor;
  uint32_t* err;    // device flag word (kErr*), may be null
};

// Codec selector shared by all dispatchers: kind 0 identity, 2 fixed-rate,
// 3 zfp-rate (1 = lossless predictor, handled separately).
struct CodecSel {
  int kind;
  int rate;
};

// Bytes of one 256-value warp group for the codec (payload stride of a group).
uint32_t group_bytes(CodecSel c);
// Payload size law for n values (src/codec.cpp:47-61 for kinds 0 and 2).
uint64_t payload_bytes(CodecSel c, uint64_t n);
// Pointer alignment the codec's word path needs (4 or 32 bytes).
uint32_t fast_align(CodecSel c);

// Launch one step kernel; returns the CUDA error of the launch.
cudaError_t launch_step(CodecSel c, int op, const StepParams& p, cudaStream_t stream);

// Kernel launches issued by this library since load (for bench accounting).
uint64_t launch_count();
void count_launch(uint64_t k = 1);

// Grid size for a streaming kernel over `work_items` warp groups.
int stream_grid(const void* kernel, uint64_t work_items);
// Persistent grid for the TMA kernel: min(work_items, SMs x resident CTAs).
int tma_grid(const void* kernel, int threads, uint32_t smem, uint64_t work_items);

}  // namespace hccx
