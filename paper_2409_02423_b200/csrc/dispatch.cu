// dispatch.cu -- codec selection, size laws, grid sizing and launch accounting
// for the step kernels.
#include <atomic>
#include <mutex>
#include <unordered_map>

#include "codec_fixed_rate.cuh"
#include "codec_identity.cuh"
#include "codec_zfp.cuh"
#include "step_launch.cuh"

namespace hccx {

cudaError_t launch_fr_lo(int rate, int op, const StepParams& p, cudaStream_t s);
cudaError_t launch_fr_hi(int rate, int op, const StepParams& p, cudaStream_t s);
cudaError_t launch_zfp_a(int rate, int op, const StepParams& p, cudaStream_t s);
cudaError_t launch_zfp_b(int rate, int op, const StepParams& p, cudaStream_t s);

namespace {
std::atomic<uint64_t> g_launches{0};
}

uint64_t launch_count() { return g_launches.load(); }
void count_launch(uint64_t k) { g_launches.fetch_add(k); }

uint32_t group_bytes(CodecSel c) {
  switch (c.kind) {
    case 0: return IdentityCodec::kGroupBytes;
    case 2: return 4u * (1u + 8u * static_cast<uint32_t>(c.rate));
    case 3: return 32u * static_cast<uint32_t>(c.rate);
    default: return 0;
  }
}

uint64_t payload_bytes(CodecSel c, uint64_t n) {
  switch (c.kind) {
    case 0: return 4 * n;
    case 2: return ((n + 63) / 64) * (1 + 8 * static_cast<uint64_t>(c.rate));
    case 3: return (((n + 3) / 4) * 4 * static_cast<uint64_t>(c.rate) + 7) / 8;
    default: return 0;
  }
}

uint32_t fast_align(CodecSel c) { return c.kind == 0 ? 32u : 4u; }

cudaError_t launch_step(CodecSel c, int op, const StepParams& p, cudaStream_t s) {
  switch (c.kind) {
    case 0: return launch_codec_step<IdentityCodec>(op, p, s);
    case 2: return c.rate <= 16 ? launch_fr_lo(c.rate, op, p, s) : launch_fr_hi(c.rate, op, p, s);
    case 3: return c.rate <= 16 ? launch_zfp_a(c.rate, op, p, s) : launch_zfp_b(c.rate, op, p, s);
    default: return cudaErrorInvalidValue;
  }
}

int stream_grid(const void* kernel, uint64_t work_items) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;
  static int sms = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int blocks_per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (sms == 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto it = per_sm.find(kernel);
    if (it == per_sm.end()) {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kStepThreads, 0) != cudaSuccess || b < 1)
        b = 1;
      it = per_sm.emplace(kernel, b).first;
    }
    blocks_per_sm = it->second;
  }
  const uint64_t want = (work_items + kStepWarps - 1) / kStepWarps;
  const uint64_t cap = static_cast<uint64_t>(blocks_per_sm) * static_cast<uint64_t>(sms > 0 ? sms : 148);
  return static_cast<int>(want < cap ? want : cap);
}

int tma_grid(const void* kernel, int threads, uint32_t smem, uint64_t work_items) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm;
  static int sms = 0;
  int blocks_per_sm = 1;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (sms == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    auto it = per_sm.find(kernel);
    if (it == per_sm.end()) {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1) b = 1;
      it = per_sm.emplace(kernel, b).first;
    }
    blocks_per_sm = it->second;
  }
  const uint64_t cap = static_cast<uint64_t>(blocks_per_sm) * static_cast<uint64_t>(sms > 0 ? sms : 148);
  const uint64_t g = work_items < cap ? work_items : cap;
  return static_cast<int>(g > 0 ? g : 1);
}

}  // namespace hccx
