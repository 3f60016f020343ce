// fused_launch.cuh -- cooperative launch of ring_fused_kernel<Codec>; included
// by the per-rate-range translation units.
#pragma once
#include <atomic>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "oneshot.cuh"
#include "ring_fused.cuh"

namespace hccx {

// Co-resident CTAs of the fused kernel on this device (cooperative-launch cap).
int fused_capacity(const void* kernel, int threads, uint32_t smem);

template <class Codec>
cudaError_t launch_oneshot_codec(const FusedParams& p, cudaStream_t stream) {
  const void* k = reinterpret_cast<const void*>(&oneshot_allreduce_kernel<Codec>);
  const uint64_t groups = (p.n_chunk + kGroupVals - 1) / kGroupVals;
  if (groups == 0) return cudaSuccess;
  // co-resident (cooperative) so no CTA waits on a peer while another CTA of
  // this launch is still queued; ~8 groups per CTA, at most one CTA per SM
  const uint64_t cap = static_cast<uint64_t>(fused_capacity(k, kOsWarps * 32, 0));
  uint64_t grid = (groups + 7) / 8;
  const uint64_t lim = cap < 148 ? cap : 148;
  grid = grid < lim ? grid : lim;
  grid = grid < kAckIdx ? grid : kAckIdx;
  void* args[] = {const_cast<FusedParams*>(&p)};
  count_launch();
  return cudaLaunchCooperativeKernel(k, dim3(static_cast<unsigned>(grid)), dim3(kOsWarps * 32), args, 0, stream);
}

template <class Codec>
cudaError_t launch_fused_codec(const FusedParams& p, cudaStream_t stream) {
  if (p.op == kFOneShotAllReduce) return launch_oneshot_codec<Codec>(p, stream);
  const void* k = reinterpret_cast<const void*>(&ring_fused_kernel<Codec>);
  const uint64_t groups = (p.n_chunk + kGroupVals - 1) / kGroupVals;
  const uint64_t nseg = (groups + kSegGroups - 1) / kSegGroups;
  if (nseg == 0) return cudaSuccess;
  constexpr uint32_t smem = sizeof(FusedSmem2<Codec>);
  static_assert(smem <= 232448, "fused kernel shared memory exceeds the 227 KiB per-CTA limit");
  static std::atomic<uint64_t> configured{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured.load() & (1ull << (dev & 63)))) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured.fetch_or(1ull << (dev & 63));
  }
  const uint64_t cap = static_cast<uint64_t>(fused_capacity(k, kFThreads2, smem));
  const uint64_t cap_ack = cap < kAckIdx ? cap : kAckIdx;
  const int grid = static_cast<int>(nseg < cap_ack ? nseg : cap_ack);
  FusedParams q = p;
  if (q.step_segs == 0) {  // auto: about three published steps per phase per CTA, 2..16 segments each
    const uint64_t myseg = (nseg + grid - 1) / grid;
    const uint64_t s = (myseg + 2) / 3;
    q.step_segs = static_cast<uint32_t>(s < 2 ? 2 : (s > 16 ? 16 : s));
  }
  if (q.first_segs == 0) q.first_segs = q.step_segs;
  void* args[] = {&q};
  count_launch();
  if (p.debug & 64) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kFThreads2, smem);
    std::fprintf(stderr, "hccx fused launch rank %d: op %d n_chunk %llu nseg %llu cap %llu grid %d smem %u occ %d\n",
                 p.rank, p.op, static_cast<unsigned long long>(p.n_chunk), static_cast<unsigned long long>(nseg),
                 static_cast<unsigned long long>(cap), grid, smem, b);
  }
  return cudaLaunchCooperativeKernel(k, dim3(grid), dim3(kFThreads2), args, smem, stream);
}

}  // namespace hccx
