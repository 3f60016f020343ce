// fused_launch.cuh -- cooperative launch of the NVLink-engine kernels
// (ring_fused_kernel / oneshot_allreduce_kernel and their virtual-rank
// twins); included by the per-rate-range translation units.
#pragma once
#include <atomic>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include "oneshot.cuh"
#include "ring_fused.cuh"

namespace hccx {

// Co-resident CTAs of the fused kernel on this device (cooperative-launch cap).
int fused_capacity(const void* kernel, int threads, uint32_t smem);

// CTAs per rank: every rank of a communicator must use the same grid (CTA b
// of a rank only talks to CTA b of its peers), so the cap shared by all
// ranks (P.max_grid, set for single-process communicators) wins over this
// device's own capacity split over its nv virtual ranks.
inline uint64_t rank_grid_cap(const FusedParams& p, uint64_t cap, int nv) {
  uint64_t g = cap / static_cast<uint64_t>(nv);
  if (p.max_grid && p.max_grid < g) g = p.max_grid;
  if (g > kAckIdx) g = kAckIdx;
  return g < 1 ? 1 : g;
}

inline cudaError_t launch_ranks(const void* kernel_1, const void* kernel_v, const FusedParams* P, int nv, uint32_t G, int threads,
                         uint32_t smem, cudaStream_t stream) {
  count_launch();
  if (nv == 1) {
    void* args[] = {const_cast<FusedParams*>(P)};
    // One rank per GPU: a CTA only ever waits on CTAs of OTHER GPUs, so a
    // plain launch is enough (every CTA runs once its GPU has a free SM);
    // HCCX_COOP=1 keeps the cooperative launch (co-residency guaranteed).
    const char* e = std::getenv("HCCX_COOP");
    if (!(e && e[0] == '1')) {
      // HCCX_PDL=1: programmatic stream serialization -- the grid is
      // scheduled while the previous kernel of the stream drains (the kernel
      // waits for it with griddepcontrol.wait before touching memory).
      // Measured (profiles/r02_small_pdl.jsonl): 4 KiB 0.9-1.5 us faster,
      // 64-256 KiB 0.4-0.6 us slower, 256 MiB flat -- off by default.
      const char* pe = std::getenv("HCCX_PDL");
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = (pe && pe[0] == '1') ? 1 : 0;
      return cudaLaunchKernelExC(&cfg, kernel_1, args);
    }
    return cudaLaunchCooperativeKernel(kernel_1, dim3(G), dim3(threads), args, smem,
                                       stream);
  }
  static thread_local VParams V;  // copied into the launch's parameter buffer at the call
  for (int v = 0; v < nv; ++v) V.r[v] = P[v];
  V.G = G;
  void* args[] = {&V};
  return cudaLaunchCooperativeKernel(kernel_v, dim3(G * static_cast<uint32_t>(nv)),
                                     dim3(threads), args, smem, stream);
}

template <class Codec>
cudaError_t launch_oneshot_codec(const FusedParams* P, int nv, cudaStream_t stream) {
  const uint64_t groups = (P[0].n_chunk + kGroupVals - 1) / kGroupVals;
  if (groups == 0) return cudaSuccess;
  const void* kv = reinterpret_cast<const void*>(&oneshot_allreduce_vkernel<Codec>);
  // co-resident (cooperative) so no CTA waits on a peer while another CTA of
  // this launch is still queued; ~2 groups per CTA, at most one CTA per SM
  uint64_t cap = static_cast<uint64_t>(fused_capacity(kv, kOsWarps * 32, 0));
  cap = cap < 148 ? cap : 148;
  // groups per CTA (HCCX_OS_GPC, development knob). Measured at p = 4,
  // 64 KiB-256 KiB (profiles/r02_small_p4_gpc.jsonl): 2 groups per CTA
  // 1.07-1.15x faster than 8 (more CTAs pull peer data in parallel), 1 flat.
  const char* ge = std::getenv("HCCX_OS_GPC");
  const uint64_t gpc = ge && std::atoi(ge) > 0 ? static_cast<uint64_t>(std::atoi(ge)) : 2u;
  uint64_t grid = (groups + gpc - 1) / gpc;
  const uint64_t lim = rank_grid_cap(P[0], cap, nv);
  grid = grid < lim ? grid : lim;
  return launch_ranks(reinterpret_cast<const void*>(&oneshot_allreduce_kernel<Codec>), kv, P, nv,
                      static_cast<uint32_t>(grid), kOsWarps * 32, 0, stream);
}

// Launch one collective (or one pass of it) for the nv ranks P[0..nv) that
// live on the current device: one cooperative kernel either way.
template <class Codec>
cudaError_t launch_fused_codec(const FusedParams* P, int nv, cudaStream_t stream) {
  if (nv < 1 || nv > kMaxRanks) return cudaErrorInvalidValue;
  if (P[0].op == kFOneShotAllReduce) return launch_oneshot_codec<Codec>(P, nv, stream);
  const uint64_t groups = (P[0].n_chunk + kGroupVals - 1) / kGroupVals;
  const uint64_t nseg = (groups + kSegGroups - 1) / kSegGroups;
  if (nseg == 0) return cudaSuccess;
  constexpr uint32_t smem = sizeof(FusedSmem2<Codec>);
  static_assert(smem <= 232448, "fused kernel shared memory exceeds the 227 KiB per-CTA limit");
  const void* k1 = reinterpret_cast<const void*>(&ring_fused_kernel<Codec>);
  const void* kv = reinterpret_cast<const void*>(&ring_fused_vkernel<Codec>);
  static std::atomic<uint64_t> configured{0};  // one bit per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(configured.load() & (1ull << (dev & 63)))) {
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    configured.fetch_or(1ull << (dev & 63));
  }
  const uint64_t cap = static_cast<uint64_t>(fused_capacity(nv == 1 ? k1 : kv, kFThreads2, smem));
  const uint64_t gcap = rank_grid_cap(P[0], cap, nv);
  const uint32_t grid = static_cast<uint32_t>(nseg < gcap ? nseg : gcap);
  FusedParams q[kMaxRanks];
  for (int v = 0; v < nv; ++v) {
    q[v] = P[v];
    q[v].ack_span = static_cast<uint32_t>(gcap);
    if (q[v].step_segs == 0) {
      // auto: ~16 published steps per phase per CTA, 1..8 segments each.
      // Measured (tools/nvl_ab.py, 256 MiB r8): p = 4 1.07-1.10x faster
      // with 1-2 segment steps than with 3 steps per phase (consumers start
      // earlier; the signaller batches its system fences); p = 2 flat.
      const uint64_t myseg = (nseg + grid - 1) / grid;
      const uint64_t s = (myseg + 15) / 16;
      q[v].step_segs = static_cast<uint32_t>(s < 1 ? 1 : (s > 8 ? 8 : s));
    }
    if (q[v].first_segs == 0) q[v].first_segs = q[v].step_segs;
  }
  if (P[0].debug & 64) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, nv == 1 ? k1 : kv, kFThreads2, smem);
    std::fprintf(stderr, "hccx fused launch rank %d (+%d virtual): op %d n_chunk %llu nseg %llu cap %llu grid %u smem %u occ %d\n",
                 P[0].rank, nv - 1, P[0].op, static_cast<unsigned long long>(P[0].n_chunk),
                 static_cast<unsigned long long>(nseg), static_cast<unsigned long long>(cap), grid, smem, b);
  }
  return launch_ranks(k1, kv, q, nv, grid, kFThreads2, smem, stream);
}

}  // namespace hccx
