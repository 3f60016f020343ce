// step_kernel.cuh -- the one streaming kernel behind the codec entry points and
// every stage of the single-device ring (virtual ranks).
//
// A "step" applies one operation to up to kMaxJobs independent chunks of n
// values, one warp per 256-value group, grid-stride over groups:
//
//   kOpEncode     floats -> payload                      compress; ring send 0;
//                                                        allgather origin compress
//   kOpDecode     payload -> floats (x nouts, / divisor) decompress; allgather
//                                                        delivery; p2p receive
//   kOpDAR        payload + local floats -> payload      fused decompress-add-
//                 (+ decoded copy / divisor)             recompress ring hop
//   kOpDecodeAdd  payload + local floats -> floats       last reduce-scatter hop
//
// The add is acc = received + local with no FMA contraction (the reference
// builds with -ffp-contract=off, proj/CMakeLists.txt:15-17, and adds at
// src/collectives.cpp:50-52).  Average mode divides by float(p) after the
// gather (src/collectives.cpp:234-239): an exact reciprocal multiply when p
// is a power of two, else an IEEE divide.
#pragma once
#include "device_common.cuh"
#include "hccx_kernels.h"

namespace hccx {

constexpr int kStepThreads = 256;
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStageBytes = 1056;  // >= largest group (4*(1+8*32) = 1028) + slack, 16B multiple

__device__ __forceinline__ void copy_out_bytes(const uint8_t* sm, uint8_t* dst, uint32_t nb, int lane) {
  if ((reinterpret_cast<uintptr_t>(dst) & 3u) == 0) {
    const uint32_t nw = nb >> 2;
    for (uint32_t w = lane; w < nw; w += 32)
      reinterpret_cast<uint32_t*>(dst)[w] = reinterpret_cast<const uint32_t*>(sm)[w];
    for (uint32_t b = (nw << 2) + lane; b < nb; b += 32) dst[b] = sm[b];
  } else {
    for (uint32_t b = lane; b < nb; b += 32) dst[b] = sm[b];
  }
}

__device__ __forceinline__ void copy_in_bytes(uint8_t* sm, const uint8_t* src, uint32_t nb,
                                              uint32_t cap, int lane) {
  if ((reinterpret_cast<uintptr_t>(src) & 3u) == 0) {
    const uint32_t nw = nb >> 2;
    for (uint32_t w = lane; w < nw; w += 32)
      reinterpret_cast<uint32_t*>(sm)[w] = ldg_u32_coherent(reinterpret_cast<const uint32_t*>(src) + w);
    for (uint32_t b = (nw << 2) + lane; b < nb; b += 32) sm[b] = src[b];
  } else {
    for (uint32_t b = lane; b < nb; b += 32) sm[b] = src[b];
  }
  for (uint32_t b = nb + lane; b < cap; b += 32) sm[b] = 0;
}

// Per-lane value I/O: lane owns values [base + 8*lane, base + 8*lane + 8).
template <bool kStream>
__device__ __forceinline__ void load_vals(const float* src, uint64_t base, uint32_t live, bool vec,
                                          int lane, float (&v)[8]) {
  if (vec && live == kGroupVals) {
    if (kStream)
      ldg8_stream(src + base + 8 * lane, v);
    else
      ldg8_coherent(src + base + 8 * lane, v);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t e = 8 * lane + i;
      v[i] = e < live ? src[base + e] : 0.0f;
    }
  }
}

__device__ __forceinline__ void store_vals(float* dst, uint64_t base, uint32_t live, bool vec, int lane,
                                           const float (&v)[8]) {
  if (vec && live == kGroupVals) {
    stg8(dst + base + 8 * lane, v);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t e = 8 * lane + i;
      if (e < live) dst[base + e] = v[i];
    }
  }
}

__device__ __forceinline__ void apply_div(float (&v)[8], int mode, float recip, float divisor) {
  if (mode == 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fmul_rn(v[i], recip);
  } else if (mode == 2) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fdiv_rn(v[i], divisor);
  }
}

template <class Codec, bool kStream>
__device__ __forceinline__ void group_store(const typename Codec::Lane& s, uint8_t* dst, uint32_t live,
                                            bool fast, uint8_t* sm, int lane) {
  if constexpr (Codec::kFastPath) {
    if (fast && live == kGroupVals) {
      Codec::store_fast(s, reinterpret_cast<uint32_t*>(dst), lane);
      return;
    }
  }
  Codec::to_stage(s, sm, lane);
  __syncwarp();
  copy_out_bytes(sm, dst, Codec::group_bytes_live(live), lane);
  __syncwarp();
}

template <class Codec, bool kStream>
__device__ __forceinline__ void group_load(typename Codec::Lane& s, const uint8_t* src, uint32_t live,
                                           bool fast, uint8_t* sm, int lane) {
  if constexpr (Codec::kFastPath) {
    if (fast && live == kGroupVals) {
      Codec::template load_fast<kStream>(s, reinterpret_cast<const uint32_t*>(src), lane);
      return;
    }
  }
  copy_in_bytes(sm, src, Codec::group_bytes_live(live), Codec::kGroupBytes, lane);
  __syncwarp();
  Codec::from_stage(s, sm, lane);
  __syncwarp();
}

__device__ __forceinline__ uint32_t lane_live(uint32_t live, int lane) {
  const int r = static_cast<int>(live) - 8 * lane;
  return static_cast<uint32_t>(r < 0 ? 0 : (r > 8 ? 8 : r));
}

// One group of one job.  Returns the non-finite flag contribution in `bad`.
template <class Codec, int kOp, bool kStream>
__device__ __forceinline__ void step_group(const StepJob& J, uint64_t g, uint64_t n, bool vec,
                                           bool fast, int div_mode, float recip, float divisor,
                                           uint8_t* sm, int lane, uint32_t& bad) {
  const uint64_t base = g * kGroupVals;
  const uint32_t live = static_cast<uint32_t>(n - base < kGroupVals ? n - base : kGroupVals);
  const uint64_t goff = g * static_cast<uint64_t>(Codec::kGroupBytes);
  typename Codec::Lane s;
  float v[8];
  if constexpr (kOp == kOpEncode) {
    load_vals<kStream>(static_cast<const float*>(J.src), base, live, vec, lane, v);
    Codec::encode(v, s, bad, lane_live(live, lane));
    group_store<Codec, kStream>(s, static_cast<uint8_t*>(J.dst) + goff, live, fast, sm, lane);
  } else {
    group_load<Codec, kStream>(s, static_cast<const uint8_t*>(J.src) + goff, live, fast, sm, lane);
    Codec::decode(s, v);
    if constexpr (kOp == kOpDecode) {
      apply_div(v, div_mode, recip, divisor);
      for (int o = 0; o < J.nouts; ++o) store_vals(J.outs[o], base, live, vec, lane, v);
    } else {
      float loc[8];
      load_vals<kStream>(J.local, base, live, vec, lane, loc);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], loc[i]);
      if constexpr (kOp == kOpDecodeAdd) {
        store_vals(static_cast<float*>(J.dst), base, live, vec, lane, v);
      } else {
        Codec::encode(v, s, bad, lane_live(live, lane));
        group_store<Codec, kStream>(s, static_cast<uint8_t*>(J.dst) + goff, live, fast, sm, lane);
        if (J.nouts > 0) {
          Codec::decode(s, v);
          apply_div(v, div_mode, recip, divisor);
          store_vals(J.outs[0], base, live, vec, lane, v);
        }
      }
    }
  }
}

// Full groups with aligned pointers: U groups per warp iteration, all of
// their loads issued before any group is assembled, so each warp keeps
// U x 1 KiB (Encode) or U x (payload + 1 KiB) (DAR) in flight.
template <int kOp>
struct StepUnroll {
  static constexpr int value = (kOp == kOpEncode || kOp == kOpDecode) ? 4 : 2;
};

template <class Codec, int kOp, int U>
__device__ __forceinline__ void step_fast(const StepJob& J, uint64_t g0, uint64_t S, uint64_t nfull,
                                          int div_mode, float recip, float divisor, int lane,
                                          uint32_t& bad) {
  constexpr uint64_t GB = Codec::kGroupBytes;
  float v[U][8];
  float loc[U][8];
  typename Codec::Raw raw[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t g = g0 + u * S;
    if (g < nfull) {
      if constexpr (kOp == kOpEncode) {
        ldg8_stream(static_cast<const float*>(J.src) + g * kGroupVals + 8 * lane, v[u]);
      } else {
        Codec::template load_raw<0>(
            raw[u], reinterpret_cast<const uint32_t*>(static_cast<const uint8_t*>(J.src) + g * GB), lane);
        if constexpr (kOp == kOpDAR || kOp == kOpDecodeAdd)
          ldg8_stream(J.local + g * kGroupVals + 8 * lane, loc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t g = g0 + u * S;
    if (g >= nfull) continue;
    typename Codec::Lane s;
    const uint64_t vo = g * kGroupVals + 8 * lane;
    if constexpr (kOp == kOpEncode) {
      Codec::encode(v[u], s, bad, 8u);
      Codec::store_fast(s, reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(J.dst) + g * GB), lane);
    } else {
      Codec::assemble(s, raw[u], lane);
      float w[8];
      Codec::decode(s, w);
      if constexpr (kOp == kOpDecode) {
        apply_div(w, div_mode, recip, divisor);
        for (int o = 0; o < J.nouts; ++o) stg8(J.outs[o] + vo, w);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = __fadd_rn(w[i], loc[u][i]);
        if constexpr (kOp == kOpDecodeAdd) {
          stg8(static_cast<float*>(J.dst) + vo, w);
        } else {
          Codec::encode(w, s, bad, 8u);
          Codec::store_fast(s, reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(J.dst) + g * GB), lane);
          if (J.nouts > 0) {
            Codec::decode(s, w);
            apply_div(w, div_mode, recip, divisor);
            stg8(J.outs[0] + vo, w);
          }
        }
      }
    }
  }
}

template <class Codec, int kOp>
__global__ void __launch_bounds__(kStepThreads) step_kernel(const __grid_constant__ StepParams P) {
  __shared__ __align__(16) uint8_t stage[kStepWarps][kStageBytes];
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const uint64_t ngroups = (P.n + kGroupVals - 1) / kGroupVals;
  const uint64_t S = static_cast<uint64_t>(gridDim.x) * kStepWarps;
  const uint64_t wid = static_cast<uint64_t>(blockIdx.x) * kStepWarps + warp;
  uint32_t bad = 0;
  uint64_t g_generic = wid;
  if constexpr (Codec::kNeedsInit) {
    Codec::kernel_init();
    __syncthreads();
  }
  pdl_wait_and_release();
  if constexpr (Codec::kFastPath) {
    if (P.vec_ok && P.fast_ok) {
      constexpr int U = StepUnroll<kOp>::value;
      const uint64_t nfull = P.n / kGroupVals;
      for (uint64_t g0 = wid; g0 < nfull; g0 += S * U)
        for (int j = 0; j < P.njobs; ++j)
          step_fast<Codec, kOp, U>(P.jobs[j], g0, S, nfull, P.div_mode, P.recip, P.divisor, lane, bad);
      g_generic = nfull + wid;  // only the trailing partial group is left
    }
  }
  for (uint64_t g = g_generic; g < ngroups; g += S) {
    for (int j = 0; j < P.njobs; ++j)
      step_group<Codec, kOp, true>(P.jobs[j], g, P.n, P.vec_ok, P.fast_ok, P.div_mode, P.recip,
                                   P.divisor, stage[warp], lane, bad);
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

// ---------------------------------------------------------------------------
// TMA-staged streaming kernel (the production path for aligned buffers).
//
// 8 consumer warps + 1 producer warp per CTA, persistent over "tiles" of 8
// full groups of one job.  The producer's elected lane streams each tile's
// source bytes (payload and/or fp32) into a kTmaStages-deep shared-memory
// ring with cp.async.bulk, completing on a per-stage "full" mbarrier; every
// consumer warp decodes/encodes one group of the tile from shared memory,
// writes its result with coalesced global stores and arrives on the stage's
// "empty" mbarrier.  Loads are therefore always in flight (kTmaStages tiles per
// CTA) no matter what the consumers are computing.  Leftover groups (fewer
// than 8 at the end of a job, and the partial last group) use the per-warp
// path above.
// ---------------------------------------------------------------------------

#ifndef HCCX_TMA_STAGES
#define HCCX_TMA_STAGES 4
#endif
#ifndef HCCX_TMA_CONSUMERS
#define HCCX_TMA_CONSUMERS 8
#endif
constexpr int kTmaStages = HCCX_TMA_STAGES;
constexpr int kTmaConsumers = HCCX_TMA_CONSUMERS;
constexpr int kTmaThreads = (kTmaConsumers + 1) * 32;
constexpr int kTileGroups = kTmaConsumers;

template <class Codec, int kOp>
struct TmaLayout {
  static constexpr uint32_t kA = (kOp == kOpEncode ? 4u * kGroupVals : Codec::kGroupBytes) * kTileGroups;
  static constexpr uint32_t kAPad = (kA + 127u) / 128u * 128u;
  static constexpr uint32_t kB = (kOp == kOpDAR || kOp == kOpDecodeAdd) ? 4u * kGroupVals * kTileGroups : 0u;
  static constexpr uint32_t kStage = kAPad + kB;
  static constexpr uint32_t kBarOff = kStage * kTmaStages;
  static constexpr uint32_t kStageOff = kBarOff + 2 * 8 * kTmaStages;  // per-warp staging for leftovers
  static constexpr uint32_t kSmem = kStageOff + kTmaConsumers * kStageBytes;
};

template <class Codec, int kOp>
__device__ __forceinline__ void tma_group(const StepJob& J, uint64_t g, const uint8_t* a, const float* b,
                                          int div_mode, float recip, float divisor, int lane, uint32_t& bad) {
  constexpr uint64_t GB = Codec::kGroupBytes;
  typename Codec::Lane s;
  const uint64_t vo = g * kGroupVals + 8 * lane;
  if constexpr (kOp == kOpEncode) {
    float v[8];
    ld_vals<2>(reinterpret_cast<const float*>(a) + 8 * lane, v);
    Codec::encode(v, s, bad, 8u);
    Codec::store_fast(s, reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(J.dst) + g * GB), lane);
  } else {
    typename Codec::Raw raw;
    Codec::template load_raw<2>(raw, reinterpret_cast<const uint32_t*>(a), lane);
    Codec::assemble(s, raw, lane);
    float w[8];
    Codec::decode(s, w);
    if constexpr (kOp == kOpDecode) {
      apply_div(w, div_mode, recip, divisor);
      for (int o = 0; o < J.nouts; ++o) stg8(J.outs[o] + vo, w);
    } else {
      float loc[8];
      ld_vals<2>(b + 8 * lane, loc);
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = __fadd_rn(w[i], loc[i]);
      if constexpr (kOp == kOpDecodeAdd) {
        stg8(static_cast<float*>(J.dst) + vo, w);
      } else {
        Codec::encode(w, s, bad, 8u);
        Codec::store_fast(s, reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(J.dst) + g * GB), lane);
        if (J.nouts > 0) {
          Codec::decode(s, w);
          apply_div(w, div_mode, recip, divisor);
          stg8(J.outs[0] + vo, w);
        }
      }
    }
  }
}

template <class Codec, int kOp>
__global__ void __launch_bounds__(kTmaThreads) step_tma_kernel(const __grid_constant__ StepParams P) {
  using L = TmaLayout<Codec, kOp>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* empty = full + kTmaStages;
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const uint64_t nfull = P.n / kGroupVals;
  const uint64_t tiles_per_job = nfull / kTileGroups;
  const uint64_t total = tiles_per_job * static_cast<uint64_t>(P.njobs);
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTmaStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kTmaConsumers);
    }
    fence_mbar_init();
  }
  Codec::kernel_init();
  __syncthreads();
  // programmatic dependent launch: the barrier setup above overlapped the
  // previous kernel's tail; global memory is touched only after it finished
  pdl_wait_and_release();
  uint32_t bad = 0;
  // (job, tile) of this CTA's tiles t = blockIdx.x, +gridDim.x, ...: one
  // division up front, then carried (a 64-bit divide per tile cost ~14% of
  // the codec kernels' issue slots)
  const uint64_t t0 = blockIdx.x;
  const int j0 = total ? static_cast<int>(t0 / tiles_per_job) : 0;
  const uint64_t tile0 = total ? t0 - static_cast<uint64_t>(j0) * tiles_per_job : 0;
  auto advance = [&](int& j, uint64_t& tile) {
    tile += gridDim.x;
    while (tile >= tiles_per_job && j < P.njobs) {
      tile -= tiles_per_job;
      ++j;
    }
  };
  if (warp == kTmaConsumers) {
    if (lane == 0) {
      int st = 0;
      uint32_t phase = 0;
      int j = j0;
      uint64_t tile = tile0;
      for (uint64_t t = t0; t < total; t += gridDim.x, advance(j, tile)) {
        mbar_wait(&empty[st], phase ^ 1u);
        const StepJob& J = P.jobs[j];
        uint8_t* base = smem + st * L::kStage;
        mbar_arrive_expect_tx(&full[st], L::kA + L::kB);
        bulk_g2s(base, static_cast<const uint8_t*>(J.src) + tile * L::kA, L::kA, &full[st]);
        if constexpr (L::kB != 0)
          bulk_g2s(base + L::kAPad, reinterpret_cast<const uint8_t*>(J.local) + tile * L::kB, L::kB, &full[st]);
        if (++st == kTmaStages) {
          st = 0;
          phase ^= 1u;
        }
      }
    }
  } else {
    int st = 0;
    uint32_t phase = 0;
    constexpr uint32_t kAGroup = L::kA / kTileGroups;
    int j = j0;
    uint64_t tile = tile0;
    for (uint64_t t = t0; t < total; t += gridDim.x, advance(j, tile)) {
      mbar_wait(&full[st], phase);
      const uint8_t* base = smem + st * L::kStage;
      tma_group<Codec, kOp>(P.jobs[j], tile * kTileGroups + warp, base + warp * kAGroup,
                            reinterpret_cast<const float*>(base + L::kAPad) + warp * kGroupVals, P.div_mode,
                            P.recip, P.divisor, lane, bad);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == kTmaStages) {
        st = 0;
        phase ^= 1u;
      }
    }
    // leftovers: groups [tiles_per_job*8, ngroups) of every job
    const uint64_t ngroups = (P.n + kGroupVals - 1) / kGroupVals;
    const uint64_t first = tiles_per_job * kTileGroups;
    const uint64_t per_job = ngroups - first;
    const uint64_t wid = static_cast<uint64_t>(blockIdx.x) * kTmaConsumers + warp;
    uint8_t* sm = smem + L::kStageOff + warp * kStageBytes;
    for (uint64_t r = wid; r < per_job * P.njobs; r += static_cast<uint64_t>(gridDim.x) * kTmaConsumers) {
      const int j = static_cast<int>(r / per_job);
      step_group<Codec, kOp, true>(P.jobs[j], first + (r - j * per_job), P.n, P.vec_ok, P.fast_ok, P.div_mode,
                                   P.recip, P.divisor, sm, lane, bad);
    }
  }
  if constexpr (Codec::kCheckFinite) {
    if (warp < kTmaConsumers && __any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

}  // namespace hccx
