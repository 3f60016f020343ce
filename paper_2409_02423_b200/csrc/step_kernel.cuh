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

template <class Codec, int kOp>
__global__ void __launch_bounds__(kStepThreads) step_kernel(const __grid_constant__ StepParams P) {
  __shared__ __align__(16) uint8_t stage[kStepWarps][kStageBytes];
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const uint64_t ngroups = (P.n + kGroupVals - 1) / kGroupVals;
  uint32_t bad = 0;
  for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * kStepWarps + warp; g < ngroups;
       g += static_cast<uint64_t>(gridDim.x) * kStepWarps) {
    for (int j = 0; j < P.njobs; ++j)
      step_group<Codec, kOp, true>(P.jobs[j], g, P.n, P.vec_ok, P.fast_ok, P.div_mode, P.recip,
                                   P.divisor, stage[warp], lane, bad);
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

}  // namespace hccx
