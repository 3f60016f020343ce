// codec_identity.cuh -- Identity codec (raw fp32 bytes) in the warp-group
// form used by every hccx kernel.  Reference: src/codec_serial.cpp:20-25
// (payload = memcpy of the input).  In the ring kernels this makes the
// uncompressed ring: the per-hop add is the reference's acc = rx + acc.
#pragma once
#include "device_common.cuh"

namespace hccx {

struct IdentityCodec {
  static constexpr int kKind = 0;
  static constexpr int kRate = 0;
  static constexpr bool kCheckFinite = false;
  static constexpr uint32_t kGroupBytes = 4 * kGroupVals;
  static constexpr int kWords = 8;
  static constexpr bool kFastPath = true;
  static constexpr bool kNeedsInit = false;
  __device__ __forceinline__ static void kernel_init() {}

  __host__ __device__ static uint64_t wire_bytes(uint64_t n) { return 4 * n; }
  __host__ __device__ static uint32_t group_bytes_live(uint32_t live) { return 4 * live; }

  struct Lane {
    uint32_t d[8];
    uint32_t hdr;
  };

  __device__ __forceinline__ static void encode(const float (&v)[8], Lane& s, uint32_t&, uint32_t /*lane_live*/) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s.d[i] = __float_as_uint(v[i]);
    s.hdr = 0;
  }
  __device__ __forceinline__ static void decode(const Lane& s, float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(s.d[i]);
  }
  // fast path: 32-byte aligned payload
  __device__ __forceinline__ static void store_fast(const Lane& s, uint32_t* gw, int lane) {
    float v[8];
    decode(s, v);
    stg8(reinterpret_cast<float*>(gw) + 8 * lane, v);
  }
  struct Raw {
    float v[8];
  };
  __device__ __forceinline__ static void store_fast_generic(const Lane& s, uint32_t* gw, int lane) {
    uint4* w = reinterpret_cast<uint4*>(gw + 8 * lane);
    w[0] = make_uint4(s.d[0], s.d[1], s.d[2], s.d[3]);
    w[1] = make_uint4(s.d[4], s.d[5], s.d[6], s.d[7]);
  }
  template <int kSrc>
  __device__ __forceinline__ static void load_raw(Raw& r, const uint32_t* gw, int lane) {
    ld_vals<kSrc>(reinterpret_cast<const float*>(gw) + 8 * lane, r.v);
  }
  __device__ __forceinline__ static void assemble(Lane& s, const Raw& r, int) {
    uint32_t dummy = 0;
    encode(r.v, s, dummy, 8);
  }
  template <bool kStream>
  __device__ __forceinline__ static void load_fast(Lane& s, const uint32_t* gw, int lane) {
    Raw r;
    load_raw<kStream ? 0 : 1>(r, gw, lane);
    assemble(s, r, lane);
  }
  __device__ __forceinline__ static void to_stage(const Lane& s, uint8_t* sm, int lane) {
    uint32_t* w = reinterpret_cast<uint32_t*>(sm) + 8 * lane;
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = s.d[i];
  }
  __device__ __forceinline__ static void from_stage(Lane& s, const uint8_t* sm, int lane) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(sm) + 8 * lane;
#pragma unroll
    for (int i = 0; i < 8; ++i) s.d[i] = w[i];
    s.hdr = 0;
  }
};

}  // namespace hccx
