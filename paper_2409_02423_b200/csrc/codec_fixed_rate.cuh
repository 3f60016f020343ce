// codec_fixed_rate.cuh -- the reference's FixedRate block quantizer as a
// warp-cooperative sm_100a codec.
//
// Format (bit-exact with /root/reference/proj/src/codec_kernels.hpp:85-163):
//   64-value blocks, block b at byte b*(1+8R); byte 0 = E_b (max IEEE exponent
//   field of the block, 0 for all-zero/denormal); then 64 fields of R bits,
//   LSB-first, field = clamp(RNE(v / 2^(E_b-127-R+2))) + 2^(R-1).
//
// Warp mapping: one warp owns a *group* of 4 blocks (256 values, 4*(1+8R)
// bytes -- a whole number of 32-bit words).  Lane L holds values 8l..8l+7 of
// block k = L/8 (l = L%8), i.e. one 256-bit load per lane, and packs its 8
// fields into R contiguous bytes of the block's data.
//
// Arithmetic (no fp64 divide, no llrint):
//   * E_b = max over the block of (bits & 0x7f800000), a shuffle-xor max over
//     the 8 lanes of the block; field 255 flags NaN/Inf.
//   * x = v * 2^(R-2-E) is exact in fp32 (split into two power-of-two
//     multiplies when the factor exceeds 2^127; underflow only happens when
//     |x| < 2^-126, which rounds to 0 either way).
//   * R <= 22: RNE via one FFMA with the 1.5*2^23 magic constant (|x| <=
//     2^21, single rounding); R > 22: cvt.rni on the exact product.
//   * decode: (float)q is exact for R <= 25, so q*2^k with one rounding
//     (split multiply in the subnormal range) equals the reference's
//     (float)((double)q*step); R >= 26 uses fp64 then one fp32 rounding.
#pragma once
#include "device_common.cuh"

namespace hccx {

template <int R>
struct FixedRateCodec {
  static_assert(R >= 2 && R <= 32, "rate out of range");
  static constexpr int kKind = 2;
  static constexpr int kRate = R;
  static constexpr bool kCheckFinite = true;
  static constexpr uint32_t kBlockBytes = 1 + 8 * R;
  static constexpr uint32_t kGroupBytes = 4 * kBlockBytes;  // 256 values
  static constexpr int kWords = (R + 3) / 4;                // lane chunk (R bytes) in words
  static constexpr bool kFastPath = (R % 4) == 0;
  static constexpr bool kNeedsInit = false;
  __device__ __forceinline__ static void kernel_init() {}
  static constexpr uint32_t kBias = 1u << (R - 1);
  static constexpr uint32_t kMask = R == 32 ? 0xffffffffu : ((1u << R) - 1u);

  __host__ __device__ static uint64_t wire_bytes(uint64_t n) {
    return ((n + 63) / 64) * static_cast<uint64_t>(kBlockBytes);
  }
  // Bytes that exist for a group holding `live` (<= 256) values.
  __host__ __device__ static uint32_t group_bytes_live(uint32_t live) {
    return ((live + 63) / 64) * kBlockBytes;
  }

  struct Lane {
    uint32_t d[kWords];  // 8 fields, LSB-first
    uint32_t hdr;        // E_b of this lane's block
  };

  // ---- quantize / dequantize (lane-local + 3 shuffles) --------------------

  // Field i of the lane chunk (R bits at bit offset i*R).
  __device__ __forceinline__ static uint32_t field(const Lane& s, int i) {
    const int off = i * R, w = off >> 5, b = off & 31;
    uint32_t u = s.d[w] >> b;
    if (b + R > 32) u |= s.d[w + 1] << (32 - b);
    return u & kMask;
  }

  // 0x4B000000 | u as a float is exactly 2^23 + u (u < 2^23): the
  // dequantisation q*2^k = (2^23+u)*2^k - (2^23+bias)*2^k is then ONE FFMA
  // with a single rounding of the exact value (fma has no intermediate
  // rounding or overflow).  R = 8 / 16 build it with one PRMT.
  __device__ __forceinline__ static float magic_field(const Lane& s, int i) {
    if constexpr (R == 8) {
      return __uint_as_float(__byte_perm(s.d[i >> 2], 0x4B000000u, 0x7650u | (i & 3)));
    } else if constexpr (R == 16) {
      return __uint_as_float(__byte_perm(s.d[i >> 1], 0x4B000000u, 0x7600u | (((i & 1) * 2 + 1) << 4) | ((i & 1) * 2)));
    } else {
      return __uint_as_float(field(s, i) | 0x4B000000u);
    }
  }

  __device__ __forceinline__ static void pack(Lane& s, const uint32_t (&u)[8]) {
    if constexpr (R == 8) {
      s.d[0] = __byte_perm(__byte_perm(u[0], u[1], 0x0040u), __byte_perm(u[2], u[3], 0x0040u), 0x5410u);
      s.d[1] = __byte_perm(__byte_perm(u[4], u[5], 0x0040u), __byte_perm(u[6], u[7], 0x0040u), 0x5410u);
    } else if constexpr (R == 16) {
#pragma unroll
      for (int w = 0; w < 4; ++w) s.d[w] = __byte_perm(u[2 * w], u[2 * w + 1], 0x5410u);
    } else {
#pragma unroll
      for (int w = 0; w < kWords; ++w) s.d[w] = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int off = i * R, w = off >> 5, b = off & 31;
        s.d[w] |= u[i] << b;
        if (b + R > 32) s.d[w + 1] |= u[i] >> (32 - b);
      }
    }
  }

  __device__ __forceinline__ static void encode(const float (&v)[8], Lane& s, uint32_t& bad, uint32_t /*lane_live*/) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) m = max(m, __float_as_uint(v[i]) & 0x7f800000u);
    m = max(m, __shfl_xor_sync(kFull, m, 1));
    m = max(m, __shfl_xor_sync(kFull, m, 2));
    m = max(m, __shfl_xor_sync(kFull, m, 4));
    const int eb = static_cast<int>(m >> 23);
    bad |= static_cast<uint32_t>(eb == 255);
    s.hdr = static_cast<uint32_t>(eb);
    const int k = R + 125 - eb;  // x = v * 2^k, k in [R-130, R+125]
    uint32_t u[8];
    if (__all_sync(kFull, k >= -126 && k <= 127)) {
      // common case: 2^k is a normal float, one rounding per value
      const float sb = __uint_as_float(static_cast<uint32_t>(k + 127) << 23);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if constexpr (R <= 22) {
          const float y = __fmaf_rn(v[i], sb, 12582912.0f);  // 1.5 * 2^23
          u[i] = min(__float_as_uint(y) - (0x4B400000u - kBias), kMask);
        } else {
          u[i] = min(static_cast<uint32_t>(__float2int_rn(__fmul_rn(v[i], sb))) + kBias, kMask);
        }
      }
    } else {
      // tiny blocks (2^k > 2^127: two exact power-of-two multiplies) and
      // the denormal factor 2^-127 (R = 2, E_b = 254)
      const bool split = k > 127;
      const float sa = split ? exp2i(64) : 1.0f;
      const float sb = exp2i(split ? k - 64 : max(k, -149));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float t = __fmul_rn(v[i], sa);
        if constexpr (R <= 22) {
          const float y = __fmaf_rn(t, sb, 12582912.0f);
          u[i] = min(__float_as_uint(y) - (0x4B400000u - kBias), kMask);
        } else {
          u[i] = min(static_cast<uint32_t>(__float2int_rn(__fmul_rn(t, sb))) + kBias, kMask);
        }
      }
    }
    pack(s, u);
  }

  __device__ __forceinline__ static void decode(const Lane& s, float (&v)[8]) {
    const int k = static_cast<int>(s.hdr) - 125 - R;  // step = 2^k, k in [-125-R, 129-R]
    if constexpr (R <= 22) {
      if (__all_sync(kFull, k >= -126 && k <= 103)) {
        const float step = __uint_as_float(static_cast<uint32_t>(k + 127) << 23);
        const float c = __fmul_rn(-(8388608.0f + static_cast<float>(kBias)), step);  // exact
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __fmaf_rn(magic_field(s, i), step, c);
        return;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = static_cast<int>(field(s, i) - kBias);
      if constexpr (R <= 25) {
        const bool split = k < -126;
        const float sa = exp2i(split ? k + 64 : k);
        const float sb = split ? exp2i(-64) : 1.0f;
        v[i] = __fmul_rn(__fmul_rn(static_cast<float>(q), sa), sb);
      } else {
        const double step = __longlong_as_double(static_cast<long long>(k + 1023) << 52);
        v[i] = __double2float_rn(__dmul_rn(static_cast<double>(q), step));
      }
    }
  }

  // ---- group stream I/O ---------------------------------------------------
  // Group stream = [H0][D0: 8R B][H1][D1][H2][D2][H3][D3] = 8R+1 words.
  // Block k's data starts at byte 8Rk + k + 1, i.e. misaligned by a = k+1
  // bytes for k < 3 and word-aligned for k = 3.

  // Full group, R % 4 == 0, 4-byte-aligned destination: every lane emits R/4
  // whole words with funnel shifts (plus the boundary word carrying the next
  // block's header); lane 0 also emits word 0.
  __device__ __forceinline__ static void store_fast(const Lane& s, uint32_t* gw, int lane) {
    store_words<0>(s, gw, lane);
  }
  // Same layout into shared memory (or any generic address).
  __device__ __forceinline__ static void store_fast_generic(const Lane& s, uint32_t* gw, int lane) {
    store_words<2>(s, gw, lane);
  }

  template <int kDst>
  __device__ __forceinline__ static void store_words(const Lane& s, uint32_t* gw, int lane) {
    static_assert(kFastPath, "fast path needs R % 4 == 0");
    constexpr int R4 = R / 4;
    const int k = lane >> 3, l = lane & 7;
    const uint32_t nxt0 = __shfl_down_sync(kFull, s.d[0], 1);
    const uint32_t nxth = __shfl_down_sync(kFull, s.hdr, 1);
    if (k < 3) {
      const int a = k + 1;
      uint32_t* dst = gw + 2 * R * k + R4 * l + 1;
#pragma unroll
      for (int q = 1; q < R4; ++q) st_word<kDst>(dst + q - 1, __funnelshift_r(s.d[q - 1], s.d[q], 8 * (4 - a)));
      uint32_t last;
      if (l < 7) {
        last = __funnelshift_r(s.d[R4 - 1], nxt0, 8 * (4 - a));
      } else {
        last = (s.d[R4 - 1] >> (8 * (4 - a))) | (nxth << (8 * a));
        if (a < 3) last |= nxt0 << (8 * (a + 1));
      }
      st_word<kDst>(dst + R4 - 1, last);
      if (lane == 0) st_word<kDst>(gw, s.hdr | (s.d[0] << 8));
    } else {
      uint32_t* dst = gw + 6 * R + 1 + R4 * l;
#pragma unroll
      for (int q = 0; q < R4; ++q) st_word<kDst>(dst + q, s.d[q]);
    }
  }

  // Fast-path loads are split so a warp can put several groups' loads in
  // flight before it assembles any of them (memory-level parallelism).
  struct Raw {
    uint32_t w[kFastPath ? R / 4 : 1];
    uint32_t w0;
  };

  template <int kSrc>
  __device__ __forceinline__ static void load_raw(Raw& r, const uint32_t* gw, int lane) {
    static_assert(kFastPath, "fast path needs R % 4 == 0");
    constexpr int R4 = R / 4;
    const int k = lane >> 3, l = lane & 7;
    const uint32_t* src = (k < 3) ? gw + 2 * R * k + R4 * l + 1 : gw + 6 * R + 1 + R4 * l;
#pragma unroll
    for (int q = 0; q < R4; ++q) r.w[q] = ld_word<kSrc>(src + q);
    r.w0 = (lane == 0) ? ld_word<kSrc>(gw) : 0u;
  }

  __device__ __forceinline__ static void assemble(Lane& s, const Raw& r, int lane) {
    constexpr int R4 = R / 4;
    const int k = lane >> 3;
    uint32_t prev = __shfl_up_sync(kFull, r.w[R4 - 1], 1);
    if (lane == 0) prev = r.w0;
    const uint32_t hsrc = __shfl_sync(kFull, lane == 0 ? r.w0 : r.w[R4 - 1], k == 0 ? 0 : 8 * k - 1);
    s.hdr = (hsrc >> (8 * k)) & 0xffu;
    if (k < 3) {
      const int a = k + 1;
      s.d[0] = __funnelshift_r(prev, r.w[0], 8 * a);
#pragma unroll
      for (int q = 1; q < R4; ++q) s.d[q] = __funnelshift_r(r.w[q - 1], r.w[q], 8 * a);
    } else {
#pragma unroll
      for (int q = 0; q < R4; ++q) s.d[q] = r.w[q];
    }
  }

  template <bool kStream>
  __device__ __forceinline__ static void load_fast(Lane& s, const uint32_t* gw, int lane) {
    Raw r;
    load_raw<kStream ? 0 : 1>(r, gw, lane);
    assemble(s, r, lane);
  }

  // Any rate / partial group: bytes staged through this warp's shared
  // memory slice `sm` (>= kGroupBytes + 4 bytes, 4-byte aligned).
  __device__ __forceinline__ static void to_stage(const Lane& s, uint8_t* sm, int lane) {
    const int k = lane >> 3, l = lane & 7;
    uint8_t* base = sm + k * kBlockBytes;
    if (l == 0) base[0] = static_cast<uint8_t>(s.hdr);
    uint8_t* c = base + 1 + l * R;
#pragma unroll
    for (int m = 0; m < R; ++m) c[m] = static_cast<uint8_t>(s.d[m >> 2] >> (8 * (m & 3)));
  }

  __device__ __forceinline__ static void from_stage(Lane& s, const uint8_t* sm, int lane) {
    const int k = lane >> 3, l = lane & 7;
    const uint8_t* base = sm + k * kBlockBytes;
    s.hdr = base[0];
    const uint8_t* c = base + 1 + l * R;
#pragma unroll
    for (int w = 0; w < kWords; ++w) s.d[w] = 0;
#pragma unroll
    for (int m = 0; m < R; ++m) s.d[m >> 2] |= static_cast<uint32_t>(c[m]) << (8 * (m & 3));
  }
};

}  // namespace hccx
