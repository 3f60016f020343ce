// rng.hpp -- hcc::Rng for the B200 drop-in: the reference's deterministic
// synthetic-data stream (proj/include/hcc/rng.hpp:14-40).  The bench and the
// parity tests draw their fp32 "gradients" from it, so GPU and CPU sides see
// identical inputs for a given seed.
//
// Stream contract (must match bit for bit):
//   engine    std::mt19937_64(seed)           -- fully specified by the standard
//   uniform() top 24 bits of one draw x 2^-24  -- exact float in [0, 1)
//   normal()  Box-Muller on two uniforms, u1 floored at 2^-24, float math
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

namespace hcc {

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : engine_(seed) {}

  std::uint64_t next_u64() { return engine_(); }
  std::uint32_t next_u32() { return static_cast<std::uint32_t>(engine_() >> 32); }

  float uniform() {
    constexpr float kInv24 = 1.0f / 16777216.0f;  // 2^-24
    return static_cast<float>(engine_() >> 40) * kInv24;
  }
  float uniform(float lo, float hi) { return lo + (hi - lo) * uniform(); }

  float normal() {
    constexpr float kFloor = 1.0f / 16777216.0f;
    constexpr float kTwoPi = 6.2831853071795864769f;
    float a = uniform();
    const float b = uniform();
    a = a < kFloor ? kFloor : a;
    const float radius = std::sqrt(-2.0f * std::log(a));
    return radius * std::cos(kTwoPi * b);
  }

 private:
  std::mt19937_64 engine_;
};

}  // namespace hcc
