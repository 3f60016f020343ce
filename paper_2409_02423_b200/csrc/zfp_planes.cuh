// zfp_planes.cuh -- embedded bit-plane coder of the 1-D zfp block (4
// negabinary coefficients), one bit PLANE per step instead of one bit.
//
// The published coder walks each plane bit by bit: n coefficients are
// already significant and send their plane bit verbatim; the rest are coded
// by group tests ("any bit left?") followed by a unary run to the next
// significant coefficient, whose own 1 is implicit when it is the last one.
// Every bit decrements a budget of 4R-9 bits and the block stops mid-plane
// when it runs out.  With four coefficients a plane's codeword is at most 7
// bits and follows in closed form from (n, plane bits): one put per plane on
// the encode side, one 64-bit peek per plane on the decode side, and no
// per-bit data-dependent loops (the per-bit version diverged across the
// warp's lanes).  Budget truncation keeps the per-bit semantics exactly: the
// encoder emits the codeword's prefix; the decoder replays the truncated
// reads (tests/cpp/test_zfp_planes.cpp checks both against the per-bit loops
// exhaustively over planes and budgets).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define HCCX_HD __host__ __device__ __forceinline__
#else
#define HCCX_HD inline
#endif

namespace hccx {
namespace zfp_planes {

HCCX_HD uint32_t ctz32(uint32_t v) {  // v != 0
#if defined(__CUDA_ARCH__)
  return static_cast<uint32_t>(__ffs(static_cast<int>(v)) - 1);
#else
  return static_cast<uint32_t>(__builtin_ctz(v));
#endif
}

// Codeword of one plane (LSB-first bits in *code, length returned) given n
// significant coefficients and the plane's 4 bits x (coefficient i at bit
// i); *n_out = significant coefficients after the plane.
HCCX_HD uint32_t plane_code(uint32_t n, uint32_t x, uint32_t* code, uint32_t* n_out) {
  uint32_t c = x & ((1u << n) - 1u);
  uint32_t len = n;
  uint32_t y = x >> n;
  uint32_t pos = n;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    if (pos >= 4) break;
    if (y == 0) {  // group test: nothing left in this plane
      len += 1;
      break;
    }
    c |= 1u << len;  // group test: something left
    len += 1;
    const uint32_t z = ctz32(y);
    const uint32_t a = pos + z;
    if (a < 3) {  // z zeros, then the significant coefficient's 1
      c |= 1u << (len + z);
      len += z + 1;
    } else {  // zeros up to position 3, whose 1 is implicit
      len += 3 - pos;
    }
    const uint32_t sig = a < 3 ? a : 3u;
    y >>= (sig - pos + 1);
    pos = sig + 1;
  }
  *code = c;
  *n_out = pos > n ? pos : n;
  return len;
}

// Decode one plane from the peeked stream bits `w` (bit 0 = next bit) with
// `budget` bits left.  Returns the plane bits x; *used = bits consumed;
// *n_io updated.  Matches the per-bit decoder including truncation.
HCCX_HD uint32_t plane_decode(uint64_t w, uint32_t budget, uint32_t* n_io, uint32_t* used) {
  uint32_t n = *n_io;
  const uint32_t m = n < budget ? n : budget;
  uint32_t x = static_cast<uint32_t>(w) & ((1u << m) - 1u);
  uint32_t c = m;
  uint32_t rem = budget - m;
  uint32_t pos = n;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    if (pos >= 4 || rem == 0) break;
    const uint32_t t = static_cast<uint32_t>(w >> c) & 1u;  // group test
    c += 1;
    rem -= 1;
    if (!t) break;
    const uint32_t zmax = 3 - pos;  // explicit positions pos..2
    const uint64_t rest = w >> c;
    // length of the zero run, capped at 4 (only runs < 3 are explicit)
    const uint32_t z = ctz32(static_cast<uint32_t>(rest) | 0x10u);
    uint32_t a;
    if (z < zmax && z + 1 <= rem) {  // run of z zeros ended by a 1
      c += z + 1;
      rem -= z + 1;
      a = pos + z;
    } else if (z >= zmax && zmax <= rem) {  // zeros up to position 3, implicit 1
      c += zmax;
      rem -= zmax;
      a = 3;
    } else {  // budget ends inside the zero run: the per-bit decoder still marks position pos+rem
      c += rem;
      a = pos + rem;
      rem = 0;
    }
    x |= 1u << a;
    pos = a + 1;
  }
  *used = c;
  *n_io = pos > n ? pos : n;
  return x;
}

}  // namespace zfp_planes
}  // namespace hccx
