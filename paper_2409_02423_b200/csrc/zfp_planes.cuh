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

#if !defined(__CUDACC__)
#include <algorithm>
using std::max;
#endif

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


// 128-bit LSB-first bit accumulator / reader (host + device).
struct Bits {
  uint64_t lo = 0, hi = 0;
  int pos = 0;
  HCCX_HD void put(uint64_t val, int nbits) {  // nbits <= 64, val < 2^nbits
    if (nbits == 0) return;
    if (pos < 64) {
      lo |= val << pos;
      if (pos + nbits > 64) hi |= val >> (64 - pos);
    } else {
      hi |= val << (pos - 64);
    }
    pos += nbits;
  }
  HCCX_HD uint64_t peek() const {  // the next 64 bits (zeros past the end)
    if (pos == 0) return lo;
    if (pos < 64) return (lo >> pos) | (hi << (64 - pos));
    return pos < 128 ? hi >> (pos - 64) : 0ull;
  }
  HCCX_HD uint64_t get(int nbits) {  // nbits <= 32
    const uint64_t v = nbits ? peek() & ((1ull << nbits) - 1ull) : 0ull;
    pos += nbits;
    return v;
  }
};

HCCX_HD int top_bit(uint32_t v) {  // index of the highest set bit, -1 for 0
#if defined(__CUDA_ARCH__)
  return 31 - __clz(static_cast<int>(v));
#else
  return v ? 31 - __builtin_clz(v) : -1;
#endif
}

HCCX_HD uint32_t plane_bits(const uint32_t (&u)[4], int k) {
  return ((u[0] >> k) & 1u) | (((u[1] >> k) & 1u) << 1) | (((u[2] >> k) & 1u) << 2) | (((u[3] >> k) & 1u) << 3);
}

// Embedded coding of one block's negabinary coefficients with `budget` bits
// (4R-9 after the header), same bits as the per-bit coder.  Three regimes:
// planes above the highest set bit each cost one '0' group test (emitted as
// a run); planes while fewer than four coefficients are significant use
// plane_code; once all four are, every plane is its 4 bits verbatim.
HCCX_HD void encode_planes(const uint32_t (&u)[4], uint32_t budget, Bits& b) {
  const int G = max(max(top_bit(u[0]), top_bit(u[1])), max(top_bit(u[2]), top_bit(u[3])));
  const uint32_t lead = static_cast<uint32_t>(31 - G);  // all-zero planes (32 when the block is zero)
  const uint32_t e = lead < budget ? lead : budget;
  b.pos += static_cast<int>(e);  // '0' group tests: zeros already in place
  budget -= e;
  int k = G;
  uint32_t n = 0;
  while (budget && k >= 0 && n < 4) {
    uint32_t code, nn;
    const uint32_t len = plane_code(n, plane_bits(u, k), &code, &nn);
    const uint32_t m = len < budget ? len : budget;
    b.put(code & ((1u << m) - 1u), static_cast<int>(m));
    budget -= m;
    n = nn;
    --k;
  }
  while (budget && k >= 0) {  // verbatim planes
    const uint32_t m = budget < 4 ? budget : 4u;
    b.put(plane_bits(u, k) & ((1u << m) - 1u), static_cast<int>(m));
    budget -= m;
    --k;
  }
}

HCCX_HD void decode_planes(Bits& b, uint32_t budget, uint32_t (&u)[4]) {
  u[0] = u[1] = u[2] = u[3] = 0;
  // leading all-zero planes: a run of '0' group tests
  const uint64_t w = b.peek();
  uint32_t lead = w ? static_cast<uint32_t>(
#if defined(__CUDA_ARCH__)
                          __ffsll(static_cast<long long>(w)) - 1
#else
                          __builtin_ctzll(w)
#endif
                          )
                    : 64u;
  if (lead > 32) lead = 32;
  if (lead > budget) lead = budget;
  b.pos += static_cast<int>(lead);
  budget -= lead;
  int k = 31 - static_cast<int>(lead);
  uint32_t n = 0;
  while (budget && k >= 0 && n < 4) {
    uint32_t used;
    const uint32_t x = plane_decode(b.peek(), budget, &n, &used);
    b.pos += static_cast<int>(used);
    budget -= used;
    u[0] |= (x & 1u) << k;
    u[1] |= ((x >> 1) & 1u) << k;
    u[2] |= ((x >> 2) & 1u) << k;
    u[3] |= ((x >> 3) & 1u) << k;
    --k;
  }
  while (budget && k >= 0) {  // verbatim planes
    const uint32_t m = budget < 4 ? budget : 4u;
    const uint32_t x = static_cast<uint32_t>(b.peek()) & ((1u << m) - 1u);
    b.pos += static_cast<int>(m);
    budget -= m;
    u[0] |= (x & 1u) << k;
    u[1] |= ((x >> 1) & 1u) << k;
    u[2] |= ((x >> 2) & 1u) << k;
    u[3] |= ((x >> 3) & 1u) << k;
    --k;
  }
}


// Plane codes by table lookup.  enc[n*16 + x] (n < 4 significant
// coefficients, plane bits x) = code | len << 8 | n_out << 12; dec[n*128 + w]
// (the next 7 stream bits w; a codeword is at most 7 bits, so with >= 7
// bits of budget left the truncation rule never applies) = x | used << 4 |
// n_out << 8.  Built from plane_code / plane_decode above (one entry per
// thread at kernel start on the device), so the tables carry exactly their
// bits; a lookup replaces the per-plane loop over group tests and runs.
// On the device they live in shared memory: 64 enc entries are 32 words,
// one per bank (conflict-free for any index pattern).
// enc2[n*256 + y] (n < 4; y = two consecutive planes' bits, low nibble the
// higher plane) = the two codewords concatenated | total len << 16 | n_out << 24
// (at most 14 bits: two planes per lookup in the significance phase).
// dec[512 + n*128 + ((1 << b) | bits)] (b = 1..6 bits of budget left, the
// block's last plane): the truncated decode, which depends only on those b
// bits -- every plane decodes by one lookup.
// enc2[1024 + n*16 + x]: the one-plane codes in enc2's packing (for the
// window stepper's last plane of a window or of the block).
struct Lut {
  uint16_t enc[64];
  uint16_t dec[1024];
  uint32_t enc2[1024 + 64];
};
constexpr uint32_t kLutEntries = 64 + 1024 + 1024 + 64;

HCCX_HD void lut_build_entry(uint32_t i, Lut& t) {
  if (i < 64) {
    uint32_t code, nn;
    const uint32_t len = plane_code(i >> 4, i & 15u, &code, &nn);
    t.enc[i] = static_cast<uint16_t>(code | (len << 8) | (nn << 12));
  } else if (i < 64 + 512) {
    const uint32_t j = i - 64;
    uint32_t nn = j >> 7, used;
    const uint32_t x = plane_decode(j & 127u, 7, &nn, &used);
    t.dec[j] = static_cast<uint16_t>(x | (used << 4) | (nn << 8));
  } else if (i < 64 + 1024) {
    const uint32_t j = i - 64 - 512;
    uint32_t nn = j >> 7, used = 0;
    const uint32_t v = j & 127u;  // (1 << b) | bits
    uint32_t x = 0;
    if (v >= 2) {
      const uint32_t b = 31u - static_cast<uint32_t>(
#if defined(__CUDA_ARCH__)
                                   __clz(v)
#else
                                   __builtin_clz(v)
#endif
                               );
      if (b <= 6) x = plane_decode(v & ((1u << b) - 1u), b, &nn, &used);
    }
    t.dec[512 + j] = static_cast<uint16_t>(x | (used << 4) | (nn << 8));
  } else if (i < 64 + 1024 + 1024) {
    const uint32_t j = i - 64 - 1024;
    uint32_t c1, n1, c2, n2;
    const uint32_t l1 = plane_code(j >> 8, j & 15u, &c1, &n1);
    const uint32_t l2 = plane_code(n1, (j >> 4) & 15u, &c2, &n2);
    t.enc2[j] = (c1 | (c2 << l1)) | ((l1 + l2) << 16) | (n2 << 24);
  } else if (i < kLutEntries) {
    const uint32_t j = i - 64 - 2048;
    uint32_t c1, n1;
    const uint32_t l1 = plane_code(j >> 4, j & 15u, &c1, &n1);
    t.enc2[1024 + j] = c1 | (l1 << 16) | (n1 << 24);
  }
}

#if defined(__CUDACC__)
__shared__ Lut g_lut;  // one per CTA (of the kernels that use it); filled by lut_init() before first use
__device__ __forceinline__ Lut& lut_dev() { return g_lut; }
// every thread of the CTA, then a CTA barrier before any lookup
__device__ __forceinline__ void lut_init() {
  for (uint32_t i = threadIdx.x; i < kLutEntries; i += blockDim.x) lut_build_entry(i, lut_dev());
}
#endif

HCCX_HD Lut& lut() {
#if defined(__CUDA_ARCH__)
  return g_lut;
#else
  static Lut t = [] {
    Lut x{};
    for (uint32_t i = 0; i < kLutEntries; ++i) lut_build_entry(i, x);
    return x;
  }();
  return t;
#endif
}

// Narrow stream accumulators: a block's 4R bits fit in 32 bits for R <= 8
// and in 64 bits for R <= 16, where put/peek are one shift and one OR.
template <class W>
struct BitsN {
  static constexpr int kWidth = 8 * static_cast<int>(sizeof(W));
  W v = 0;
  int pos = 0;
  HCCX_HD void put(uint64_t val, int nbits) {  // pos + nbits <= kWidth, val < 2^nbits
    if (nbits) v |= static_cast<W>(val) << pos;
    pos += nbits;
  }
  HCCX_HD uint64_t peek() const { return pos < kWidth ? static_cast<uint64_t>(v >> pos) : 0ull; }
  HCCX_HD uint64_t get(int nbits) {
    const uint64_t x = nbits ? peek() & ((1ull << nbits) - 1ull) : 0ull;
    pos += nbits;
    return x;
  }
};
using Bits32 = BitsN<uint32_t>;
using Bits64 = BitsN<uint64_t>;

HCCX_HD uint32_t brev32(uint32_t v) {
#if defined(__CUDA_ARCH__)
  return __brev(v);
#else
  v = ((v >> 1) & 0x55555555u) | ((v & 0x55555555u) << 1);
  v = ((v >> 2) & 0x33333333u) | ((v & 0x33333333u) << 2);
  v = ((v >> 4) & 0x0f0f0f0fu) | ((v & 0x0f0f0f0fu) << 4);
  v = ((v >> 8) & 0x00ff00ffu) | ((v & 0x00ff00ffu) << 8);
  return (v >> 16) | (v << 16);
#endif
}

// bit q of an 8-bit value -> bit 4q, and back
HCCX_HD uint32_t spread4(uint32_t x) {
  x = (x | (x << 12)) & 0x000f000fu;
  x = (x | (x << 6)) & 0x03030303u;
  return (x | (x << 3)) & 0x11111111u;
}
HCCX_HD uint32_t compact4(uint32_t x) {
  x &= 0x11111111u;
  x = (x | (x >> 3)) & 0x03030303u;
  x = (x | (x >> 6)) & 0x000f000fu;
  return (x | (x >> 12)) & 0xffu;
}

// Once all four coefficients are significant every plane is its 4 bits
// verbatim, so the rest of the block is the plane-major interleave of the
// coefficients' remaining bits, 8 planes per 32-bit word: nibble q = plane
// k-q (bit i = coefficient i), truncated at the budget like the per-plane
// codes.
template <class B>
HCCX_HD void put_verbatim(const uint32_t (&u)[4], int k, uint32_t budget, B& b) {
  while (budget && k >= 0) {
    const int m8 = k + 1 < 8 ? k + 1 : 8;
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) v |= spread4((brev32(u[i]) >> (31 - k)) & 0xffu) << i;
    const uint32_t bits = budget < 4u * m8 ? budget : 4u * m8;
    b.put(bits >= 32 ? v : v & ((1u << bits) - 1u), static_cast<int>(bits));
    budget -= bits;
    k -= m8;
  }
}

template <class B>
HCCX_HD void get_verbatim(B& b, int k, uint32_t budget, uint32_t (&u)[4]) {
  while (budget && k >= 0) {
    const int m8 = k + 1 < 8 ? k + 1 : 8;
    const uint32_t bits = budget < 4u * m8 ? budget : 4u * m8;
    uint32_t w = static_cast<uint32_t>(b.peek());
    if (bits < 32) w &= (1u << bits) - 1u;
    b.pos += static_cast<int>(bits);
#pragma unroll
    for (int i = 0; i < 4; ++i) u[i] |= brev32(compact4(w >> i)) >> (31 - k);
    budget -= bits;
    k -= m8;
  }
}

// Steppers for coding two blocks in one loop (a lane owns two blocks: the
// joint loop runs max(planes) iterations instead of their sum and gives the
// two independent dependency chains to the scheduler side by side).  Same
// bits as encode_planes / decode_planes.
struct PlaneEnc {
  uint32_t u[4];
  uint32_t budget, n;
  int k;
  template <class B>
  HCCX_HD void init(const uint32_t (&uu)[4], uint32_t bud, B& b) {
    u[0] = uu[0], u[1] = uu[1], u[2] = uu[2], u[3] = uu[3];
    const int G = max(max(top_bit(u[0]), top_bit(u[1])), max(top_bit(u[2]), top_bit(u[3])));
    const uint32_t lead = static_cast<uint32_t>(31 - G);
    const uint32_t e = lead < bud ? lead : bud;
    b.pos += static_cast<int>(e);
    budget = bud - e;
    k = G;
    n = 0;
  }
  HCCX_HD bool active() const { return budget != 0 && k >= 0; }
  // significance phase: planes until all four coefficients are significant
  HCCX_HD bool sig_active() const { return budget != 0 && k >= 0 && n < 4; }
  // then the verbatim tail in one go
  template <class B>
  HCCX_HD void tail(B& b) {
    put_verbatim(u, k, budget, b);
    budget = 0;
  }
  template <class B>
  HCCX_HD void step(B& b) {
    const uint32_t x = plane_bits(u, k);
    uint32_t code = x, nn = 4, len = 4;  // all significant: verbatim plane
    if (n < 4) {
      const uint32_t e = lut().enc[n * 16 + x];
      code = e & 0x7fu;
      len = (e >> 8) & 7u;
      nn = e >> 12;
    }
    const uint32_t m = len < budget ? len : budget;
    b.put(code & ((1u << m) - 1u), static_cast<int>(m));
    budget -= m;
    n = nn;
    --k;
  }
};

struct PlaneDec {
  uint32_t u[4];
  uint32_t budget, n;
  int k;
  template <class B>
  HCCX_HD void init(B& b, uint32_t bud) {
    u[0] = u[1] = u[2] = u[3] = 0;
    const uint64_t w = b.peek();
    uint32_t lead = w ? static_cast<uint32_t>(
#if defined(__CUDA_ARCH__)
                            __ffsll(static_cast<long long>(w)) - 1
#else
                            __builtin_ctzll(w)
#endif
                            )
                      : 64u;
    if (lead > 32) lead = 32;
    if (lead > bud) lead = bud;
    b.pos += static_cast<int>(lead);
    budget = bud - lead;
    k = 31 - static_cast<int>(lead);
    n = 0;
  }
  HCCX_HD bool active() const { return budget != 0 && k >= 0; }
  HCCX_HD bool sig_active() const { return budget != 0 && k >= 0 && n < 4; }
  template <class B>
  HCCX_HD void tail(B& b) {
    get_verbatim(b, k, budget, u);
    budget = 0;
  }
  template <class B>
  HCCX_HD void step(B& b) {
    uint32_t used, x;
    const uint64_t w = b.peek();
    if (n == 4) {
      used = budget < 4 ? budget : 4u;
      x = static_cast<uint32_t>(w) & ((1u << used) - 1u);
    } else if (budget >= 7) {
      const uint32_t e = lut().dec[n * 128 + (static_cast<uint32_t>(w) & 127u)];
      x = e & 15u;
      used = (e >> 4) & 15u;
      n = e >> 8;
    } else {  // the block's last, truncated plane
      x = plane_decode(w, budget, &n, &used);
    }
    b.pos += static_cast<int>(used);
    budget -= used;
    u[0] |= (x & 1u) << k;
    u[1] |= ((x >> 1) & 1u) << k;
    u[2] |= ((x >> 2) & 1u) << k;
    u[3] |= ((x >> 3) & 1u) << k;
    --k;
  }
};

// ---- window steppers -------------------------------------------------------
// The coefficients' next 8 planes as one 32-bit word (nibble q = plane k-q,
// bit i = coefficient i; zero below plane 0), built once per 8 planes from
// the bit-reversed coefficients.  The encoder reads two planes per table
// lookup (enc2) and copies the verbatim tail straight out of the window; the
// decoder collects decoded planes into a window and scatters it into the
// coefficients once per 8 planes.  Same bits as PlaneEnc / PlaneDec
// (tests/cpp/test_zfp_planes.cpp).
HCCX_HD uint32_t plane_window(const uint32_t (&r)[4], int k) {
  uint32_t v = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) v |= spread4((r[i] >> (31 - k)) & 0xffu) << i;
  return v;
}

struct PlaneEnc2 {
  uint32_t r[4];  // bit-reversed coefficients
  uint32_t w;     // window: nibble q = plane k + q0 - q (q0 = nibbles already used)
  uint32_t budget, n;
  int k, q;
  template <class B>
  HCCX_HD void init(const uint32_t (&uu)[4], uint32_t bud, B& b) {
    const int G = max(max(top_bit(uu[0]), top_bit(uu[1])), max(top_bit(uu[2]), top_bit(uu[3])));
    const uint32_t lead = static_cast<uint32_t>(31 - G);
    const uint32_t e = lead < bud ? lead : bud;
    b.pos += static_cast<int>(e);
    budget = bud - e;
    k = G;
    n = 0;
    q = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = brev32(uu[i]);
    w = k >= 0 ? plane_window(r, k) : 0u;
  }
  HCCX_HD bool sig_active() const { return budget != 0 && k >= 0 && n < 4; }
  template <class B>
  HCCX_HD void step(B& b) {
    if (q == 8) {
      w = plane_window(r, k);
      q = 0;
    }
    uint32_t code, len, nn;
    int planes;
    if (k >= 1 && q <= 6) {
      const uint32_t e = lut().enc2[n * 256 + ((w >> (4 * q)) & 0xffu)];
      code = e & 0xffffu;
      len = (e >> 16) & 0xffu;
      nn = e >> 24;
      planes = 2;
    } else {
      const uint32_t e = lut().enc[n * 16 + ((w >> (4 * q)) & 15u)];
      code = e & 0x7fu;
      len = (e >> 8) & 7u;
      nn = e >> 12;
      planes = 1;
    }
    const uint32_t m = len < budget ? len : budget;
    b.put(code & ((1u << m) - 1u), static_cast<int>(m));
    budget -= m;
    n = nn;
    k -= planes;
    q += planes;
  }
  // step() when `act`, else no change -- branch-free apart from the rare
  // window refill, so two blocks advance in one converged loop
  template <class B>
  HCCX_HD void step_if(B& b, bool act) {
    if (act && q == 8) {
      w = plane_window(r, k);
      q = 0;
    }
    const bool two = k >= 1 && q <= 6;
    const uint32_t nn0 = act ? n : 0u;
    const uint32_t sh = 4u * static_cast<uint32_t>(q & 7);
    const uint32_t idx = two ? nn0 * 256u + ((w >> sh) & 0xffu) : 1024u + nn0 * 16u + ((w >> sh) & 15u);
    const uint32_t e = lut().enc2[idx];
    const uint32_t len = (e >> 16) & 0xffu;
    const uint32_t m = act ? (len < budget ? len : budget) : 0u;
    b.put((e & 0xffffu) & ((1u << m) - 1u), static_cast<int>(m));
    budget -= m;
    const int planes = act ? (two ? 2 : 1) : 0;
    n = act ? (e >> 24) : n;
    k -= planes;
    q += planes;
  }
  // all four significant: every remaining plane is its nibble, verbatim
  template <class B>
  HCCX_HD void tail(B& b) {
    while (budget && k >= 0) {
      if (q == 8) {
        w = plane_window(r, k);
        q = 0;
      }
      const int avail = 8 - q < k + 1 ? 8 - q : k + 1;
      const uint32_t bits = budget < 4u * avail ? budget : 4u * avail;
      const uint32_t v = w >> (4 * q);
      b.put(bits >= 32 ? v : v & ((1u << bits) - 1u), static_cast<int>(bits));
      budget -= bits;
      k -= avail;
      q += avail;
    }
    budget = 0;
  }
};

struct PlaneDec2 {
  uint32_t u[4];
  uint32_t budget, n;
  int k, top;  // next plane; the window's top plane
  uint32_t w;  // decoded planes since `top`, nibble q = plane top - q
  template <class B>
  HCCX_HD void init(B& b, uint32_t bud) {
    u[0] = u[1] = u[2] = u[3] = 0;
    const uint64_t pk = b.peek();
    uint32_t lead = pk ? static_cast<uint32_t>(
#if defined(__CUDA_ARCH__)
                             __ffsll(static_cast<long long>(pk)) - 1
#else
                             __builtin_ctzll(pk)
#endif
                             )
                       : 64u;
    if (lead > 32) lead = 32;
    if (lead > bud) lead = bud;
    b.pos += static_cast<int>(lead);
    budget = bud - lead;
    k = 31 - static_cast<int>(lead);
    top = k;
    w = 0;
    n = 0;
  }
  HCCX_HD bool sig_active() const { return budget != 0 && k >= 0 && n < 4; }
  HCCX_HD void flush() {
    if (w && top >= 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) u[i] |= brev32(compact4(w >> i)) >> (31 - top);
    }
    w = 0;
    top = k;
  }
  template <class B>
  HCCX_HD void step(B& b) {
    if (top - k == 8) flush();
    const uint32_t pk = static_cast<uint32_t>(b.peek());
    // full plane: the next 7 bits; the block's last, truncated plane: its b < 7 bits
    const uint32_t idx = budget >= 7 ? (pk & 127u) : (512u | (1u << budget) | (pk & ((1u << budget) - 1u)));
    const uint32_t e = lut().dec[n * 128 + idx];
    const uint32_t x = e & 15u, used = (e >> 4) & 15u;
    n = e >> 8;
    b.pos += static_cast<int>(used);
    budget -= used;
    w |= x << (4 * (top - k));
    --k;
  }
  // step() when `act`, else no change (see PlaneEnc2::step_if)
  template <class B>
  HCCX_HD void step_if(B& b, bool act) {
    if (act && top - k == 8) flush();
    const uint32_t pk = static_cast<uint32_t>(b.peek());
    const uint32_t bud = budget < 7 ? budget : 7u;
    const uint32_t idx = bud >= 7 ? (pk & 127u) : (512u | (1u << bud) | (pk & ((1u << bud) - 1u)));
    const uint32_t e = lut().dec[(act ? n : 0u) * 128 + idx];
    const uint32_t used = act ? (e >> 4) & 15u : 0u;
    b.pos += static_cast<int>(used);
    budget -= used;
    n = act ? (e >> 8) : n;
    const int sh = 4 * (top - k);
    w |= act ? (e & 15u) << (sh & 31) : 0u;
    k -= act ? 1 : 0;
  }
  template <class B>
  HCCX_HD void tail(B& b) {
    flush();
    get_verbatim(b, k, budget, u);
    budget = 0;
  }
};

}  // namespace zfp_planes
}  // namespace hccx
