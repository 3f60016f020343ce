// test_zfp_planes.cpp -- the plane-at-a-time zfp coder (csrc/zfp_planes.cuh)
// against the per-bit loops of the published coder (the ones in
// oracle/hcc_oracle.c zfp_encode_block / zfp_decode_block), exhaustively
// over (significant count n, plane bits x, remaining budget) with random
// trailing stream bits.  CPU only.
#include <cstdint>
#include <cstdio>
#include <random>

#include "zfp_planes.cuh"

using namespace hccx::zfp_planes;

// per-bit encoder of one plane: returns emitted bits (LSB-first) and count
static uint32_t ref_encode(uint32_t& n, uint32_t x, uint32_t& bits, uint32_t& code) {
  uint32_t len = 0;
  code = 0;
  auto put = [&](uint32_t b) { code |= (b & 1u) << len; ++len; };
  const uint32_t m = n < bits ? n : bits;
  bits -= m;
  for (uint32_t i = 0; i < m; ++i) { put(x); x >>= 1; }
  while (n < 4 && bits) {
    bits--;
    const uint32_t any = x != 0;
    put(any);
    if (!any) break;
    while (n < 3 && bits) {
      bits--;
      const uint32_t b = x & 1u;
      put(b);
      if (b) break;
      x >>= 1;
      n++;
    }
    x >>= 1;
    n++;
  }
  return len;
}

static uint32_t ref_decode(uint64_t w, uint32_t& bits, uint32_t& n, uint32_t& used) {
  used = 0;
  auto get = [&]() { return static_cast<uint32_t>((w >> used++) & 1u); };
  const uint32_t m = n < bits ? n : bits;
  bits -= m;
  uint32_t x = 0;
  for (uint32_t i = 0; i < m; ++i) x |= get() << i;
  while (n < 4 && bits) {
    bits--;
    if (!get()) break;
    while (n < 3 && bits) {
      bits--;
      if (get()) break;
      n++;
    }
    x += 1u << n;
    n++;
  }
  return x;
}

// per-bit block coder (the loops of oracle/hcc_oracle.c zfp_encode_block /
// zfp_decode_block after the header) on a Bits accumulator
static void ref_block_encode(const uint32_t (&u)[4], uint32_t bits, Bits& b) {
  uint32_t n = 0;
  for (int k = 31; bits && k >= 0; --k) {
    uint32_t x = plane_bits(u, k), code;
    const uint32_t len = ref_encode(n, x, bits, code);
    b.put(code, static_cast<int>(len));
  }
}

static void ref_block_decode(Bits& b, uint32_t bits, uint32_t (&u)[4]) {
  u[0] = u[1] = u[2] = u[3] = 0;
  uint32_t n = 0;
  for (int k = 31; bits && k >= 0; --k) {
    uint32_t used;
    const uint32_t x = ref_decode(b.peek(), bits, n, used);
    b.pos += static_cast<int>(used);
    for (int i = 0; i < 4; ++i) u[i] |= ((x >> i) & 1u) << k;
  }
}

int main() {
  int fails = 0, checks = 0;
  std::mt19937_64 rng(7);
  for (uint32_t n0 = 0; n0 <= 4; ++n0)
    for (uint32_t x = 0; x < 16; ++x) {
      // plane values must agree with the significance state: coefficients
      // below n0 are significant already, any bit pattern is valid
      uint32_t code, nn;
      const uint32_t len = plane_code(n0, x, &code, &nn);
      for (uint32_t budget = 0; budget <= 12; ++budget) {
        uint32_t n = n0, bits = budget, rc;
        const uint32_t rl = ref_encode(n, x, bits, rc);
        const uint32_t m = len < budget ? len : budget;
        ++checks;
        if (rl != m || (rc & ((1u << m) - 1u)) != (code & ((1u << m) - 1u)) || (len <= budget && n != nn)) {
          if (fails++ < 10) std::printf("encode n=%u x=%u budget=%u: ref len %u code %x n %u | new len %u code %x n %u\n",
                                        n0, x, budget, rl, rc, n, len, code, nn);
        }
        for (int t = 0; t < 8; ++t) {  // decode the (possibly truncated) codeword + random trailing bits
          uint64_t w = (rng() << m) | (code & ((1u << m) - 1u));
          uint32_t rn = n0, rb = budget, ru;
          const uint32_t rx = ref_decode(w, rb, rn, ru);
          uint32_t dn = n0, du;
          const uint32_t dx = plane_decode(w, budget, &dn, &du);
          ++checks;
          if (rx != dx || ru != du || rn != dn) {
            if (fails++ < 20)
              std::printf("decode n=%u x=%u budget=%u w=%llx: ref x %u used %u n %u | new x %u used %u n %u\n", n0, x,
                          budget, static_cast<unsigned long long>(w), rx, ru, rn, dx, du, dn);
          }
        }
      }
    }
  // random streams (not produced by the encoder) through the decoder
  for (int t = 0; t < 200000; ++t) {
    const uint64_t w = rng();
    const uint32_t n0 = rng() % 5, budget = rng() % 40;
    uint32_t rn = n0, rb = budget, ru, dn = n0, du;
    const uint32_t rx = ref_decode(w, rb, rn, ru);
    const uint32_t dx = plane_decode(w, budget, &dn, &du);
    ++checks;
    if (rx != dx || ru != du || rn != dn) {
      if (fails++ < 30) std::printf("random decode n=%u budget=%u w=%llx: ref %u/%u/%u new %u/%u/%u\n", n0, budget,
                                    static_cast<unsigned long long>(w), rx, ru, rn, dx, du, dn);
    }
  }
  // whole blocks: random negabinary coefficients of mixed magnitudes, every budget
  for (int t = 0; t < 60000; ++t) {
    uint32_t u[4];
    for (int i = 0; i < 4; ++i) {
      const int sh = static_cast<int>(rng() % 33);
      u[i] = sh == 32 ? 0u : static_cast<uint32_t>(rng()) >> sh;
    }
    const uint32_t budget = 3 + rng() % 117;  // 4R-9 for R in [3, 32]
    Bits a, b;
    ref_block_encode(u, budget, a);
    encode_planes(u, budget, b);
    ++checks;
    if (a.lo != b.lo || a.hi != b.hi) {
      if (fails++ < 40) std::printf("block encode u=%x,%x,%x,%x budget %u\n", u[0], u[1], u[2], u[3], budget);
      continue;
    }
    {  // the two-block stepper form must give the same bits
      Bits c;
      PlaneEnc e;
      e.init(u, budget, c);
      while (e.active()) e.step(c);
      ++checks;
      if (c.lo != b.lo || c.hi != b.hi) {
        if (fails++ < 40) std::printf("stepper encode mismatch budget %u\n", budget);
      }
      Bits c2;
      c2.lo = a.lo;
      c2.hi = a.hi;
      PlaneDec dd;
      dd.init(c2, budget);
      while (dd.active()) dd.step(c2);
      Bits c3;
      c3.lo = a.lo;
      c3.hi = a.hi;
      uint32_t r3[4];
      ref_block_decode(c3, budget, r3);
      ++checks;
      if (dd.u[0] != r3[0] || dd.u[1] != r3[1] || dd.u[2] != r3[2] || dd.u[3] != r3[3] || c2.pos != c3.pos) {
        if (fails++ < 40) std::printf("stepper decode mismatch budget %u\n", budget);
      }
    }
    // decode the stream plus random trailing garbage past the budget
    Bits s1, s2;
    s1.lo = s2.lo = a.lo;
    s1.hi = s2.hi = a.hi;
    uint32_t r[4], d[4];
    ref_block_decode(s1, budget, r);
    decode_planes(s2, budget, d);
    ++checks;
    if (r[0] != d[0] || r[1] != d[1] || r[2] != d[2] || r[3] != d[3] || s1.pos != s2.pos) {
      if (fails++ < 40) std::printf("block decode u=%x,%x,%x,%x budget %u: ref pos %d new pos %d\n", u[0], u[1], u[2], u[3],
                                    budget, s1.pos, s2.pos);
    }
  }
  // rate-specialised accumulators (Bits32 for R <= 8, Bits64 for R <= 16)
  // with the significance-loop + verbatim-tail split, after a 9-bit header,
  // against the per-bit reference on the full 128-bit accumulator
  for (int t = 0; t < 200000; ++t) {
    uint32_t u[4];
    for (int i = 0; i < 4; ++i) {
      const int sh = static_cast<int>(rng() % 33);
      u[i] = sh == 32 ? 0u : static_cast<uint32_t>(rng()) >> sh;
    }
    const int R = 3 + static_cast<int>(rng() % 30);
    const uint32_t budget = 4u * R - 9u;
    const uint64_t hdr = rng() & 0x1ffu;
    Bits ref;
    ref.put(hdr, 9);
    ref_block_encode(u, budget, ref);
    auto run = [&](auto acc) {
      using B = decltype(acc);
      B b;
      b.put(hdr, 9);
      PlaneEnc e;
      e.init(u, budget, b);
      while (e.sig_active()) e.step(b);
      e.tail(b);
      // compare the 4R stream bits
      Bits got;
      for (int pos = 0; pos < 4 * R; pos += 16) {
        B tmp = b;
        tmp.pos = pos;
        got.put(tmp.peek() & 0xffffu, 16);
      }
      Bits want = ref;
      const uint64_t m0 = 4 * R >= 64 ? ~0ull : ((1ull << (4 * R)) - 1ull);
      const uint64_t m1 = 4 * R >= 128 ? ~0ull : (4 * R <= 64 ? 0ull : ((1ull << (4 * R - 64)) - 1ull));
      ++checks;
      if ((got.lo & m0) != (want.lo & m0) || (got.hi & m1) != (want.hi & m1)) {
        if (fails++ < 60) std::printf("narrow encode R=%d u=%x,%x,%x,%x\n", R, u[0], u[1], u[2], u[3]);
        return;
      }
      // decode from the narrow accumulator
      B d = b;
      d.pos = 9;
      PlaneDec dd;
      dd.init(d, budget);
      while (dd.sig_active()) dd.step(d);
      dd.tail(d);
      Bits r2 = ref;
      r2.pos = 9;
      uint32_t ru[4];
      ref_block_decode(r2, budget, ru);
      ++checks;
      if (dd.u[0] != ru[0] || dd.u[1] != ru[1] || dd.u[2] != ru[2] || dd.u[3] != ru[3]) {
        if (fails++ < 60) std::printf("narrow decode R=%d u=%x,%x,%x,%x\n", R, u[0], u[1], u[2], u[3]);
      }
    };
    if (R <= 8) run(Bits32{});
    if (R <= 16) run(Bits64{});
    run(Bits{});
    // the window steppers (two planes per lookup, windowed tails)
    auto run2 = [&](auto acc) {
      using B = decltype(acc);
      B b;
      b.put(hdr, 9);
      PlaneEnc2 e;
      e.init(u, budget, b);
      while (e.sig_active()) e.step(b);
      e.tail(b);
      Bits got;
      for (int pos = 0; pos < 4 * R; pos += 16) {
        B tmp = b;
        tmp.pos = pos;
        got.put(tmp.peek() & 0xffffu, 16);
      }
      const uint64_t m0 = 4 * R >= 64 ? ~0ull : ((1ull << (4 * R)) - 1ull);
      const uint64_t m1 = 4 * R >= 128 ? ~0ull : (4 * R <= 64 ? 0ull : ((1ull << (4 * R - 64)) - 1ull));
      ++checks;
      if ((got.lo & m0) != (ref.lo & m0) || (got.hi & m1) != (ref.hi & m1)) {
        if (fails++ < 60) std::printf("window encode R=%d u=%x,%x,%x,%x\n", R, u[0], u[1], u[2], u[3]);
        return;
      }
      B d = b;
      d.pos = 9;
      PlaneDec2 dd;
      dd.init(d, budget);
      while (dd.sig_active()) dd.step(d);
      dd.tail(d);
      Bits r2 = ref;
      r2.pos = 9;
      uint32_t ru[4];
      ref_block_decode(r2, budget, ru);
      ++checks;
      if (dd.u[0] != ru[0] || dd.u[1] != ru[1] || dd.u[2] != ru[2] || dd.u[3] != ru[3]) {
        if (fails++ < 60) std::printf("window decode R=%d u=%x,%x,%x,%x\n", R, u[0], u[1], u[2], u[3]);
      }
    };
    if (R <= 8) run2(Bits32{});
    if (R <= 16) run2(Bits64{});
    run2(Bits{});
    // the predicated steppers in a joint two-block loop (the device's form),
    // the second block a different random block
    {
      uint32_t u2[4];
      for (int i = 0; i < 4; ++i) {
        const int sh = static_cast<int>(rng() % 33);
        u2[i] = sh == 32 ? 0u : static_cast<uint32_t>(rng()) >> sh;
      }
      Bits ref2;
      ref2.put(hdr, 9);
      ref_block_encode(u2, budget, ref2);
      Bits b0, b1;
      b0.put(hdr, 9);
      b1.put(hdr, 9);
      PlaneEnc2 e0, e1;
      e0.init(u, budget, b0);
      e1.init(u2, budget, b1);
      for (;;) {
        const bool a0 = e0.sig_active(), a1 = e1.sig_active();
        if (!(a0 || a1)) break;
        e0.step_if(b0, a0);
        e1.step_if(b1, a1);
      }
      e0.tail(b0);
      e1.tail(b1);
      ++checks;
      if (b0.lo != ref.lo || b0.hi != ref.hi || b1.lo != ref2.lo || b1.hi != ref2.hi) {
        if (fails++ < 60) std::printf("joint encode R=%d\n", R);
      } else {
        Bits c0 = ref, c1 = ref2;
        c0.pos = 9;
        c1.pos = 9;
        PlaneDec2 d0, d1;
        d0.init(c0, budget);
        d1.init(c1, budget);
        for (;;) {
          const bool a0 = d0.sig_active(), a1 = d1.sig_active();
          if (!(a0 || a1)) break;
          d0.step_if(c0, a0);
          d1.step_if(c1, a1);
        }
        d0.tail(c0);
        d1.tail(c1);
        Bits r0 = ref, r1 = ref2;
        r0.pos = 9;
        r1.pos = 9;
        uint32_t w0[4], w1[4];
        ref_block_decode(r0, budget, w0);
        ref_block_decode(r1, budget, w1);
        ++checks;
        bool ok = true;
        for (int i = 0; i < 4; ++i) ok = ok && d0.u[i] == w0[i] && d1.u[i] == w1[i];
        if (!ok && fails++ < 60) std::printf("joint decode R=%d\n", R);
      }
    }
  }
  std::printf("zfp plane coder: %d checks, %d failures\n", checks, fails);
  return fails ? 1 : 0;
}
