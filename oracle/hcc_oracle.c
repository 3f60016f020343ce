/*
 * hcc_oracle.c -- CPU restatement of the reference's compressed-collective
 * hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 kernels in
 * paper_2409_02423_b200/csrc.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links, imports or falls back to it.
 *
 * Every function restates one piece of the reference (arxiv/paper_2409_02423,
 * the `hybridcomm` C++ simulator) and cites the file:line it follows, with
 * paths relative to /root/reference/proj.  Parity of this restatement is
 * pinned two ways (see tests/test_oracle_pins.py):
 *   1. the known-answer tests of proj/tests/test_codec.cpp and
 *      proj/tests/test_collectives.cpp, re-expressed in tests/;
 *   2. byte/bit comparisons against the reference library itself, compiled
 *      here from its own sources into oracle/_ref (oracle/build_ref.sh), and
 *      the golden fixtures generated from it (tests/golden/make_golden.py).
 *
 * The ZFP-mode codec at the bottom (kind 3, "zfp-rate:N") has NO reference
 * implementation: the reference ships no ZFP.  Its
 * parity is UNPINNED; this file's restatement of the published 1-D zfp
 * fixed-rate algorithm is its only oracle.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (the reference
 * builds with -ffp-contract=off, proj/CMakeLists.txt:15-17, so float adds are
 * never fused).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NONFINITE 1
#define ORC_CORRUPT 2
#define ORC_BADCHUNK 4
#define ORC_INVALID 9

enum { KIND_IDENTITY = 0, KIND_LOSSLESS = 1, KIND_FIXED = 2, KIND_ZFP = 3 };

/* ------------------------------------------------------------------------ */
/* Deterministic RNG: std::mt19937_64 plus the hand-rolled distributions of  */
/* include/hcc/rng.hpp:14-40.                                                */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t rng_u64(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:19 */
static uint32_t rng_u32(orc_rng* r) { return (uint32_t)(rng_u64(r) >> 32); }
/* rng.hpp:22-24: 24 random bits on the exact float grid */
static float rng_unit(orc_rng* r) { return (float)(rng_u64(r) >> 40) * 0x1.0p-24f; }
/* rng.hpp:26 */
static float rng_range(orc_rng* r, float lo, float hi) { return lo + (hi - lo) * rng_unit(r); }
/* rng.hpp:29-35: Box-Muller, two uniforms per draw */
static float rng_normal(orc_rng* r) {
  float u1 = rng_unit(r);
  float u2 = rng_unit(r);
  if (u1 < 0x1.0p-24f) u1 = 0x1.0p-24f;
  float rad = sqrtf(-2.0f * logf(u1));
  return rad * cosf(6.2831853071795864769f * u2);
}

/* Buffer generators of tests/support/oracles.cpp:9-36.  mode:
 * 0 bits, 1 finite (2^-20..2^20), 2 uniform[lo,hi), 3 sparse(zero_frac=lo),
 * 4 scaled normal (lo * normal()), the gradient-like bench input. */
void orc_fill(uint64_t seed, int mode, uint64_t n, float lo, float hi, float* out) {
  orc_rng r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; ++i) {
    switch (mode) {
      case 0: {
        uint32_t u = rng_u32(&r);
        memcpy(&out[i], &u, 4);
        break;
      }
      case 1: {
        int e = (int)(rng_u32(&r) % 41u) - 20;
        out[i] = ldexpf(rng_range(&r, -1.0f, 1.0f), e);
        break;
      }
      case 2: out[i] = rng_range(&r, lo, hi); break;
      case 3: out[i] = (rng_unit(&r) < lo) ? 0.0f : rng_normal(&r); break;
      default: out[i] = lo * rng_normal(&r); break;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* LSB-first bit packing (src/codec_kernels.hpp:25-83).                      */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* out;
  uint64_t pos; /* bytes written */
  uint64_t acc;
  int filled;
} bitw;

static uint32_t low_mask(int nbits) { return nbits >= 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u); }

static void bw_put(bitw* w, uint32_t value, int nbits) {
  w->acc |= (uint64_t)(value & low_mask(nbits)) << w->filled;
  w->filled += nbits;
  while (w->filled >= 8) {
    w->out[w->pos++] = (uint8_t)w->acc;
    w->acc >>= 8;
    w->filled -= 8;
  }
}

static void bw_flush(bitw* w) {
  if (w->filled > 0) {
    w->out[w->pos++] = (uint8_t)w->acc;
    w->acc = 0;
    w->filled = 0;
  }
}

typedef struct {
  const uint8_t* in;
  uint64_t size, pos;
  uint64_t acc;
  int filled;
} bitr;

static int br_get(bitr* r, int nbits, uint32_t* value) {
  while (r->filled < nbits) {
    if (r->pos >= r->size) return 0;
    r->acc |= (uint64_t)r->in[r->pos++] << r->filled;
    r->filled += 8;
  }
  *value = (uint32_t)r->acc & low_mask(nbits);
  r->acc >>= nbits;
  r->filled -= nbits;
  return 1;
}

/* ------------------------------------------------------------------------ */
/* FixedRate codec (src/codec_kernels.hpp:85-163, src/codec.cpp:47-61).     */
/* ------------------------------------------------------------------------ */

#define FR_BLOCK 64

/* src/codec_kernels.hpp:94-96 */
static uint64_t fr_block_bytes(int rate) { return 1 + (uint64_t)rate * FR_BLOCK / 8; }

/* src/codec.cpp:47-61 (identity and fixed-rate; lossless has no law) */
uint64_t orc_wire_size(int kind, int rate, uint64_t n) {
  if (kind == KIND_IDENTITY) return 4 * n;
  if (kind == KIND_FIXED) return ((n + FR_BLOCK - 1) / FR_BLOCK) * fr_block_bytes(rate);
  if (kind == KIND_ZFP) return (((n + 3) / 4) * 4 * (uint64_t)rate + 7) / 8;
  return UINT64_MAX;
}

/* src/codec_kernels.hpp:100-140: block max exponent, then RNE quantisation
 * of v / 2^(E - rate + 2) into a biased rate-bit field, LSB-first. */
static int fr_encode_block(const float* v, uint64_t n, int rate, uint8_t* out) {
  int emax = -127;
  for (uint64_t i = 0; i < n; ++i) {
    if (!isfinite(v[i])) return 0;
    if (v[i] != 0.0f) {
      int e = ilogbf(v[i]);
      if (e < -127) e = -127;
      if (e > emax) emax = e;
    }
  }
  out[0] = (uint8_t)(emax + 127);
  const double step = ldexp(1.0, emax - rate + 2);
  const int64_t hi = ((int64_t)1 << (rate - 1)) - 1;
  const int64_t lo = -((int64_t)1 << (rate - 1));
  const int64_t bias = (int64_t)1 << (rate - 1);
  bitw w = {out + 1, 0, 0, 0};
  for (uint64_t i = 0; i < FR_BLOCK; ++i) {
    int64_t q = 0;
    if (i < n && v[i] != 0.0f) {
      q = llrint((double)v[i] / step); /* default FP env: round-half-even */
      if (q > hi) q = hi;
      if (q < lo) q = lo;
    }
    bw_put(&w, (uint32_t)(q + bias), rate);
  }
  return 1;
}

/* src/codec_kernels.hpp:142-163 */
static void fr_decode_block(const uint8_t* in, int rate, float* out, uint64_t n) {
  const int emax = (int)in[0] - 127;
  const double step = ldexp(1.0, emax - rate + 2);
  const int64_t bias = (int64_t)1 << (rate - 1);
  bitr r = {in + 1, (uint64_t)rate * 8, 0, 0, 0};
  for (uint64_t i = 0; i < FR_BLOCK; ++i) {
    uint32_t u = 0;
    br_get(&r, rate, &u);
    if (i < n) out[i] = (float)((double)((int64_t)u - bias) * step);
  }
}

/* Buffer driver, src/codec_serial.cpp:34-47.  Returns ORC_NONFINITE when any
 * live value is NaN/Inf (codec_omp.cpp:45). */
int orc_fr_compress(int rate, const float* in, uint64_t n, uint8_t* out) {
  const uint64_t nb = (n + FR_BLOCK - 1) / FR_BLOCK, bb = fr_block_bytes(rate);
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t off = b * FR_BLOCK;
    const uint64_t live = (n - off < FR_BLOCK) ? n - off : FR_BLOCK;
    if (!fr_encode_block(in + off, live, rate, out + b * bb)) return ORC_NONFINITE;
  }
  return ORC_OK;
}

/* src/codec_serial.cpp:70-84 */
void orc_fr_decompress(int rate, const uint8_t* in, uint64_t n, float* out) {
  const uint64_t nb = (n + FR_BLOCK - 1) / FR_BLOCK, bb = fr_block_bytes(rate);
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t off = b * FR_BLOCK;
    const uint64_t live = (n - off < FR_BLOCK) ? n - off : FR_BLOCK;
    fr_decode_block(in + b * bb, rate, out + off, live);
  }
}

/* ------------------------------------------------------------------------ */
/* LosslessPredictor codec (src/codec_kernels.hpp:165-239,                   */
/* src/codec_serial.cpp:48-66, :85-107).                                     */
/* ------------------------------------------------------------------------ */

#define PRED_CHUNK 4096

static int lzc32(uint32_t x) { return x ? __builtin_clz(x) : 32; }

/* codec_kernels.hpp:203-215 */
static uint64_t pred_chunk_size(const float* v, uint64_t n) {
  uint64_t bits = 0;
  uint32_t prev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t x;
    memcpy(&x, &v[i], 4);
    const uint32_t res = x ^ prev;
    prev = x;
    int z = lzc32(res);
    if (z > 31) z = 31;
    bits += 5 + (uint64_t)(32 - z);
  }
  const uint64_t enc = (bits + 7) / 8;
  return enc < 4 * n ? enc : 4 * n;
}

uint64_t orc_pred_size(const float* in, uint64_t n) {
  const uint64_t nc = (n + PRED_CHUNK - 1) / PRED_CHUNK;
  uint64_t total = (nc + 7) / 8;
  for (uint64_t c = 0; c < nc; ++c) {
    const uint64_t off = c * PRED_CHUNK;
    const uint64_t live = (n - off < PRED_CHUNK) ? n - off : PRED_CHUNK;
    total += pred_chunk_size(in + off, live);
  }
  return total;
}

/* codec_kernels.hpp:177-199 plus the flag-byte prefix of
 * codec_serial.cpp:48-66.  `out` must hold orc_pred_size() bytes. */
uint64_t orc_pred_compress(const float* in, uint64_t n, uint8_t* out) {
  const uint64_t nc = (n + PRED_CHUNK - 1) / PRED_CHUNK;
  const uint64_t flag_bytes = (nc + 7) / 8;
  memset(out, 0, flag_bytes);
  uint64_t pos = flag_bytes;
  for (uint64_t c = 0; c < nc; ++c) {
    const uint64_t off = c * PRED_CHUNK;
    const uint64_t live = (n - off < PRED_CHUNK) ? n - off : PRED_CHUNK;
    const uint64_t sz = pred_chunk_size(in + off, live);
    if (sz >= 4 * live) {
      /* raw fallback: enc size reached raw size */
      memcpy(out + pos, in + off, 4 * live);
      out[c / 8] |= (uint8_t)(1u << (c % 8));
      pos += 4 * live;
      continue;
    }
    bitw w = {out + pos, 0, 0, 0};
    uint32_t prev = 0;
    for (uint64_t i = 0; i < live; ++i) {
      uint32_t x;
      memcpy(&x, &in[off + i], 4);
      const uint32_t res = x ^ prev;
      prev = x;
      int z = lzc32(res);
      if (z > 31) z = 31;
      bw_put(&w, (uint32_t)z, 5);
      bw_put(&w, res, 32 - z);
    }
    bw_flush(&w);
    pos += w.pos;
  }
  return pos;
}

/* codec_kernels.hpp:220-239, codec_serial.cpp:85-107 */
int orc_pred_decompress(const uint8_t* in, uint64_t size, uint64_t n, float* out) {
  const uint64_t nc = (n + PRED_CHUNK - 1) / PRED_CHUNK;
  const uint64_t flag_bytes = (nc + 7) / 8;
  if (size < flag_bytes) return ORC_CORRUPT;
  uint64_t pos = flag_bytes;
  for (uint64_t c = 0; c < nc; ++c) {
    const uint64_t off = c * PRED_CHUNK;
    const uint64_t live = (n - off < PRED_CHUNK) ? n - off : PRED_CHUNK;
    if ((in[c / 8] >> (c % 8)) & 1u) {
      if (size - pos < 4 * live) return ORC_CORRUPT;
      memcpy(out + off, in + pos, 4 * live);
      pos += 4 * live;
      continue;
    }
    bitr r = {in + pos, size - pos, 0, 0, 0};
    uint32_t prev = 0;
    for (uint64_t i = 0; i < live; ++i) {
      uint32_t z = 0, low = 0;
      if (!br_get(&r, 5, &z)) return ORC_CORRUPT;
      if (!br_get(&r, 32 - (int)z, &low)) return ORC_CORRUPT;
      const uint32_t x = low ^ prev;
      memcpy(&out[off + i], &x, 4);
      prev = x;
    }
    pos += r.pos;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ZFP-mode fixed-rate codec (kind 3).  NOT IN THE REFERENCE; parity         */
/* unpinned.  Restates the published 1-D zfp fixed-rate float path (zfp      */
/* 0.5.x encode/decode: common exponent, block-floating-point cast,          */
/* forward lifting, negabinary, embedded bit-plane group coding) with two    */
/* defined deviations: the cast is computed exactly in double (zfp's float  */
/* scale overflows for emax < -97), and non-finite input is rejected as in   */
/* FixedRate.  Each 4-value block takes exactly 4*rate bits, LSB-first.     */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint8_t* buf;
  uint64_t bit;
} zbw;

static void zbw_bit(zbw* w, uint32_t b) {
  if (b & 1u) w->buf[w->bit >> 3] |= (uint8_t)(1u << (w->bit & 7));
  w->bit++;
}

static uint32_t zbr_bit(const uint8_t* buf, uint64_t* bit) {
  uint32_t b = (buf[*bit >> 3] >> (*bit & 7)) & 1u;
  (*bit)++;
  return b;
}

/* Lifting steps use wrapping 32-bit adds (zfp relies on two's-complement
 * wrap; plain signed overflow would be UB in C) and arithmetic right shifts. */
static int32_t wadd(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static int32_t wsub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
static int32_t wshl1(int32_t a) { return (int32_t)((uint32_t)a << 1); }

static void zfp_fwd_lift(int32_t* p) {
  int32_t x = p[0], y = p[1], z = p[2], w = p[3];
  x = wadd(x, w); x >>= 1; w = wsub(w, x);
  z = wadd(z, y); z >>= 1; y = wsub(y, z);
  x = wadd(x, z); x >>= 1; z = wsub(z, x);
  w = wadd(w, y); w >>= 1; y = wsub(y, w);
  w = wadd(w, y >> 1); y = wsub(y, w >> 1);
  p[0] = x; p[1] = y; p[2] = z; p[3] = w;
}

static void zfp_inv_lift(int32_t* p) {
  int32_t x = p[0], y = p[1], z = p[2], w = p[3];
  y = wadd(y, w >> 1); w = wsub(w, y >> 1);
  y = wadd(y, w); w = wshl1(w); w = wsub(w, y);
  z = wadd(z, x); x = wshl1(x); x = wsub(x, z);
  y = wadd(y, z); z = wshl1(z); z = wsub(z, y);
  w = wadd(w, x); x = wshl1(x); x = wsub(x, w);
  p[0] = x; p[1] = y; p[2] = z; p[3] = w;
}

#define NBMASK 0xaaaaaaaau

/* one 4-value block at bit offset `bit0`; budget = 4*rate bits */
static int zfp_encode_block(const float* v, int rate, uint8_t* buf, uint64_t bit0) {
  zbw w = {buf, bit0};
  float amax = 0.0f;
  for (int i = 0; i < 4; ++i) {
    if (!isfinite(v[i])) return 0;
    const float a = fabsf(v[i]);
    if (a > amax) amax = a;
  }
  if (amax == 0.0f) {
    zbw_bit(&w, 0); /* zero block; remaining bits stay zero (padding) */
    return 1;
  }
  int emax;
  frexpf(amax, &emax);
  if (emax < -126) emax = -126;
  const uint32_t ebits = (uint32_t)(emax + 127);
  zbw_bit(&w, 1);
  for (int i = 0; i < 8; ++i) zbw_bit(&w, ebits >> i);
  int32_t q[4];
  for (int i = 0; i < 4; ++i) q[i] = (int32_t)((double)v[i] * ldexp(1.0, 30 - emax));
  zfp_fwd_lift(q);
  uint32_t u[4];
  for (int i = 0; i < 4; ++i) u[i] = ((uint32_t)q[i] + NBMASK) ^ NBMASK;
  uint32_t bits = 4 * (uint32_t)rate - 9;
  uint32_t n = 0;
  for (int k = 32; bits && k-- > 0;) {
    uint64_t x = 0;
    for (int i = 0; i < 4; ++i) x |= (uint64_t)((u[i] >> k) & 1u) << i;
    uint32_t m = n < bits ? n : bits;
    bits -= m;
    for (uint32_t i = 0; i < m; ++i) {
      zbw_bit(&w, (uint32_t)x);
      x >>= 1;
    }
    /* group test of the remaining values, unary run-length on the next one */
    while (n < 4 && bits) {
      bits--;
      const uint32_t any = x != 0;
      zbw_bit(&w, any);
      if (!any) break;
      while (n < 3 && bits) {
        bits--;
        const uint32_t b = (uint32_t)(x & 1u);
        zbw_bit(&w, b);
        if (b) break;
        x >>= 1;
        n++;
      }
      x >>= 1;
      n++;
    }
  }
  return 1;
}

static void zfp_decode_block(const uint8_t* buf, uint64_t bit0, int rate, float* out) {
  uint64_t bit = bit0;
  if (!zbr_bit(buf, &bit)) {
    for (int i = 0; i < 4; ++i) out[i] = 0.0f;
    return;
  }
  uint32_t ebits = 0;
  for (int i = 0; i < 8; ++i) ebits |= zbr_bit(buf, &bit) << i;
  const int emax = (int)ebits - 127;
  uint32_t u[4] = {0, 0, 0, 0};
  uint32_t bits = 4 * (uint32_t)rate - 9;
  uint32_t n = 0;
  for (int k = 32; bits && k-- > 0;) {
    uint32_t m = n < bits ? n : bits;
    bits -= m;
    uint64_t x = 0;
    for (uint32_t i = 0; i < m; ++i) x |= (uint64_t)zbr_bit(buf, &bit) << i;
    while (n < 4 && bits) {
      bits--;
      if (!zbr_bit(buf, &bit)) break;
      while (n < 3 && bits) {
        bits--;
        if (zbr_bit(buf, &bit)) break;
        n++;
      }
      x += (uint64_t)1 << n;
      n++;
    }
    for (int i = 0; x; ++i, x >>= 1) u[i] += (uint32_t)(x & 1u) << k;
  }
  int32_t q[4];
  for (int i = 0; i < 4; ++i) q[i] = (int32_t)((u[i] ^ NBMASK) - NBMASK);
  zfp_inv_lift(q);
  for (int i = 0; i < 4; ++i) out[i] = (float)((double)q[i] * ldexp(1.0, emax - 30));
}

/* zfp pad_block for a partial 1-D block of `live` values */
static void zfp_pad(const float* in, uint64_t live, float* blk) {
  for (uint64_t i = 0; i < live; ++i) blk[i] = in[i];
  switch (live) {
    case 0: blk[0] = 0.0f; /* fall through */
    case 1: blk[1] = blk[0]; /* fall through */
    case 2: blk[2] = blk[1]; /* fall through */
    case 3: blk[3] = blk[0]; /* fall through */
    default: break;
  }
}

int orc_zfp_compress(int rate, const float* in, uint64_t n, uint8_t* out) {
  const uint64_t nb = (n + 3) / 4;
  memset(out, 0, orc_wire_size(KIND_ZFP, rate, n));
  for (uint64_t b = 0; b < nb; ++b) {
    float blk[4];
    const uint64_t live = (n - 4 * b < 4) ? n - 4 * b : 4;
    zfp_pad(in + 4 * b, live, blk);
    if (!zfp_encode_block(blk, rate, out, b * 4 * (uint64_t)rate)) return ORC_NONFINITE;
  }
  return ORC_OK;
}

void orc_zfp_decompress(int rate, const uint8_t* in, uint64_t n, float* out) {
  const uint64_t nb = (n + 3) / 4;
  for (uint64_t b = 0; b < nb; ++b) {
    float blk[4];
    zfp_decode_block(in, b * 4 * (uint64_t)rate, rate, blk);
    const uint64_t live = (n - 4 * b < 4) ? n - 4 * b : 4;
    for (uint64_t i = 0; i < live; ++i) out[4 * b + i] = blk[i];
  }
}

/* ------------------------------------------------------------------------ */
/* Generic codec round trip used by the collectives: dec(comp(x)).           */
/* Returns the payload size through *wire.                                   */
/* ------------------------------------------------------------------------ */

static int codec_roundtrip(int kind, int rate, const float* in, uint64_t n, float* out,
                           uint64_t* wire) {
  if (kind == KIND_IDENTITY) {
    memmove(out, in, 4 * n);
    *wire = 4 * n;
    return ORC_OK;
  }
  if (kind == KIND_LOSSLESS) {
    /* lossless: bit-exact round trip; only the payload size matters */
    *wire = orc_pred_size(in, n);
    memmove(out, in, 4 * n);
    return ORC_OK;
  }
  const uint64_t w = orc_wire_size(kind, rate, n);
  uint8_t* tmp = (uint8_t*)malloc(w ? w : 1);
  int st = (kind == KIND_FIXED) ? orc_fr_compress(rate, in, n, tmp) : orc_zfp_compress(rate, in, n, tmp);
  if (st == ORC_OK) {
    if (kind == KIND_FIXED)
      orc_fr_decompress(rate, tmp, n, out);
    else
      orc_zfp_decompress(rate, tmp, n, out);
  }
  free(tmp);
  *wire = w;
  return st;
}

int orc_codec_roundtrip(int kind, int rate, const float* in, uint64_t n, float* out) {
  uint64_t w;
  return codec_roundtrip(kind, rate, in, n, out, &w);
}

/* ------------------------------------------------------------------------ */
/* Ring collectives, value + byte accounting (src/collectives.cpp).          */
/* Buffers are rank-major: rank j's n values at inputs + j*n.                */
/* acct[0] = raw bytes per rank, acct[1] = wire bytes per rank,             */
/* acct[2] = rounds (src/collectives.cpp:113-126).                           */
/* ------------------------------------------------------------------------ */

/* src/collectives.cpp:27-66: p-1 rounds; every member first stages
 * Q(chunk (j-1-round) mod p) from the previous round's values, then member
 * j+1 adds the decoded message on the left: acc = dec + acc. */
static int rs_core(int p, uint64_t n, float* work, int kind, int rate, uint64_t* raw,
                   uint64_t* wire) {
  const uint64_t c = n / (uint64_t)p;
  float* msgs = (float*)malloc(sizeof(float) * (c ? c : 1) * (uint64_t)p);
  int* send_chunk = (int*)malloc(sizeof(int) * (size_t)p);
  int st = ORC_OK;
  for (int round = 0; round < p - 1 && st == ORC_OK; ++round) {
    for (int j = 0; j < p; ++j) {
      const int ch = ((j - 1 - round) % p + p) % p;
      uint64_t w = 0;
      send_chunk[j] = ch;
      st = codec_roundtrip(kind, rate, work + (uint64_t)j * n + (uint64_t)ch * c, c,
                           msgs + (uint64_t)j * c, &w);
      if (st != ORC_OK) break;
      *raw += 4 * c;
      *wire += w;
    }
    if (st != ORC_OK) break;
    for (int j = 0; j < p; ++j) {
      const int dst = (j + 1) % p;
      float* acc = work + (uint64_t)dst * n + (uint64_t)send_chunk[j] * c;
      const float* rx = msgs + (uint64_t)j * c;
      for (uint64_t e = 0; e < c; ++e) acc[e] = rx[e] + acc[e];
    }
  }
  free(msgs);
  free(send_chunk);
  return st;
}

/* src/collectives.cpp:69-111: each shard compressed once at its origin;
 * every member (origin included) keeps dec(shard). */
static int ag_core(int p, uint64_t c, const float* shards, float* out, int kind, int rate,
                   uint64_t* raw, uint64_t* wire) {
  float* dec = (float*)malloc(sizeof(float) * (c ? c : 1) * (uint64_t)p);
  uint64_t* wsz = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)p);
  int st = ORC_OK;
  for (int j = 0; j < p && st == ORC_OK; ++j)
    st = codec_roundtrip(kind, rate, shards + (uint64_t)j * c, c, dec + (uint64_t)j * c, &wsz[j]);
  if (st == ORC_OK) {
    const uint64_t n = c * (uint64_t)p;
    for (int i = 0; i < p; ++i)
      for (int ch = 0; ch < p; ++ch)
        memcpy(out + (uint64_t)i * n + (uint64_t)ch * c, dec + (uint64_t)ch * c, 4 * c);
    for (int round = 0; round < p - 1; ++round)
      for (int j = 0; j < p; ++j) {
        const int ch = ((j - round) % p + p) % p;
        *raw += 4 * c;
        *wire += wsz[ch];
      }
  }
  free(dec);
  free(wsz);
  return st;
}

/* src/collectives.cpp:154-181 */
int orc_reduce_scatter(int p, uint64_t n, const float* inputs, int kind, int rate, float* shards,
                       uint64_t* acct) {
  if (p < 1) return ORC_INVALID;
  if (n % (uint64_t)p) return ORC_BADCHUNK;
  const uint64_t c = n / (uint64_t)p;
  acct[0] = acct[1] = acct[2] = 0;
  if (p == 1) {
    memcpy(shards, inputs, 4 * n);
    return ORC_OK;
  }
  float* work = (float*)malloc(4 * n * (uint64_t)p + 4);
  memcpy(work, inputs, 4 * n * (uint64_t)p);
  uint64_t raw = 0, wire = 0;
  int st = rs_core(p, n, work, kind, rate, &raw, &wire);
  if (st == ORC_OK) {
    for (int i = 0; i < p; ++i)
      memcpy(shards + (uint64_t)i * c, work + (uint64_t)i * n + (uint64_t)i * c, 4 * c);
    acct[0] = raw / (uint64_t)p;
    acct[1] = wire / (uint64_t)p;
    acct[2] = (uint64_t)(p - 1);
  }
  free(work);
  return st;
}

/* src/collectives.cpp:183-200 */
int orc_allgather(int p, uint64_t c, const float* shards, int kind, int rate, float* out,
                  uint64_t* acct) {
  if (p < 1) return ORC_INVALID;
  acct[0] = acct[1] = acct[2] = 0;
  if (p == 1) {
    memcpy(out, shards, 4 * c);
    return ORC_OK;
  }
  uint64_t raw = 0, wire = 0;
  int st = ag_core(p, c, shards, out, kind, rate, &raw, &wire);
  if (st == ORC_OK) {
    acct[0] = raw / (uint64_t)p;
    acct[1] = wire / (uint64_t)p;
    acct[2] = (uint64_t)(p - 1);
  }
  return st;
}

/* src/collectives.cpp:202-248: RS then AG; Average divides by float(p)
 * after the gather.  p == 1 returns the input untouched (:217-219). */
int orc_allreduce(int p, uint64_t n, const float* inputs, int kind, int rate, int average,
                  float* out, uint64_t* acct) {
  if (p < 1) return ORC_INVALID;
  if (n % (uint64_t)p) return ORC_BADCHUNK;
  acct[0] = acct[1] = acct[2] = 0;
  if (p == 1) {
    memcpy(out, inputs, 4 * n);
    return ORC_OK;
  }
  const uint64_t c = n / (uint64_t)p;
  float* work = (float*)malloc(4 * n * (uint64_t)p + 4);
  float* shards = (float*)malloc(4 * n + 4);
  memcpy(work, inputs, 4 * n * (uint64_t)p);
  uint64_t raw = 0, wire = 0;
  int st = rs_core(p, n, work, kind, rate, &raw, &wire);
  if (st == ORC_OK) {
    for (int i = 0; i < p; ++i)
      memcpy(shards + (uint64_t)i * c, work + (uint64_t)i * n + (uint64_t)i * c, 4 * c);
    st = ag_core(p, c, shards, out, kind, rate, &raw, &wire);
  }
  if (st == ORC_OK) {
    if (average) {
      const float scale = (float)p;
      for (uint64_t i = 0; i < n * (uint64_t)p; ++i) out[i] = out[i] / scale;
    }
    acct[0] = raw / (uint64_t)p;
    acct[1] = wire / (uint64_t)p;
    acct[2] = 2 * (uint64_t)(p - 1);
  }
  free(work);
  free(shards);
  return st;
}

/* src/collectives.cpp:130-152: dst receives dec(comp(buf)). */
int orc_p2p(uint64_t n, const float* in, int kind, int rate, float* out, uint64_t* acct) {
  uint64_t w = 0;
  int st = codec_roundtrip(kind, rate, in, n, out, &w);
  acct[0] = 4 * n;
  acct[1] = w;
  acct[2] = 1;
  return st;
}

/* Broadcast is NOT in the reference.  Defined by analogy
 * with the allgather single-shard rule (src/collectives.cpp:77-84): the root
 * compresses once, compressed bytes are forwarded, and every member, root
 * included, holds dec(comp(buf)).  Accounting follows the ring AG: p-1
 * rounds, one message per round. */
int orc_broadcast(int p, uint64_t n, const float* in, int kind, int rate, float* out,
                  uint64_t* acct) {
  acct[0] = acct[1] = acct[2] = 0;
  if (p == 1) {
    memcpy(out, in, 4 * n);
    return ORC_OK;
  }
  uint64_t w = 0;
  int st = codec_roundtrip(kind, rate, in, n, out, &w);
  if (st != ORC_OK) return st;
  for (int i = 1; i < p; ++i) memcpy(out + (uint64_t)i * n, out, 4 * n);
  acct[0] = 4 * n * (uint64_t)(p - 1) / (uint64_t)p;
  acct[1] = w * (uint64_t)(p - 1) / (uint64_t)p;
  acct[2] = (uint64_t)(p - 1);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Test-support restatements (tests/support/oracles.cpp:38-84).              */
/* ------------------------------------------------------------------------ */

/* oracles.cpp:38-50 (frexp-derived exponent, clamped at -127) */
double orc_block_bound(const float* v, uint64_t n, int rate) {
  int emax = -127;
  for (uint64_t i = 0; i < n; ++i) {
    if (v[i] != 0.0f) {
      int e;
      frexpf(v[i], &e);
      e -= 1;
      if (e < -127) e = -127;
      if (e > emax) emax = e;
    }
  }
  return ldexp(1.0, emax - rate + 2);
}

/* oracles.cpp:61-78: chunk i folded left over positions i+1, ..., i+p. */
void orc_ring_fold(int p, uint64_t n, const float* inputs, float* out) {
  const uint64_t c = n / (uint64_t)p;
  for (int ch = 0; ch < p; ++ch)
    for (uint64_t e = 0; e < c; ++e) {
      const uint64_t idx = (uint64_t)ch * c + e;
      float acc = inputs[(uint64_t)((ch + 1) % p) * n + idx];
      for (int s = 2; s <= p; ++s) acc = acc + inputs[(uint64_t)((ch + s) % p) * n + idx];
      out[idx] = acc;
    }
}
