// lossless.cu -- the reference's LosslessPredictor codec on the GPU
// (format of /root/reference/proj/src/codec_kernels.hpp:165-239
// and src/codec_serial.cpp:48-66, :85-107).
//
// Payload = [ceil(nchunks/8) fallback-flag bytes][chunk 0][chunk 1]...; a
// 4096-value chunk is either its raw bytes (flag set, when the coded size
// reaches 4*live) or, per value, the XOR residual against the previous
// value (0 before the chunk) as a 5-bit leading-zero count capped at 31
// followed by the 32-lzc low residual bits, LSB-first, flushed to a byte.
//
// compress: (1) size pass, one warp per chunk -> chunk bytes + flag;
//           (2) exclusive scan of chunk bytes -> offsets (one CTA);
//           (3) emit, one warp per chunk: lanes own 128 consecutive values,
//               write their codes into a shared-memory copy of the chunk
//               stream (word-exclusive stores + atomicOr on the 2 shared
//               boundary words), the warp copies it to its byte offset.
// decompress: the format stores no offsets, so a single-warp walk parses
//           each coded chunk's 5-bit fields to find where the next chunk
//           starts (fallback chunks cost O(1)); then one warp per chunk
//           decodes in parallel from the recovered offsets.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "hccx.h"
#include "hccx_internal.h"
#include "hccx_kernels.h"
#include "lossless_msg.h"

namespace hccx {
namespace {

constexpr int kChunk = 4096;
constexpr int kLaneVals = kChunk / 32;  // 128
constexpr int kLLWarps = 4;             // warps per CTA (16 KiB smem stream each)
constexpr int kStreamWords = kChunk;    // >= 4096 codes * 37 bits / 32

__device__ __forceinline__ uint32_t code_bits(uint32_t r) {
  const uint32_t z = min(__clz(r), 31);
  return 5u + 32u - z;
}

// (1) per-chunk coded bytes / fallback flag
__global__ void __launch_bounds__(kLLWarps * 32) ll_size_kernel(const float* __restrict__ in, uint64_t n,
                                                                uint64_t nchunks, uint32_t* __restrict__ sizes,
                                                                uint8_t* __restrict__ fallback) {
  const int lane = threadIdx.x & 31;
  for (uint64_t c = (static_cast<uint64_t>(blockIdx.x) * kLLWarps + (threadIdx.x >> 5)); c < nchunks;
       c += static_cast<uint64_t>(gridDim.x) * kLLWarps) {
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    const uint32_t* x = reinterpret_cast<const uint32_t*>(in) + base;
    uint64_t bits = 0;
    for (uint32_t i = lane; i < live; i += 32) {
      const uint32_t prev = i ? x[i - 1] : 0u;
      bits += code_bits(x[i] ^ prev);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bits += __shfl_xor_sync(kFull, bits, o);
    if (lane == 0) {
      const uint64_t enc = (bits + 7) / 8;
      const uint64_t raw = 4ull * live;
      sizes[c] = static_cast<uint32_t>(enc < raw ? enc : raw);
      fallback[c] = enc >= raw ? 1 : 0;
    }
  }
}

// (2) exclusive scan of sizes (+ flag bytes), single CTA; offsets[nchunks] = total
__global__ void __launch_bounds__(1024) ll_scan_kernel(const uint32_t* __restrict__ sizes, uint64_t nchunks,
                                                       uint64_t flag_bytes, uint64_t* __restrict__ offsets) {
  __shared__ uint64_t part[1024];
  const uint64_t per = (nchunks + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = threadIdx.x * per, hi = min(nchunks, lo + per);
  uint64_t s = 0;
  for (uint64_t i = lo; i < hi; ++i) s += sizes[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = flag_bytes;
    for (unsigned t = 0; t < blockDim.x; ++t) {
      const uint64_t v = part[t];
      part[t] = acc;
      acc += v;
    }
    offsets[nchunks] = acc;
  }
  __syncthreads();
  uint64_t acc = part[threadIdx.x];
  for (uint64_t i = lo; i < hi; ++i) {
    offsets[i] = acc;
    acc += sizes[i];
  }
}

// flag bytes: bit c%8 of byte c/8 (codec_serial.cpp:63)
__global__ void ll_flags_kernel(const uint8_t* __restrict__ fallback, uint64_t nchunks, uint8_t* __restrict__ out) {
  const uint64_t nb = (nchunks + 7) / 8;
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint8_t v = 0;
    for (int k = 0; k < 8; ++k) {
      const uint64_t c = b * 8 + k;
      if (c < nchunks && fallback[c]) v |= static_cast<uint8_t>(1u << k);
    }
    out[b] = v;
  }
}

// Byte copy of `len` bytes from a word-aligned shared stream to an arbitrary
// global byte offset: interior words stored whole (funnel-shifted), the
// edges bytewise.
__device__ void copy_stream_out(const uint32_t* sm, uint8_t* dst, uint32_t len, int lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  const uint32_t head = static_cast<uint32_t>((4 - (a & 3)) & 3) < len ? static_cast<uint32_t>((4 - (a & 3)) & 3) : len;
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(sm);
  for (uint32_t b = lane; b < head; b += 32) dst[b] = sb[b];
  const uint32_t nw = (len - head) / 4;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
  for (uint32_t w = lane; w < nw; w += 32) {
    const uint32_t byte = head + 4 * w;  // source byte offset
    const uint32_t lo = sm[byte >> 2], hi = (byte & 3) ? sm[(byte >> 2) + 1] : 0u;
    dw[w] = __funnelshift_r(lo, hi, 8 * (byte & 3));
  }
  for (uint32_t b = head + 4 * nw + lane; b < len; b += 32) dst[b] = sb[b];
}

// (3) emit
__global__ void __launch_bounds__(kLLWarps * 32) ll_emit_kernel(const float* __restrict__ in, uint64_t n,
                                                                uint64_t nchunks, const uint64_t* __restrict__ offsets,
                                                                const uint8_t* __restrict__ fallback,
                                                                uint8_t* __restrict__ out) {
  extern __shared__ uint32_t llsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* sm = llsm + warp * (kStreamWords + 2);
  for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * kLLWarps + warp; c < nchunks;
       c += static_cast<uint64_t>(gridDim.x) * kLLWarps) {
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    const uint32_t* x = reinterpret_cast<const uint32_t*>(in) + base;
    uint8_t* dst = out + offsets[c];
    if (fallback[c]) {  // raw chunk (codec_kernels.hpp:190-194)
      copy_stream_out(x, dst, 4 * live, lane);
      continue;
    }
    // lane's bit count and exclusive offset
    const uint32_t i0 = lane * kLaneVals, i1 = min(live, i0 + kLaneVals);
    uint32_t mybits = 0;
    for (uint32_t i = i0; i < i1; ++i) mybits += code_bits(x[i] ^ (i ? x[i - 1] : 0u));
    uint32_t incl = mybits;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    const uint32_t words = (total + 31) / 32;
    for (uint32_t w = lane; w < words + 1; w += 32) sm[w] = 0;
    __syncwarp();
    uint32_t pos = incl - mybits;  // bit offset of this lane's first code
    uint64_t acc = 0;
    uint32_t fill = pos & 31, wi = pos >> 5;
    const uint32_t first_word = wi;
    bool first = true;
    auto put = [&](uint32_t v, uint32_t nb) {  // append nb (<= 32) bits
      acc |= static_cast<uint64_t>(v) << fill;
      fill += nb;
      if (fill >= 32) {
        const uint32_t wv = static_cast<uint32_t>(acc);
        if (first && wi == first_word) atomicOr(&sm[wi], wv);  // shared with the previous lane
        else sm[wi] = wv;
        first = false;
        ++wi;
        acc >>= 32;
        fill -= 32;
      }
    };
    for (uint32_t i = i0; i < i1; ++i) {
      const uint32_t r = x[i] ^ (i ? x[i - 1] : 0u);
      const uint32_t z = min(__clz(r), 31);
      put(z, 5);
      const uint32_t nb = 32 - z;
      put(nb == 32 ? r : (r & ((1u << nb) - 1u)), nb);
    }
    if (fill > 0) atomicOr(&sm[wi], static_cast<uint32_t>(acc));  // may be shared with the next lane
    __syncwarp();
    copy_stream_out(sm, dst, (total + 7) / 8, lane);
    __syncwarp();
  }
}

// decompress (a): offsets by walking coded chunks' 5-bit length fields.
// Serial by format (no stored offsets).  The chain per code is
// pos += 37 - field(pos); the stream is read through a register window of
// two aligned 64-bit words (read-only path), refilled only when the position
// crosses a word, so the dependent chain is a funnel shift, a mask and an add.
__device__ __forceinline__ uint64_t ll_word(const uint8_t* in, uint64_t in_bytes, uint64_t w) {
  const uint64_t b0 = w * 8;
  if (b0 + 8 <= in_bytes) {
    if ((reinterpret_cast<uintptr_t>(in) & 7u) == 0) return __ldg(reinterpret_cast<const unsigned long long*>(in) + w);
    uint64_t v = 0;
    for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(__ldg(in + b0 + k)) << (8 * k);
    return v;
  }
  uint64_t v = 0;
  for (uint64_t k = 0; b0 + k < in_bytes && k < 8; ++k) v |= static_cast<uint64_t>(__ldg(in + b0 + k)) << (8 * k);
  return v;
}

__global__ void ll_walk_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t n, uint64_t nchunks,
                               uint64_t* __restrict__ offsets, uint32_t* __restrict__ err) {
  if (threadIdx.x != 0) return;
  uint64_t pos = (nchunks + 7) / 8;
  const uint64_t end_bit = 8 * in_bytes;
  for (uint64_t c = 0; c < nchunks; ++c) {
    offsets[c] = pos;
    const uint32_t live = static_cast<uint32_t>(n - c * kChunk < kChunk ? n - c * kChunk : kChunk);
    if ((__ldg(in + c / 8) >> (c % 8)) & 1u) {
      pos += 4ull * live;
    } else {
      uint64_t bit = pos * 8;
      uint64_t wi = bit >> 6;
      uint64_t lo = ll_word(in, in_bytes, wi), hi = ll_word(in, in_bytes, wi + 1);
      for (uint32_t i = 0; i < live; ++i) {
        if (bit + 5 > end_bit) {
          bit = end_bit + 1;  // truncated inside a length field
          break;
        }
        const uint64_t w = bit >> 6;
        if (w != wi) {  // advance the window (codes are <= 37 bits: at most one word)
          lo = hi;
          hi = ll_word(in, in_bytes, w + 1);
          if (w != wi + 1) lo = ll_word(in, in_bytes, w);
          wi = w;
        }
        const uint32_t sh = static_cast<uint32_t>(bit & 63);
        const uint64_t win = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
        bit += 5 + (32 - static_cast<uint32_t>(win & 31u));
      }
      pos = bit > end_bit ? in_bytes + 1 : (bit + 7) / 8;
    }
    if (pos > in_bytes) {
      atomicOr(err, 8u);  // truncated stream
      pos = in_bytes;
    }
  }
  offsets[nchunks] = pos;
}

// decompress (a'): the same offsets by pointer doubling.  J0[x] = the bit
// position after the code starting at bit x; twelve rounds of J <- J o J give
// the position after 4096 codes, so a coded chunk starting at byte B ends at
// byte ceil(J12[8B] / 8): the serial walk shrinks to one lookup per chunk.
// Every position of the stream is a candidate start because the chunk starts
// are unknown (the format stores no offsets).
__global__ void ll_jump_kernel(const uint32_t* __restrict__ Jin, uint32_t* __restrict__ Jout, uint64_t total) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    Jout[x] = Jin[Jin[x]];
}

// decompress (a''), memory-bounded: the same doubling over slabs of the
// stream.  A chain of 4096 codes from a slab position ends at most
// kChainBits later, so slab [lo, hi) needs the jump table only over
// [lo, hi + kChainBits): positions are slab-relative (u32), `sent` is the
// absorbing "past the end" index, and the result is kept per payload BYTE
// (chunks start byte-aligned): F[B] = the byte after a coded chunk starting
// at byte B, or ~0u when it would run past the payload.
constexpr uint64_t kChainBits = 4096ull * 37ull;


// The first doublings in 16-bit relative form (a jump of 2^k codes spans at
// most 37 * 2^k bits: < 2^16 up to k = 10), half the table traffic of the
// 32-bit rounds; 0xFFFF = past the end.
constexpr uint16_t kRel16End = 0xFFFFu;
constexpr int kRel16Rounds = 10;

__global__ void ll_jump0_rel16_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t S, uint64_t lo,
                                      uint64_t ext, uint16_t* __restrict__ D) {
  const uint64_t span = ext - lo;
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x <= span;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint16_t d = kRel16End;
    const uint64_t pos = lo + x;
    if (x < span && pos + 5 <= S) {
      const uint64_t B = pos >> 3;
      uint32_t w = __ldg(in + B);
      if (B + 1 < in_bytes) w |= static_cast<uint32_t>(__ldg(in + B + 1)) << 8;
      const uint32_t len = 37u - ((w >> (pos & 7)) & 31u);
      if (pos + len <= S && pos + len <= ext) d = static_cast<uint16_t>(len);
    }
    D[x] = d;
  }
}

__global__ void ll_jump_rel16_kernel(const uint16_t* __restrict__ Din, uint16_t* __restrict__ Dout, uint64_t entries) {
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < entries;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t d = Din[x];
    uint16_t o = kRel16End;
    if (d != kRel16End) {
      const uint32_t d2 = Din[x + d];
      if (d2 != kRel16End) o = static_cast<uint16_t>(d + d2);
    }
    Dout[x] = o;
  }
}

// Last 16-bit doubling, written as 32-bit slab positions (sentinel span + 1).
__global__ void ll_jump_rel16_to32_kernel(const uint16_t* __restrict__ Din, uint32_t* __restrict__ J, uint64_t span) {
  const uint32_t sent = static_cast<uint32_t>(span + 1);
  for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x <= span + 1;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t o = sent;
    if (x <= span) {
      const uint32_t d = Din[x];
      if (d != kRel16End) {
        const uint32_t d2 = Din[x + d];
        if (d2 != kRel16End) o = static_cast<uint32_t>(x + d + d2);
      }
    }
    J[x] = o;
  }
}

__global__ void ll_jump_out_kernel(const uint32_t* __restrict__ J, uint64_t lo, uint64_t hi, uint64_t span,
                                   uint32_t* __restrict__ F) {
  const uint64_t b0 = (lo + 7) / 8, b1 = (hi + 7) / 8;  // bytes whose first bit lies in [lo, hi)
  for (uint64_t b = b0 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < b1;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t e = J[8 * b - lo];
    F[b] = e > span ? ~0u : static_cast<uint32_t>((lo + e + 7) / 8);
  }
}

// Chunk offsets from F: one dependent lookup per coded chunk.
__global__ void ll_walk_f_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t n, uint64_t nch,
                                 const uint32_t* __restrict__ F, uint64_t* __restrict__ offsets,
                                 uint32_t* __restrict__ err) {
  if (threadIdx.x != 0) return;
  uint64_t pos = (nch + 7) / 8;
  const uint64_t end_bit = 8 * in_bytes;
  for (uint64_t c = 0; c < nch; ++c) {
    offsets[c] = pos;
    const uint32_t live = static_cast<uint32_t>(n - c * kChunk < kChunk ? n - c * kChunk : kChunk);
    if ((__ldg(in + c / 8) >> (c % 8)) & 1u) {
      pos += 4ull * live;
    } else if (live == kChunk) {
      const uint32_t b = pos < in_bytes ? F[pos] : ~0u;
      pos = b == ~0u ? in_bytes + 1 : b;
    } else {  // the short last chunk: walk it
      uint64_t bit = pos * 8;
      for (uint32_t i = 0; i < live && bit <= end_bit; ++i) {
        if (bit + 5 > end_bit) {
          bit = end_bit + 1;
          break;
        }
        const uint64_t B = bit >> 3;
        uint32_t w = __ldg(in + B);
        if (B + 1 < in_bytes) w |= static_cast<uint32_t>(__ldg(in + B + 1)) << 8;
        bit += 5 + (32 - ((w >> (bit & 7)) & 31u));
      }
      pos = bit > end_bit ? in_bytes + 1 : (bit + 7) / 8;
    }
    if (pos > in_bytes) {
      atomicOr(err, 8u);
      pos = in_bytes;
    }
  }
  offsets[nch] = pos;
}

// F^(2^k) over payload bytes (F[in_bytes] = ~0u ends every chain).
__global__ void ll_fjump_kernel(const uint32_t* __restrict__ Fin, uint32_t* __restrict__ Fout, uint64_t entries) {
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < entries;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t f = Fin[b];
    Fout[b] = f < entries ? Fin[f] : ~0u;
  }
}

constexpr uint64_t kWalkBlock = 64;  // chunks per anchor block (F^64 jumps)

// Chunk-start anchors every kWalkBlock chunks: a block of full coded chunks
// is one F^64 lookup, any other block is stepped chunk by chunk.
__global__ void ll_walk_anchor_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t n, uint64_t nch,
                                      const uint32_t* __restrict__ F, const uint32_t* __restrict__ F64,
                                      uint64_t* __restrict__ offsets, uint32_t* __restrict__ err) {
  if (threadIdx.x != 0) return;
  uint64_t pos = (nch + 7) / 8;
  for (uint64_t a = 0; a < nch; a += kWalkBlock) {
    offsets[a] = pos;
    const uint64_t e = a + kWalkBlock < nch ? a + kWalkBlock : nch;
    bool uniform = e - a == kWalkBlock && e * kChunk <= n;
    for (uint64_t c = a; c < e && uniform; c += 8)
      if (__ldg(in + c / 8)) uniform = false;  // a raw chunk in the block (8-aligned blocks)
    if (uniform) {
      const uint32_t b = pos < in_bytes ? F64[pos] : ~0u;
      pos = b == ~0u ? in_bytes + 1 : b;
    } else {
      for (uint64_t c = a; c < e && pos <= in_bytes; ++c) {
        const uint32_t live = static_cast<uint32_t>(n - c * kChunk < kChunk ? n - c * kChunk : kChunk);
        if ((__ldg(in + c / 8) >> (c % 8)) & 1u) {
          pos += 4ull * live;
        } else if (live == kChunk) {
          const uint32_t b = pos < in_bytes ? F[pos] : ~0u;
          pos = b == ~0u ? in_bytes + 1 : b;
        } else {
          break;  // the short last chunk: ll_walk_fill_kernel walks it
        }
      }
    }
    if (pos > in_bytes) {
      atomicOr(err, 8u);
      pos = in_bytes;
    }
  }
}

// Every block's chunks from its anchor, one thread per block.
__global__ void ll_walk_fill_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t n, uint64_t nch,
                                    const uint32_t* __restrict__ F, uint64_t* __restrict__ offsets,
                                    uint32_t* __restrict__ err) {
  const uint64_t nblk = (nch + kWalkBlock - 1) / kWalkBlock;
  const uint64_t end_bit = 8 * in_bytes;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nblk;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t a = k * kWalkBlock, e = a + kWalkBlock < nch ? a + kWalkBlock : nch;
    uint64_t pos = offsets[a];
    for (uint64_t c = a; c < e; ++c) {
      offsets[c] = pos;
      const uint32_t live = static_cast<uint32_t>(n - c * kChunk < kChunk ? n - c * kChunk : kChunk);
      if ((__ldg(in + c / 8) >> (c % 8)) & 1u) {
        pos += 4ull * live;
      } else if (live == kChunk) {
        const uint32_t b = pos < in_bytes ? F[pos] : ~0u;
        pos = b == ~0u ? in_bytes + 1 : b;
      } else {  // the short last chunk: walk it
        uint64_t bit = pos * 8;
        for (uint32_t i = 0; i < live && bit <= end_bit; ++i) {
          if (bit + 5 > end_bit) {
            bit = end_bit + 1;
            break;
          }
          const uint64_t B = bit >> 3;
          uint32_t w = __ldg(in + B);
          if (B + 1 < in_bytes) w |= static_cast<uint32_t>(__ldg(in + B + 1)) << 8;
          bit += 5 + (32 - ((w >> (bit & 7)) & 31u));
        }
        pos = bit > end_bit ? in_bytes + 1 : (bit + 7) / 8;
      }
      if (pos > in_bytes) {
        atomicOr(err, 8u);
        pos = in_bytes;
      }
    }
    if (e == nch) offsets[nch] = pos;
  }
}

// decompress (b): raw chunks, one warp per chunk (coalesced copies)
__global__ void __launch_bounds__(kLLWarps * 32) ll_raw_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes,
                                                               uint64_t n, uint64_t nchunks,
                                                               const uint64_t* __restrict__ offsets,
                                                               float* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t c = static_cast<uint64_t>(blockIdx.x) * kLLWarps + warp; c < nchunks;
       c += static_cast<uint64_t>(gridDim.x) * kLLWarps) {
    if (!((__ldg(in + c / 8) >> (c % 8)) & 1u)) continue;
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    const uint8_t* src = in + offsets[c];
    const uint64_t avail = in_bytes - offsets[c];
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + base;
    for (uint32_t i = lane; i < live && 4ull * i + 4 <= avail; i += 32) {
      uint32_t v = 0;
      memcpy(&v, src + 4 * i, 4);
      o[i] = v;
    }
  }
}

// decompress (c): coded chunks, one thread per chunk -- the code chain is
// serial within a chunk, so chunks are the parallelism; the stream is read
// through a 128-bit register window (every code is <= 37 bits).
__global__ void __launch_bounds__(128) ll_decode_kernel(const uint8_t* __restrict__ in, uint64_t in_bytes, uint64_t n,
                                                        uint64_t nchunks, const uint64_t* __restrict__ offsets,
                                                        float* __restrict__ out) {
  for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if ((__ldg(in + c / 8) >> (c % 8)) & 1u) continue;
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    uint32_t* o = reinterpret_cast<uint32_t*>(out) + base;
    uint64_t bit = offsets[c] * 8;
    uint64_t wi = bit >> 6;
    uint64_t lo = ll_word(in, in_bytes, wi), hi = ll_word(in, in_bytes, wi + 1);
    uint32_t prev = 0;
    for (uint32_t i = 0; i < live; ++i) {
      const uint64_t w = bit >> 6;
      if (w != wi) {
        lo = hi;
        hi = ll_word(in, in_bytes, w + 1);
        if (w != wi + 1) lo = ll_word(in, in_bytes, w);
        wi = w;
      }
      const uint32_t sh = static_cast<uint32_t>(bit & 63);
      const uint64_t win = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
      const uint32_t z = static_cast<uint32_t>(win & 31u);
      const uint32_t nb = 32 - z;
      const uint32_t low = static_cast<uint32_t>(win >> 5) & (nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u));
      bit += 5 + nb;
      prev ^= low;
      o[i] = prev;
    }
  }
}

// part = part + x (the ring's "arriving partial on the left" fold,
// collectives.cpp:50-52); plain IEEE fp32 adds.
__global__ void ll_fold_kernel(float* __restrict__ part, const float* __restrict__ x, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    part[i] = __fadd_rn(part[i], x[i]);
}

int grid_for(uint64_t work, int per_block) {
  uint64_t g = (work + per_block - 1) / per_block;
  return static_cast<int>(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

// Dynamic shared memory above 48 KiB is a per-device function attribute:
// set it once per (kernel, device).
void smem_attr(const void* k, size_t bytes, std::atomic<uint64_t>& configured) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    configured.fetch_or(bit);
  }
}
std::atomic<uint64_t> g_emit_attr{0}, g_decode_attr{0};

struct Scratch {
  uint32_t* sizes = nullptr;
  uint8_t* fallback = nullptr;
  uint64_t* offsets = nullptr;
  uint32_t* err = nullptr;
  uint64_t cap = 0;
  uint32_t* jump[2] = {nullptr, nullptr};  // pointer-doubling tables (one slab)
  uint64_t jump_cap = 0;
  uint32_t* fend = nullptr;  // per payload byte: the byte after a coded chunk starting there
  uint64_t fend_cap = 0;
  ~Scratch() {
    cudaFree(jump[0]);
    cudaFree(jump[1]);
    cudaFree(fend);
    cudaFree(sizes);
    cudaFree(fallback);
    cudaFree(offsets);
    cudaFree(err);
  }
  hccx_status_t ensure(uint64_t nchunks) {
    if (nchunks + 1 <= cap && err) return HCCX_OK;
    cudaFree(sizes);
    cudaFree(fallback);
    cudaFree(offsets);
    if (!err && cudaMalloc(&err, 4) != cudaSuccess) return HCCX_CUDA_FAIL;
    const uint64_t c = nchunks + 1;
    if (cudaMalloc(&sizes, 4 * c) != cudaSuccess || cudaMalloc(&fallback, c) != cudaSuccess ||
        cudaMalloc(&offsets, 8 * c) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    cap = c;
    return HCCX_OK;
  }
  bool ensure_fend(uint64_t entries) {
    if (entries <= fend_cap && fend) return true;
    cudaFree(fend);
    fend = nullptr;
    fend_cap = 0;
    if (cudaMalloc(&fend, 4 * entries) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    fend_cap = entries;
    return true;
  }
  void drop_jump() {
    cudaFree(jump[0]);
    cudaFree(jump[1]);
    jump[0] = jump[1] = nullptr;
    jump_cap = 0;
    cudaFree(fend);
    fend = nullptr;
    fend_cap = 0;
  }
  bool ensure_jump(uint64_t entries) {
    if (entries <= jump_cap) return true;
    cudaFree(jump[0]);
    cudaFree(jump[1]);
    jump[0] = jump[1] = nullptr;
    jump_cap = 0;
    if (cudaMalloc(&jump[0], 4 * entries) != cudaSuccess || cudaMalloc(&jump[1], 4 * entries) != cudaSuccess) {
      cudaFree(jump[0]);
      cudaFree(jump[1]);
      jump[0] = jump[1] = nullptr;
      cudaGetLastError();  // clear the allocation failure: fall back to the serial walk
      return false;
    }
    jump_cap = entries;
    return true;
  }
};

hccx_status_t size_pass(const float* d_in, uint64_t n, Scratch& s, cudaStream_t st, uint64_t* total) {
  const uint64_t nch = (n + kChunk - 1) / kChunk;
  hccx_status_t r = s.ensure(nch);
  if (r != HCCX_OK) return r;
  ll_size_kernel<<<grid_for(nch, kLLWarps), kLLWarps * 32, 0, st>>>(d_in, n, nch, s.sizes, s.fallback);
  ll_scan_kernel<<<1, 1024, 0, st>>>(s.sizes, nch, (nch + 7) / 8, s.offsets);
  count_launch(2);
  if (cudaGetLastError() != cudaSuccess) return HCCX_CUDA_FAIL;
  if (total) {
    if (cudaMemcpyAsync(total, s.offsets + nch, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return HCCX_CUDA_FAIL;
  }
  return HCCX_OK;
}

// One scratch per device and host thread (a single-process communicator
// drives several GPUs from one thread).
Scratch& scratch() {
  thread_local Scratch s[16];
  int d = 0;
  cudaGetDevice(&d);
  return s[d & 15];
}

// Pointer doubling runs over slabs of at most kSlabBits stream bits (tables
// 8 bytes per slab bit + halo: ~0.5 GiB), so the scratch is bounded for any
// payload; scratch above kJumpKeepBytes is freed after the call rather than
// pinned for the thread's lifetime.
constexpr uint64_t kSlabBits = 64ull << 20;
constexpr uint64_t kJumpKeepBytes = 1ull << 30;  // slab tables (~0.5 GiB) stay allocated
constexpr uint64_t kFendKeepBytes = 1ull << 30;  // per-byte chunk ends (4 B per payload byte)

}  // namespace
}  // namespace hccx

using namespace hccx;

extern "C" hccx_status_t hccx_lossless_size(const float* d_in, uint64_t n, uint64_t* bytes, void* stream) {
  HCCX_NVTX("hccx_lossless_size");
  if (!bytes || (n && !d_in)) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) {
    *bytes = 0;
    return HCCX_OK;
  }
  return size_pass(d_in, n, scratch(), static_cast<cudaStream_t>(stream), bytes);
}

extern "C" hccx_status_t hccx_lossless_compress(const float* d_in, uint64_t n, uint8_t* d_out, uint64_t capacity,
                                                uint64_t* bytes, void* stream) {
  HCCX_NVTX("hccx_lossless_compress");
  if (!bytes || (n && (!d_in || !d_out))) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) {
    *bytes = 0;
    return HCCX_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch& t_scratch = scratch();
  hccx_status_t r = size_pass(d_in, n, t_scratch, st, bytes);
  if (r != HCCX_OK) return r;
  if (*bytes > capacity) return HCCX_ERR_INVALID_ARGUMENT;
  const uint64_t nch = (n + kChunk - 1) / kChunk;
  const size_t smem = sizeof(uint32_t) * kLLWarps * (kStreamWords + 2);
  smem_attr(reinterpret_cast<const void*>(&ll_emit_kernel), smem, g_emit_attr);
  ll_flags_kernel<<<grid_for((nch + 7) / 8, 256), 256, 0, st>>>(t_scratch.fallback, nch, d_out);
  ll_emit_kernel<<<grid_for(nch, kLLWarps), kLLWarps * 32, smem, st>>>(d_in, n, nch, t_scratch.offsets,
                                                                      t_scratch.fallback, d_out);
  count_launch(2);
  return HCCX_STATUS(cudaGetLastError());
}

extern "C" hccx_status_t hccx_lossless_decompress(const uint8_t* d_in, uint64_t in_bytes, uint64_t n, float* d_out,
                                                  void* stream) {
  HCCX_NVTX("hccx_lossless_decompress");
  if (n && (!d_in || !d_out)) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) return HCCX_OK;
  const uint64_t nch = (n + kChunk - 1) / kChunk;
  if (in_bytes < (nch + 7) / 8) return HCCX_ERR_CORRUPT_PAYLOAD;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Scratch& t_scratch = scratch();
  hccx_status_t r = t_scratch.ensure(nch);
  if (r != HCCX_OK) return r;
  cudaMemsetAsync(t_scratch.err, 0, 4, st);
  // Offsets: pointer doubling (slab by slab, bounded scratch) when there
  // are many coded chunks, else the serial walk (cheap for few or raw
  // chunks: O(1) per raw chunk).
  const uint64_t S = 8 * in_bytes;
  bool jump = nch >= 64 && in_bytes < (1ull << 32) - 1 && std::getenv("HCCX_LL_SERIAL") == nullptr;
  if (jump) {  // count the coded chunks from the flag bytes
    std::vector<uint8_t> flags((nch + 7) / 8);
    if (cudaMemcpyAsync(flags.data(), d_in, flags.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    uint64_t raw = 0;
    for (uint64_t c = 0; c < nch; ++c) raw += (flags[c / 8] >> (c % 8)) & 1u;
    const uint64_t slab = S < kSlabBits ? S : kSlabBits;
    jump = nch - raw >= 64 && t_scratch.ensure_jump(slab + kChainBits + 2) && t_scratch.ensure_fend(in_bytes + 1);
  }
  if (jump) {
    const int g = 148 * 8;
    for (uint64_t lo = 0; lo < S; lo += kSlabBits) {
      const uint64_t hi = lo + kSlabBits < S ? lo + kSlabBits : S;
      const uint64_t ext = hi + kChainBits < S ? hi + kChainBits : S;
      const uint64_t span = ext - lo;
      // J0 .. J10 as 16-bit relative jumps, J11 into 32 bits, J12
      uint16_t* d16[2] = {reinterpret_cast<uint16_t*>(t_scratch.jump[0]),
                          reinterpret_cast<uint16_t*>(t_scratch.jump[1])};
      ll_jump0_rel16_kernel<<<g, 256, 0, st>>>(d_in, in_bytes, S, lo, ext, d16[0]);
      int cur = 0;
      for (int r = 0; r < kRel16Rounds; ++r, cur ^= 1)
        ll_jump_rel16_kernel<<<g, 256, 0, st>>>(d16[cur], d16[cur ^ 1], span + 1);
      ll_jump_rel16_to32_kernel<<<g, 256, 0, st>>>(d16[cur], t_scratch.jump[cur ^ 1], span);
      cur ^= 1;
      ll_jump_kernel<<<g, 256, 0, st>>>(t_scratch.jump[cur], t_scratch.jump[cur ^ 1], span + 2);
      cur ^= 1;
      ll_jump_out_kernel<<<g, 256, 0, st>>>(t_scratch.jump[cur], lo, hi, span, t_scratch.fend);
      count_launch(4 + kRel16Rounds);
    }
    // chunk starts: F^64 by six doubling rounds over the payload's bytes
    // (in the slab tables, free now), anchors every 64 chunks, then every
    // block filled in parallel -- or the plain chain when the bytes do not fit
    const uint64_t entries = in_bytes + 1;
    if (entries <= t_scratch.jump_cap && nch >= 2 * kWalkBlock) {
      cudaMemsetAsync(t_scratch.fend + in_bytes, 0xff, 4, st);
      const int g = 148 * 8;
      const uint32_t* src = t_scratch.fend;
      int cur = 0;
      for (int r = 0; r < 6; ++r, cur ^= 1) {
        ll_fjump_kernel<<<g, 256, 0, st>>>(src, t_scratch.jump[cur], entries);
        src = t_scratch.jump[cur];
      }
      ll_walk_anchor_kernel<<<1, 32, 0, st>>>(d_in, in_bytes, n, nch, t_scratch.fend, src, t_scratch.offsets,
                                              t_scratch.err);
      ll_walk_fill_kernel<<<grid_for((nch + kWalkBlock - 1) / kWalkBlock, 128), 128, 0, st>>>(
          d_in, in_bytes, n, nch, t_scratch.fend, t_scratch.offsets, t_scratch.err);
      count_launch(8);
    } else {
      ll_walk_f_kernel<<<1, 32, 0, st>>>(d_in, in_bytes, n, nch, t_scratch.fend, t_scratch.offsets, t_scratch.err);
      count_launch();
    }
  } else {
    ll_walk_kernel<<<1, 32, 0, st>>>(d_in, in_bytes, n, nch, t_scratch.offsets, t_scratch.err);
  }
  ll_raw_kernel<<<grid_for(nch, kLLWarps), kLLWarps * 32, 0, st>>>(d_in, in_bytes, n, nch, t_scratch.offsets, d_out);
  ll_decode_kernel<<<static_cast<unsigned>((nch + 127) / 128), 128, 0, st>>>(d_in, in_bytes, n, nch, t_scratch.offsets,
                                                                          d_out);
  count_launch(1);
  count_launch(2);
  if (cudaGetLastError() != cudaSuccess) return HCCX_CUDA_FAIL;
  uint32_t e = 0;
  uint64_t end = 0;
  if (cudaMemcpyAsync(&e, t_scratch.err, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpyAsync(&end, t_scratch.offsets + nch, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return HCCX_CUDA_FAIL;
  (void)end;  // trailing bytes are ignored, as in codec_serial.cpp:85-107
  // do not pin large scratch for the thread's lifetime
  if (8 * t_scratch.jump_cap > kJumpKeepBytes || 4 * t_scratch.fend_cap > kFendKeepBytes) t_scratch.drop_jump();
  if (e) return HCCX_ERR_CORRUPT_PAYLOAD;
  return HCCX_OK;
}

extern "C" uint64_t hccx_lossless_max_bytes(uint64_t n) {
  const uint64_t nch = (n + kChunk - 1) / kChunk;
  return (nch + 7) / 8 + 4 * n;
}

extern "C" hccx_status_t hccx_lossless_compress_host(const float* h_in, uint64_t n, uint8_t* h_out,
                                                     uint64_t capacity, uint64_t* bytes, int device) {
  HCCX_NVTX("hccx_lossless_compress_host");
  if (!bytes || (n && (!h_in || !h_out))) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) {
    *bytes = 0;
    return HCCX_OK;
  }
  DeviceGuard g(device);
  float* d_in = nullptr;
  uint8_t* d_out = nullptr;
  const uint64_t cap = hccx_lossless_max_bytes(n);
  hccx_status_t r = HCCX_OK;
  if (cudaMalloc(&d_in, 4 * n) != cudaSuccess || cudaMalloc(&d_out, cap) != cudaSuccess) r = HCCX_ERR_CUDA;
  if (r == HCCX_OK && cudaMemcpy(d_in, h_in, 4 * n, cudaMemcpyHostToDevice) != cudaSuccess) r = HCCX_ERR_CUDA;
  if (r == HCCX_OK) r = hccx_lossless_compress(d_in, n, d_out, cap, bytes, nullptr);
  if (r == HCCX_OK && *bytes > capacity) r = HCCX_ERR_INVALID_ARGUMENT;
  if (r == HCCX_OK && cudaMemcpy(h_out, d_out, *bytes, cudaMemcpyDeviceToHost) != cudaSuccess) r = HCCX_ERR_CUDA;
  cudaFree(d_in);
  cudaFree(d_out);
  return r;
}

extern "C" hccx_status_t hccx_lossless_decompress_host(const uint8_t* h_in, uint64_t bytes, uint64_t n, float* h_out,
                                                       int device) {
  HCCX_NVTX("hccx_lossless_decompress_host");
  if (n && (!h_in || !h_out)) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) return HCCX_OK;
  DeviceGuard g(device);
  uint8_t* d_in = nullptr;
  float* d_out = nullptr;
  hccx_status_t r = HCCX_OK;
  if (cudaMalloc(&d_in, bytes ? bytes : 1) != cudaSuccess || cudaMalloc(&d_out, 4 * n) != cudaSuccess)
    r = HCCX_ERR_CUDA;
  if (r == HCCX_OK && bytes && cudaMemcpy(d_in, h_in, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    r = HCCX_ERR_CUDA;
  if (r == HCCX_OK) r = hccx_lossless_decompress(d_in, bytes, n, d_out, nullptr);
  if (r == HCCX_OK && cudaMemcpy(h_out, d_out, 4 * n, cudaMemcpyDeviceToHost) != cudaSuccess) r = HCCX_ERR_CUDA;
  cudaFree(d_in);
  cudaFree(d_out);
  return r;
}

// Ring wire bytes under LosslessPredictor (see hccx.h).
extern "C" hccx_status_t hccx_lossless_ring_hops(const float* const* d_in, int p, uint64_t n, int collective,
                                                 uint64_t* hop, void* stream) {
  HCCX_NVTX("hccx_lossless_ring_hops");
  if (!hop || !d_in || p < 1 || p > 16 || collective < 0 || collective > 2) return HCCX_ERR_INVALID_ARGUMENT;
  if (p == 1) return HCCX_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t sz = 0;
  hccx_status_t r = HCCX_OK;
  if (collective == 1) {  // allgather: shard j is compressed once (collectives.cpp:77-84)
    for (int j = 0; j < p && r == HCCX_OK; ++j) {
      r = n ? hccx_lossless_size(d_in[j], n, &sz, stream) : HCCX_OK;
      hop[j] = n ? sz : 0;
    }
    return r;
  }
  if (n % p) return HCCX_ERR_BAD_CHUNKING;
  const uint64_t c = n / p;
  const uint64_t nrs = static_cast<uint64_t>(p - 1) * p;
  if (c == 0) {
    for (uint64_t i = 0; i < nrs + (collective == 2 ? p : 0); ++i) hop[i] = 0;
    return HCCX_OK;
  }
  float* part = nullptr;
  if (cudaMalloc(&part, 4 * c) != cudaSuccess) return HCCX_CUDA_FAIL;
  for (int k = 0; k < p && r == HCCX_OK; ++k) {
    // chunk k: the round-t message is sent by member (k+1+t) mod p and holds
    // the fold of members k+1 .. k+1+t (collectives.cpp:34-61)
    if (cudaMemcpyAsync(part, d_in[(k + 1) % p] + k * c, 4 * c, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      r = HCCX_ERR_CUDA;
      break;
    }
    for (int t = 0; t < p - 1 && r == HCCX_OK; ++t) {
      r = hccx_lossless_size(part, c, &sz, stream);
      hop[static_cast<uint64_t>(t) * p + (k + 1 + t) % p] = sz;
      ll_fold_kernel<<<grid_for(c, 256 * 4), 256, 0, st>>>(part, d_in[(k + 2 + t) % p] + k * c, c);
      count_launch();
    }
    if (r == HCCX_OK && collective == 2) {  // allreduce: member k's reduced shard, compressed once
      r = hccx_lossless_size(part, c, &sz, stream);
      hop[nrs + k] = sz;
    }
  }
  cudaStreamSynchronize(st);
  cudaFree(part);
  return r;
}

extern "C" hccx_status_t hccx_lossless_ring_wire(const float* const* d_in, int p, uint64_t n, int collective,
                                                 uint64_t* wire, void* stream) {
  HCCX_NVTX("hccx_lossless_ring_wire");
  if (!wire || !d_in || p < 1 || p > 16 || collective < 0 || collective > 2) return HCCX_ERR_INVALID_ARGUMENT;
  *wire = 0;
  if (p == 1 || n == 0) return HCCX_OK;
  uint64_t hop[16 * 16 + 16] = {};
  const hccx_status_t r = hccx_lossless_ring_hops(d_in, p, n, collective, hop, stream);
  if (r != HCCX_OK) return r;
  const uint64_t nrs = collective == 1 ? 0 : static_cast<uint64_t>(p - 1) * p;
  for (uint64_t i = 0; i < nrs; ++i) *wire += hop[i];
  if (collective != 0)  // each compressed shard crosses p-1 allgather hops (collectives.cpp:94-106)
    for (int k = 0; k < p; ++k) *wire += static_cast<uint64_t>(p - 1) * hop[nrs + k];
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_lossless_ring_wire_host(const float* const* h_in, int p, uint64_t n, int collective,
                                                      uint64_t* wire, int device) {
  HCCX_NVTX("hccx_lossless_ring_wire_host");
  if (!wire || !h_in || p < 1 || p > 16) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard g(device);
  float* d[16] = {};
  hccx_status_t r = HCCX_OK;
  for (int j = 0; j < p && r == HCCX_OK; ++j) {
    if (cudaMalloc(&d[j], 4 * (n ? n : 1)) != cudaSuccess ||
        (n && cudaMemcpy(d[j], h_in[j], 4 * n, cudaMemcpyHostToDevice) != cudaSuccess))
      r = HCCX_ERR_CUDA;
  }
  if (r == HCCX_OK) r = hccx_lossless_ring_wire(d, p, n, collective, wire, nullptr);
  for (int j = 0; j < p; ++j) cudaFree(d[j]);
  return r;
}

extern "C" hccx_status_t hccx_lossless_ring_hops_host(const float* const* h_in, int p, uint64_t n, int collective,
                                                      uint64_t* hop, int device) {
  HCCX_NVTX("hccx_lossless_ring_hops_host");
  if (!hop || !h_in || p < 1 || p > 16) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard g(device);
  float* d[16] = {};
  hccx_status_t r = HCCX_OK;
  for (int j = 0; j < p && r == HCCX_OK; ++j) {
    if (cudaMalloc(&d[j], 4 * (n ? n : 1)) != cudaSuccess ||
        (n && cudaMemcpy(d[j], h_in[j], 4 * n, cudaMemcpyHostToDevice) != cudaSuccess))
      r = HCCX_ERR_CUDA;
  }
  if (r == HCCX_OK) r = hccx_lossless_ring_hops(d, p, n, collective, hop, nullptr);
  for (int j = 0; j < p; ++j) cudaFree(d[j]);
  return r;
}

// ---------------------------------------------------------------------------
// Framed messages with a chunk index (lossless_msg.h): the communicator's
// LosslessPredictor transport.

namespace hccx {
namespace {

__device__ __forceinline__ uint64_t ld_le64(const uint8_t* p) {
  uint64_t v = 0;
  for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(p[k]) << (8 * k);
  return v;
}

__device__ void write_frame(uint8_t* msg, uint64_t payload, uint64_t n, uint64_t nch, uint64_t idx_bytes,
                            unsigned long long* acct) {
  const uint64_t container = 18 + payload;
  uint8_t h[26];
  for (int i = 0; i < 8; ++i) h[i] = static_cast<uint8_t>(container >> (8 * i));
  h[8] = 'H', h[9] = 'C', h[10] = 'C', h[11] = '1';
  h[12] = HCCX_CODEC_LOSSLESS;  // kind
  h[13] = 0;                    // rate_bits
  for (int i = 0; i < 8; ++i) h[14 + i] = static_cast<uint8_t>(n >> (8 * i));
  for (int i = 0; i < 4; ++i) h[22 + i] = static_cast<uint8_t>(nch >> (8 * i));
  for (int i = 0; i < 26; ++i) msg[i] = h[i];
  if (acct) {
    atomicAdd(acct, static_cast<unsigned long long>(payload));
    atomicAdd(acct + 1, static_cast<unsigned long long>(kMsgHeaderBytes + idx_bytes + payload));
  }
}

// The frame of an empty message (n = 0).
__global__ void msg_header_kernel(uint8_t* msg, uint64_t* total, unsigned long long* acct) {
  if (threadIdx.x != 0) return;
  *total = 0;
  write_frame(msg, 0, 0, 0, 0, acct);
}

// ---- single-pass encoder ---------------------------------------------------
// One CTA per 4096-value chunk, chunks taken in ticket order.  The chunk is
// staged into shared memory by one bulk copy (TMA engine); each of the 256
// threads then owns 16 consecutive values (the predecessor of its first one
// is in shared memory too), counts their code bits, and a block-wide scan
// gives every thread its bit offset and the chunk its size -- so a raw
// fallback (codec_kernels.hpp:190-194) is known before anything is coded.
// Coded chunks: every thread writes its codes into a shared-memory copy of
// the chunk stream (whole words plain, the two words it may share with its
// neighbours by atomicOr).  The chunk's size is published, its byte offset
// found by a decoupled look-back over the predecessors' descriptors (warp
// 0), and the CTA writes the chunk, its index entry, the raw-flag byte of its
// group of 8 and (last chunk) the frame.
constexpr int kEncThreads = 256;
constexpr int kEncVals = kChunk / kEncThreads;  // 16
constexpr uint32_t kEncStreamWords = kChunk + 8;  // a coded chunk is < 4096 words
constexpr size_t kEncSmem = sizeof(uint32_t) * (kChunk + kEncStreamWords + 80);

// descriptor: epoch (24) | status (2: 1 aggregate, 2 inclusive prefix) | raw flag (1) | value (37).
// Self-contained (no other data is published through it): relaxed accesses.
constexpr uint64_t kDescValMask = (1ull << 37) - 1;
__device__ __forceinline__ uint64_t desc_make(uint32_t epoch, uint32_t status, uint32_t fb, uint64_t v) {
  return (static_cast<uint64_t>(epoch & 0xffffffu) << 40) | (static_cast<uint64_t>(status) << 38) |
         (static_cast<uint64_t>(fb) << 37) | (v & kDescValMask);
}
__device__ __forceinline__ void st_relaxed_gpu_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Spin until descriptor j of this epoch is published; returns it.
__device__ __forceinline__ uint64_t desc_wait(const uint64_t* desc, uint64_t j, uint32_t epoch) {
  uint64_t d = ld_relaxed_gpu_u64(desc + j);
  while (static_cast<uint32_t>(d >> 40) != (epoch & 0xffffffu) || ((d >> 38) & 3u) == 0) {
    __nanosleep(20);
    d = ld_relaxed_gpu_u64(desc + j);
  }
  return d;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Exclusive byte offset of chunk c: `base` (the flag bytes) + the sizes of
// chunks 0..c-1, from the nearest inclusive prefix back (one warp).
__device__ uint64_t lookback(const uint64_t* desc, uint64_t c, uint32_t epoch, uint64_t base, int lane) {
  uint64_t excl = 0;
  int64_t pred = static_cast<int64_t>(c) - 1;
  while (true) {
    const int64_t j = pred - lane;
    uint32_t status = 2;
    uint64_t val = base;
    if (j >= 0) {
      const uint64_t d = desc_wait(desc, static_cast<uint64_t>(j), epoch);
      status = static_cast<uint32_t>((d >> 38) & 3u);
      val = d & kDescValMask;
    }
    const uint32_t pmask = __ballot_sync(kFull, status == 2);
    const int firstp = pmask ? __ffs(pmask) - 1 : 32;
    excl += warp_sum_u64(lane <= firstp ? val : 0ull);
    if (pmask) return excl;
    pred -= 32;
  }
}

// Byte copy of `len` bytes from a word-aligned source to an arbitrary
// global byte offset by a whole CTA (interior words funnel-shifted).
__device__ void copy_out_cta(const uint32_t* src, uint8_t* dst, uint32_t len, int tid, int nt) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
  const uint32_t h4 = static_cast<uint32_t>((4 - (a & 3)) & 3);
  const uint32_t head = h4 < len ? h4 : len;
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(src);
  for (uint32_t b = tid; b < head; b += nt) dst[b] = sb[b];
  const uint32_t nw = (len - head) / 4;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
  for (uint32_t w = tid; w < nw; w += nt) {
    const uint32_t byte = head + 4 * w;
    const uint32_t lo = src[byte >> 2], hi = (byte & 3) ? src[(byte >> 2) + 1] : 0u;
    dw[w] = __funnelshift_r(lo, hi, 8 * (byte & 3));
  }
  for (uint32_t b = head + 4 * nw + tid; b < len; b += nt) dst[b] = sb[b];
}

__global__ void __launch_bounds__(kEncThreads) ll_encode_kernel(const float* __restrict__ in, uint64_t n, uint64_t nch,
                                                                int vec_ok, uint8_t* __restrict__ pay,
                                                                uint32_t* __restrict__ index, uint8_t* msg,
                                                                uint64_t idx_bytes, uint64_t* desc, uint32_t epoch,
                                                                uint64_t* total, unsigned long long* tickets,
                                                                unsigned long long* acct) {
  extern __shared__ __align__(16) uint32_t esm[];
  uint32_t* xin = esm;                       // the chunk's values
  uint32_t* sm = xin + kChunk;               // its code stream
  uint32_t* misc = sm + kEncStreamWords;     // 80 words: warp totals, block bits, broadcast slots, mbarrier
  uint32_t* wtot = misc;                     // [8]
  uint32_t* blk = misc + 8;                  // [64] bits per 64-value block (the index's sub-lane counts)
  uint64_t* bcast = reinterpret_cast<uint64_t*>(misc + 72);  // [0] ticket, [1] offset
  uint64_t* bar = reinterpret_cast<uint64_t*>(misc + 76);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  const uint64_t flag_bytes = (nch + 7) / 8;
  for (;;) {
    // chunks in ticket order: a CTA holds chunk c only after chunks < c were
    // taken by running CTAs, so the look-back cannot wait on an unscheduled one
    if (tid == 0) bcast[0] = atomicAdd(tickets, 1ull);
    __syncthreads();
    const uint64_t c = bcast[0];
    if (c >= nch) {  // the last CTA out resets the counters for the next call
      if (tid == 0 && atomicAdd(tickets + 1, 1ull) == gridDim.x - 1ull) {
        tickets[0] = 0;
        tickets[1] = 0;
      }
      break;
    }
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    const uint32_t* x = reinterpret_cast<const uint32_t*>(in) + base;
    // stage the chunk: one bulk copy of its 16-byte multiple, the tail by hand
    const uint32_t bulk = vec_ok ? (4 * live) & ~15u : 0u;
    if (bulk && tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, bulk);
      bulk_g2s(xin, x, bulk, bar);
    }
    for (uint32_t k = bulk / 4 + tid; k < live; k += kEncThreads) xin[k] = __ldg(x + k);
    if (bulk) {
      mbar_wait(bar, phase);
      phase ^= 1;
    }
    __syncthreads();
    // count: this thread's 16 values
    const uint32_t i0 = tid * kEncVals;
    const uint32_t nv = i0 >= live ? 0u : min(static_cast<uint32_t>(kEncVals), live - i0);
    // values as 4 x 128-bit shared loads (a full chunk; the tail chunk reads
    // zeros past `live`, which the counts below ignore)
    uint32_t xv[kEncVals];
#pragma unroll
    for (int q = 0; q < kEncVals / 4; ++q) {
      const uint4 t4 = *reinterpret_cast<const uint4*>(xin + i0 + 4 * q);
      xv[4 * q] = t4.x, xv[4 * q + 1] = t4.y, xv[4 * q + 2] = t4.z, xv[4 * q + 3] = t4.w;
    }
    const uint32_t before = i0 && i0 <= live ? xin[i0 - 1] : 0u;
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < kEncVals; ++k) {
      const uint32_t r = xv[k] ^ (k ? xv[k - 1] : before);
      bits += static_cast<uint32_t>(k) < nv ? 37u - min(__clz(r), 31) : 0u;
    }
    uint32_t incl = bits;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    // bits per 64-value block = 4 consecutive threads
    const uint32_t end4 = __shfl_sync(kFull, incl, (lane & ~3) + 3);
    const uint32_t beg4 = __shfl_sync(kFull, incl - bits, lane & ~3);
    if ((lane & 3) == 0) blk[warp * 8 + (lane >> 2)] = end4 - beg4;
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0, chunk_bits = 0;
#pragma unroll
    for (int w = 0; w < kEncThreads / 32; ++w) {
      const uint32_t t = wtot[w];
      wbase += w < warp ? t : 0u;
      chunk_bits += t;
    }
    const uint32_t fb = chunk_bits >= 32u * live ? 1u : 0u;
    const uint64_t size = fb ? 4ull * live : (chunk_bits + 7) / 8;
    // the size is known: publish it now, so successors' look-backs see it
    // while this chunk is still being coded
    if (tid == 0) st_relaxed_gpu_u64(desc + c, desc_make(epoch, c == 0 ? 2u : 1u, fb, c == 0 ? flag_bytes + size : size));
    if (!fb) {
      const uint32_t words = (chunk_bits + 31) / 32;
      for (uint32_t w = tid; w < words; w += kEncThreads) sm[w] = 0;
      __syncthreads();
    }
    // warp 0 looks back (and publishes the inclusive prefix) while the other
    // warps write their codes; then it writes its own
    if (warp == 0) {
      const uint64_t off = c == 0 ? flag_bytes : lookback(desc, c, epoch, flag_bytes, lane);
      if (lane == 0) {
        if (c != 0) st_relaxed_gpu_u64(desc + c, desc_make(epoch, 2u, fb, off + size));
        bcast[1] = off;
      }
    }
    if (!fb) {
      const uint32_t pos = wbase + incl - bits;
      uint64_t acc = 0;
      uint32_t fill = pos & 31, wi = pos >> 5;
      const uint32_t first_word = wi;
      auto put = [&](uint32_t val, uint32_t nb) {
        acc |= static_cast<uint64_t>(val) << fill;
        fill += nb;
        if (fill >= 32) {
          const uint32_t wv = static_cast<uint32_t>(acc);
          if (wi == first_word) atomicOr(&sm[wi], wv);  // shared with the previous thread
          else sm[wi] = wv;
          ++wi;
          acc >>= 32;
          fill -= 32;
        }
      };
#pragma unroll
      for (int k = 0; k < kEncVals; ++k) {
        if (static_cast<uint32_t>(k) < nv) {
          const uint32_t r = xv[k] ^ (k ? xv[k - 1] : before);
          const uint32_t z = min(__clz(r), 31);
          put(z, 5);
          const uint32_t nb = 32 - z;
          put(nb == 32 ? r : (r & ((1u << nb) - 1u)), nb);
        }
      }
      if (fill > 0 && bits) atomicOr(&sm[wi], static_cast<uint32_t>(acc));  // may be shared with the next thread
    }
    __syncthreads();
    const uint64_t off = bcast[1];
    copy_out_cta(fb ? xin : sm, pay + off, static_cast<uint32_t>(size), tid, kEncThreads);
    if (index && tid < static_cast<int>(kMsgIndexWords)) {  // offset, then 64 u16 block bit counts
      uint32_t* ix = index + kMsgIndexWords * c;
      ix[tid] = tid == 0 ? static_cast<uint32_t>(off)
                         : (fb ? 0u : (blk[2 * (tid - 1)] | (blk[2 * (tid - 1) + 1] << 16)));
    }
    // raw-flag byte of chunks 8k..8k+7 (codec_serial.cpp:63), by the group's last chunk
    if (warp == 1 && ((c & 7) == 7 || c == nch - 1)) {
      const uint64_t j = (c & ~7ull) + lane;
      uint32_t bit = 0;
      if (lane < 8 && j <= c) bit = j == c ? fb : static_cast<uint32_t>((desc_wait(desc, j, epoch) >> 37) & 1u);
      const uint32_t byte = __ballot_sync(kFull, bit != 0) & 0xffu;
      if (lane == 0) pay[c / 8] = static_cast<uint8_t>(byte);
    }
    if (c == nch - 1 && tid == 0) {
      *total = off + size;
      if (msg) write_frame(msg, off + size, n, nch, idx_bytes, acct);
    }
    __syncthreads();
  }
}

struct MsgDsts {
  uint8_t* d[kMsgMaxDsts];
  int nd;
};

__global__ void msg_copy_kernel(const uint8_t* __restrict__ src, MsgDsts D, uint64_t idx_bytes,
                                unsigned long long* acct) {
  const uint64_t payload = *reinterpret_cast<const uint64_t*>(src) - 18;
  const uint64_t bytes = kMsgHeaderBytes + idx_bytes + payload;
  const uint64_t vec = (bytes + 15) / 16;  // msg_max_bytes leaves 16 bytes of slack
  const uint4* s = reinterpret_cast<const uint4*>(src);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < vec;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = s[i];
    for (int k = 0; k < D.nd; ++k) reinterpret_cast<uint4*>(D.d[k])[i] = v;
  }
  if (acct && blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(acct, static_cast<unsigned long long>(payload * D.nd));
    atomicAdd(acct + 1, static_cast<unsigned long long>(bytes * D.nd));
  }
}

// ---- decoder -----------------------------------------------------------------
// One CTA (4 warps) per chunk.  The chunk's bytes (and, folding, the
// accumulator's 16 KiB) are staged into shared memory by bulk copies (TMA
// engine).  Coded chunks: warp 0's 32 lanes decode the chunk as 64
// independent 64-code chains from their indexed bit positions into lane-major
// shared memory and scan the lanes' XOR carries (x_i = x_{i-1} ^ r_i within a
// chunk); then all four warps assemble the chunk (+ accumulator)
// contiguously, and one bulk store writes it out.  Raw chunks are assembled
// by all warps straight from the staged bytes.  Unaligned outputs take plain
// loads and stores.
constexpr int kDecThreads = 128;
constexpr uint32_t kDecInWords = kChunk + 12;       // 16 KiB + alignment head/tail
constexpr uint32_t kMsgLaneStride = kLaneVals + 1;  // 129: conflict-free lane-major staging
constexpr uint32_t kDecWords = kDecInWords + 32 * kMsgLaneStride + kChunk + 64 + 8;
constexpr size_t kMsgDecodeSmem = sizeof(uint32_t) * kDecWords;
static_assert(kDecInWords % 4 == 0 && (32 * kMsgLaneStride) % 4 == 0, "16-byte aligned regions");

__global__ void __launch_bounds__(kDecThreads) msg_decode_kernel(const uint8_t* __restrict__ msg, uint64_t msg_cap,
                                                                 uint64_t n, uint64_t nch, uint64_t idx_bytes,
                                                                 float* __restrict__ out, int fold,
                                                                 uint32_t* __restrict__ err,
                                                                 unsigned long long* recv_acct) {
  extern __shared__ __align__(16) uint32_t msm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* ins = msm;
  uint32_t* sm = ins + kDecInWords;            // lane-major decoded values
  uint32_t* io = sm + 32 * kMsgLaneStride;     // contiguous chunk: accumulator in, values out
  uint32_t* carry = io + kChunk;               // [64]: lane carries, chain-a totals
  uint64_t* bar = reinterpret_cast<uint64_t*>(carry + 64);
  uint32_t* status = carry + 66;               // CTA-wide "bad chunk" flag
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  // frame checks (hcc::from_bytes, codec.cpp:101-121)
  const uint64_t container = *reinterpret_cast<const uint64_t*>(msg);
  const uint64_t flag_bytes = (nch + 7) / 8;
  const bool frame_ok = container >= 18 && msg[8] == 'H' && msg[9] == 'C' && msg[10] == 'C' && msg[11] == '1' &&
                        msg[12] == HCCX_CODEC_LOSSLESS && ld_le64(msg + 14) == n &&
                        (ld_le64(msg + 22) & 0xffffffffull) == nch && container - 18 >= flag_bytes &&
                        kMsgHeaderBytes + idx_bytes + (container - 18) + 16 <= msg_cap;
  if (!frame_ok) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(err, kErrCorrupt);
    return;
  }
  const uint64_t payload = container - 18;
  if (recv_acct && blockIdx.x == 0 && tid == 0) atomicAdd(recv_acct, static_cast<unsigned long long>(payload));
  const uint32_t* idx = reinterpret_cast<const uint32_t*>(msg + kMsgHeaderBytes);
  const uint8_t* pay = msg + kMsgHeaderBytes + idx_bytes;
  uint32_t* o32 = reinterpret_cast<uint32_t*>(out);
  const bool out_al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint64_t base = c * kChunk;
    const uint32_t live = static_cast<uint32_t>(n - base < kChunk ? n - base : kChunk);
    const uint32_t* e = idx + kMsgIndexWords * c;
    const uint64_t off = e[0];
    const uint64_t end = c + 1 < nch ? idx[kMsgIndexWords * (c + 1)] : payload;
    const bool raw = (pay[c / 8] >> (c % 8)) & 1u;
    if (off < flag_bytes || end < off || end > payload || end - off > 4ull * live || (raw && end - off != 4ull * live)) {
      if (tid == 0) atomicOr(err, kErrCorrupt);
      break;  // CTA-uniform
    }
    // stage [off & ~15, end) rounded up to 16 bytes, and the accumulator
    const uint64_t a0 = off & ~15ull;
    const uint32_t in_bytes = static_cast<uint32_t>((end - a0 + 15) & ~15ull);
    const uint32_t acc_bulk = fold && out_al ? (4 * live) & ~15u : 0u;
    if (tid == 0) bulk_wait_read<0>();  // the previous chunk's store has read io
    __syncthreads();
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(bar, in_bytes + acc_bulk);
      bulk_g2s(ins, pay + a0, in_bytes, bar);
      if (acc_bulk) bulk_g2s(io, out + base, acc_bulk, bar);
    }
    if (fold)
      for (uint32_t k = acc_bulk / 4 + tid; k < live; k += kDecThreads) io[k] = o32[base + k];
    mbar_wait(bar, phase);
    phase ^= 1;
    const uint32_t head = static_cast<uint32_t>(off - a0);  // bytes
    if (raw) {
      __syncthreads();  // the hand-loaded accumulator words
      for (uint32_t k = tid; k < live; k += kDecThreads) {
        const uint32_t b = head + 4 * k;
        const uint32_t lo = ins[b >> 2];
        const uint32_t v = (b & 3) ? __funnelshift_r(lo, ins[(b >> 2) + 1], 8 * (b & 3)) : lo;
        io[k] = fold ? __float_as_uint(__fadd_rn(__uint_as_float(io[k]), __uint_as_float(v))) : v;
      }
    } else {
      if (warp == 0) {
        // lane l decodes values [128 l, 128 l + 128) as two independent
        // chains (64-value blocks 2l and 2l+1, from their indexed offsets)
        const uint32_t cw = e[1 + lane];
        const uint32_t bits_a = cw & 0xffffu, bits_b = cw >> 16;
        const uint32_t mybits = bits_a + bits_b;
        uint32_t incl = mybits;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += t;
        }
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        bool bad = (total + 7ull) / 8 != end - off;
        if (!bad) {
          const uint32_t i0 = lane * kLaneVals;
          const uint32_t na = live > i0 ? min(live - i0, 64u) : 0u;
          const uint32_t nb2 = live > i0 + 64 ? min(live - i0 - 64, 64u) : 0u;
          uint32_t bit_a = 8 * head + (incl - mybits), bit_b = bit_a + bits_a;  // within the staged bytes
          const uint32_t a0b = bit_a, b0b = bit_b;
          uint32_t pa = 0, pb = 0;
          uint32_t* row = sm + lane * kMsgLaneStride;
          auto code_at = [&](uint32_t bit, uint32_t& low) {
            const uint32_t w = bit >> 5, sh = bit & 31;
            const uint32_t x0 = ins[w], x1 = ins[w + 1], x2 = ins[w + 2];
            const uint32_t lo = __funnelshift_r(x0, x1, sh), hi = __funnelshift_r(x1, x2, sh);
            const uint32_t nb = 32 - (lo & 31u);
            const uint32_t v = __funnelshift_r(lo, hi, 5);  // the 32 bits after the length field
            low = nb >= 32 ? v : (v & ((1u << nb) - 1u));
            return 5 + nb;
          };
          for (uint32_t i = 0; i < 64; ++i) {
            if (i < na) {
              uint32_t low;
              bit_a += code_at(bit_a, low);
              pa ^= low;
              row[i] = pa;
            }
            if (i < nb2) {
              uint32_t low;
              bit_b += code_at(bit_b, low);
              pb ^= low;
              row[64 + i] = pb;
            }
          }
          bad = bit_a - a0b != bits_a || bit_b - b0b != bits_b;
          // chain b continues chain a; an exclusive XOR scan of the lanes'
          // totals gives each lane its carry
          const uint32_t tot = pa ^ pb;
          uint32_t x = tot;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, x, d);
            if (lane >= d) x ^= t;
          }
          carry[lane] = x ^ tot;
          carry[32 + lane] = pa;
        }
        const bool any_bad = __any_sync(kFull, bad);
        if (lane == 0) status[0] = any_bad ? 1u : 0u;
      }
      __syncthreads();
      if (status[0]) {
        if (tid == 0) atomicOr(err, kErrCorrupt);
        break;  // CTA-uniform
      }
      for (uint32_t k = tid; k < live; k += kDecThreads) {
        const uint32_t l = k >> 7;
        const uint32_t v = sm[l * kMsgLaneStride + (k & 127)] ^ carry[l] ^ ((k & 64) ? carry[32 + l] : 0u);
        io[k] = fold ? __float_as_uint(__fadd_rn(__uint_as_float(io[k]), __uint_as_float(v))) : v;
      }
    }
    // write the chunk: one bulk store of the aligned 16-byte multiple, the rest by hand
    const uint32_t st_bulk = out_al ? (4 * live) & ~15u : 0u;
    for (uint32_t k = st_bulk / 4 + tid; k < live; k += kDecThreads) o32[base + k] = io[k];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0 && st_bulk) {
      bulk_s2g(out + base, io, st_bulk);
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait_all();
}

int resident_grid(const void* k, int threads, size_t smem, uint64_t want) {
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
  const uint64_t cap = static_cast<uint64_t>(sms) * static_cast<uint64_t>(occ > 0 ? occ : 1);
  return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

std::atomic<uint64_t> g_enc_attr{0};

}  // namespace

hccx_status_t MsgScratch::ensure(uint64_t nchunks) {
  if (nchunks <= cap && total) return HCCX_OK;
  release();
  const uint64_t c = nchunks ? nchunks : 1;
  if (cudaMalloc(&desc, 8 * c) != cudaSuccess || cudaMalloc(&total, 3 * 8) != cudaSuccess ||
      cudaMemset(desc, 0, 8 * c) != cudaSuccess || cudaMemset(total, 0, 3 * 8) != cudaSuccess) {
    release();
    return HCCX_CUDA_FAIL;
  }
  cap = c;
  epoch = 0;
  return HCCX_OK;
}

void MsgScratch::release() {
  cudaFree(desc);
  cudaFree(total);
  desc = nullptr;
  total = nullptr;
  cap = 0;
}

hccx_status_t msg_encode_to(const float* in, uint64_t n, uint8_t* msg, uint8_t* pay, uint32_t* index,
                            MsgScratch& s, unsigned long long* acct, cudaStream_t st) {
  const uint64_t nch = msg_chunks(n);
  if (msg_max_bytes(n) >= (1ull << 32)) return HCCX_ERR_INVALID_ARGUMENT;  // u32 chunk offsets in the index
  hccx_status_t r = s.ensure(nch);
  if (r != HCCX_OK) return r;
  if (n == 0) {
    msg_header_kernel<<<1, 32, 0, st>>>(msg, s.total, acct);
    count_launch();
    return HCCX_STATUS(cudaGetLastError());
  }
  if (++s.epoch >= (1u << 24)) {  // descriptors carry 24 epoch bits: clear on wrap
    s.epoch = 1;
    if (cudaMemsetAsync(s.desc, 0, 8 * s.cap, st) != cudaSuccess) return HCCX_CUDA_FAIL;
  }
  const void* k = reinterpret_cast<const void*>(&ll_encode_kernel);
  smem_attr(k, kEncSmem, g_enc_attr);
  const int grid = resident_grid(k, kEncThreads, kEncSmem, nch);
  const int vec_ok = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  ll_encode_kernel<<<grid, kEncThreads, kEncSmem, st>>>(in, n, nch, vec_ok, pay, index, msg, msg_index_bytes(n),
                                                         s.desc, s.epoch, s.total,
                                                         reinterpret_cast<unsigned long long*>(s.total + 1), acct);
  count_launch();
  return HCCX_STATUS(cudaGetLastError());
}

hccx_status_t msg_encode(const float* in, uint64_t n, uint8_t* msg, MsgScratch& s, unsigned long long* acct,
                         cudaStream_t st) {
  const uint64_t ib = msg_index_bytes(n);
  return msg_encode_to(in, n, msg, msg + kMsgHeaderBytes + ib, reinterpret_cast<uint32_t*>(msg + kMsgHeaderBytes), s,
                       acct, st);
}

hccx_status_t msg_copy(const uint8_t* src, uint64_t n, uint8_t* const* dsts, int ndst, unsigned long long* acct,
                       cudaStream_t st) {
  if (ndst < 1) return HCCX_OK;
  if (ndst > kMsgMaxDsts) return HCCX_ERR_INVALID_ARGUMENT;
  MsgDsts D{};
  for (int k = 0; k < ndst; ++k) D.d[k] = dsts[k];
  D.nd = ndst;
  const uint64_t vec = msg_max_bytes(n) / 16;
  msg_copy_kernel<<<grid_for(vec, 256 * 4), 256, 0, st>>>(src, D, msg_index_bytes(n), acct);
  count_launch();
  return HCCX_STATUS(cudaGetLastError());
}

hccx_status_t msg_decode(const uint8_t* msg, uint64_t msg_cap, uint64_t n, float* out, bool fold, uint32_t* err,
                         unsigned long long* recv_acct, cudaStream_t st) {
  const uint64_t nch = msg_chunks(n);
  const void* k = reinterpret_cast<const void*>(&msg_decode_kernel);
  smem_attr(k, kMsgDecodeSmem, g_decode_attr);
  const int grid = resident_grid(k, kDecThreads, kMsgDecodeSmem, nch);
  msg_decode_kernel<<<grid, kDecThreads, kMsgDecodeSmem, st>>>(msg, msg_cap, n, nch, msg_index_bytes(n), out,
                                                               fold ? 1 : 0, err, recv_acct);
  count_launch();
  return HCCX_STATUS(cudaGetLastError());
}

}  // namespace hccx

namespace hccx {
namespace {
struct FrameState {
  MsgScratch scratch;
  uint32_t* err = nullptr;
  ~FrameState() {
    scratch.release();
    cudaFree(err);
  }
};
FrameState& frame_state() {
  thread_local FrameState s[16];
  int d = 0;
  cudaGetDevice(&d);
  return s[d & 15];
}
hccx_status_t frame_err(FrameState& f) {
  if (f.err) return HCCX_OK;
  if (cudaMalloc(&f.err, 4) != cudaSuccess || cudaMemset(f.err, 0, 4) != cudaSuccess) return HCCX_CUDA_FAIL;
  return HCCX_OK;
}
}  // namespace
}  // namespace hccx

extern "C" uint64_t hccx_lossless_frame_max_bytes(uint64_t n) { return msg_max_bytes(n); }

extern "C" hccx_status_t hccx_lossless_frame_encode(const float* d_in, uint64_t n, uint8_t* d_msg, uint64_t capacity,
                                                    void* stream) {
  HCCX_NVTX("hccx_lossless_frame_encode");
  if (!d_msg || (n && !d_in) || capacity < msg_max_bytes(n) || (reinterpret_cast<uintptr_t>(d_msg) & 15))
    return HCCX_ERR_INVALID_ARGUMENT;
  return msg_encode(d_in, n, d_msg, frame_state().scratch, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_lossless_frame_decode(const uint8_t* d_msg, uint64_t capacity, uint64_t n, float* d_out,
                                                    int fold, void* stream) {
  HCCX_NVTX("hccx_lossless_frame_decode");
  if (!d_msg || (n && !d_out) || (reinterpret_cast<uintptr_t>(d_msg) & 15)) return HCCX_ERR_INVALID_ARGUMENT;
  FrameState& f = frame_state();
  const hccx_status_t st = frame_err(f);
  if (st != HCCX_OK) return st;
  return msg_decode(d_msg, capacity, n, d_out, fold != 0, f.err, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_frame_status(void* stream) {
  FrameState& f = frame_state();
  const hccx_status_t st = frame_err(f);
  if (st != HCCX_OK) return st;
  return read_flag(f.err, static_cast<cudaStream_t>(stream));
}
