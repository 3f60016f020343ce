// lossless_msg.h -- framed LosslessPredictor messages for the NVLink
// communicator (lossless_comm.cu), encoded and decoded without host syncs.
//
// A message is
//
//   [0, 32)              frame: u64 container bytes, then the HCC1 container
//                        header (proj/src/codec.cpp:89-99: magic, kind,
//                        rate, original_len, chunk_count)
//   [32, 32 + I)         chunk index (this transport's, not the reference's):
//                        per 4096-value chunk 33 u32 words -- the chunk's byte
//                        offset in the payload, then 64 u16 block bit counts
//                        (bits coded for values [64 b, 64 b + 64)); I is a
//                        multiple of 16
//   [32 + I, ...)        the LosslessPredictor payload, byte-identical to
//                        hcc::compress (codec_kernels.hpp:165-239)
//
// The reference's payload stores no offsets, so a decoder of the bare
// payload must walk the 5-bit length fields serially (lossless.cu).  The
// index costs 132 B per 16 KiB of input (0.8%) and lets the receiver decode
// every chunk with a full warp (32 lanes x two independent 64-code chains)
// straight from the slot, folding into the accumulator on the way.  The encoder writes it for
// free: the emit kernel already computes every lane's bit count.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hccx.h"

namespace hccx {

constexpr uint64_t kMsgHeaderBytes = 32;
constexpr uint64_t kMsgIndexWords = 33;  // per chunk
constexpr uint64_t kMsgChunk = 4096;
constexpr int kMsgMaxDsts = 16;  // msg_copy destinations (the communicator's kMaxRanks)

inline uint64_t msg_chunks(uint64_t n) { return (n + kMsgChunk - 1) / kMsgChunk; }
inline uint64_t msg_index_bytes(uint64_t n) { return (4 * kMsgIndexWords * msg_chunks(n) + 15) / 16 * 16; }
// Largest message for n values, plus 16 bytes of read slack for the
// decoder's word window and the copy kernel's 16-byte vectors.
inline uint64_t msg_max_bytes(uint64_t n) {
  return kMsgHeaderBytes + msg_index_bytes(n) + (msg_chunks(n) + 7) / 8 + 4 * n + 16;
}

// Per-communicator encoder scratch, one per rank so members sharing a
// device never share it: the single-pass encoder's per-chunk look-back
// descriptors (tagged with a call epoch, so never cleared between calls),
// and 3 device words: the last payload size, the chunk ticket counter and
// its done counter (reset by the kernel's last warp).
struct MsgScratch {
  uint64_t* desc = nullptr;
  uint64_t* total = nullptr;
  uint64_t cap = 0;
  uint32_t epoch = 0;
  hccx_status_t ensure(uint64_t nchunks);
  void release();
};

// Encodes n values: payload at `pay`, chunk index at `index` (optional),
// frame at `msg` (optional).  The payload size lands in s.total.
hccx_status_t msg_encode_to(const float* in, uint64_t n, uint8_t* msg, uint8_t* pay, uint32_t* index,
                            MsgScratch& s, unsigned long long* acct, cudaStream_t st);

// Encodes n values into the message at `msg` (device memory, local or a
// peer's window; 16-byte aligned; msg_max_bytes(n) < 4 GiB).  `acct` (optional, device u64[2]) gains
// payload bytes and whole-message bytes.  Stream-ordered, no host sync.
hccx_status_t msg_encode(const float* in, uint64_t n, uint8_t* msg, MsgScratch& s, unsigned long long* acct,
                         cudaStream_t st);

// Copies the message at `src` (its size read on the device) to each of
// `dsts`; acct as above, counted once per destination.
hccx_status_t msg_copy(const uint8_t* src, uint64_t n, uint8_t* const* dsts, int ndst, unsigned long long* acct,
                       cudaStream_t st);

// Validates the frame (as hcc::from_bytes, codec.cpp:101-121) and the
// index against the payload, and decodes into `out` (fold: out = out +
// value, the ring's accumulation, collectives.cpp:50).  A bad message sets
// kErrCorrupt in `err` and leaves `out` unspecified.  `recv_acct`
// (optional) gains the payload bytes.
hccx_status_t msg_decode(const uint8_t* msg, uint64_t msg_cap, uint64_t n, float* out, bool fold, uint32_t* err,
                         unsigned long long* recv_acct, cudaStream_t st);

}  // namespace hccx
