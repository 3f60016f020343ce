/*
 * hccx.h -- C ABI of the B200-native compressed-collective engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (arxiv/paper_2409_02423, "hybridcomm", /root/reference/proj).  The
 * reference has no C ABI: its interface is the C++ header API quoted beside
 * each entry point below.  The C++ host mirror of that API (namespace hcc,
 * include/hcc/hcc_b200.hpp, paper_2409_02423_b200/host/) is a thin shim over these
 * functions, and INTEGRATION.md shows the ctypes/extern "C" bindings.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Pointers named d_* are device memory on
 *     the current (or stated) CUDA device; h_* are host memory.  Caller owns
 *     all memory.  Streams are cudaStream_t passed as void* (NULL = legacy
 *     default stream).
 *   - Every function returns an hccx_status_t.  Codes map 1:1 onto the
 *     reference's exception hierarchy (proj/include/hcc/errors.hpp:15-60);
 *     HCCX_ERR_CUDA / _INVALID_ARGUMENT / _TIMEOUT / _UNSUPPORTED are
 *     device-side additions.
 *   - Device entry points are asynchronous on the given stream.  Errors found
 *     by the kernels (NaN/Inf reaching a lossy codec, a peer timing out) are
 *     OR-ed into a device flag word; *_status() / hccx_flag_status() read it
 *     back (synchronising the stream) and map it to a status.
 *   - Results are bit-identical to the reference CPU path on the same inputs
 *     (fixed-rate and identity codecs; ring schedule of
 *     proj/src/collectives.cpp).  The zfp-rate codec (kind 3) is a new codec
 *     not present in the reference.
 */
#ifndef HCCX_H
#define HCCX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCCX_ABI_VERSION 1

#if defined(__GNUC__)
#define HCCX_API __attribute__((visibility("default")))
#else
#define HCCX_API
#endif

typedef enum hccx_status {
  HCCX_OK = 0,
  HCCX_ERR_NONFINITE = 1,            /* hcc::NonFiniteInputError    errors.hpp:15-19 */
  HCCX_ERR_CORRUPT_PAYLOAD = 2,      /* hcc::CorruptPayloadError    errors.hpp:21-25 */
  HCCX_ERR_DATA_DEPENDENT_SIZE = 3,  /* hcc::DataDependentSizeError errors.hpp:27-31 */
  HCCX_ERR_BAD_CHUNKING = 4,         /* hcc::BadChunkingError       errors.hpp:33-37 */
  HCCX_ERR_BAD_LAYOUT = 5,           /* hcc::BadLayoutError         errors.hpp:39-43 */
  HCCX_ERR_INVALID_SCHEME = 6,       /* hcc::InvalidSchemeError     errors.hpp:45-49 */
  HCCX_ERR_CONFIG = 7,               /* hcc::ConfigError            errors.hpp:51-60 */
  HCCX_ERR_CUDA = 8,
  HCCX_ERR_INVALID_ARGUMENT = 9,
  HCCX_ERR_TIMEOUT = 10,
  HCCX_ERR_UNSUPPORTED = 11
} hccx_status_t;

/* hcc::CodecKind (codec.hpp:16-20) plus the zfp-mode codec. */
typedef enum hccx_codec_kind {
  HCCX_CODEC_IDENTITY = 0,
  HCCX_CODEC_LOSSLESS = 1, /* LosslessPredictor: hccx_lossless_* (data-dependent size) */
  HCCX_CODEC_FIXED_RATE = 2,
  HCCX_CODEC_ZFP_RATE = 3 /* NOT in the reference: 1-D zfp fixed-rate, 4*rate bits/block */
} hccx_codec_kind_t;

/* hcc::CodecSpec (codec.hpp:22-32). */
typedef struct hccx_codec {
  int32_t kind;      /* hccx_codec_kind_t */
  int32_t rate_bits; /* fixed-rate: [2,32]; zfp-rate: [3,32]; else 0 */
} hccx_codec_t;

/* hcc::ReduceMode (collectives.hpp:21). */
typedef enum hccx_reduce_mode { HCCX_SUM = 0, HCCX_AVERAGE = 1 } hccx_reduce_mode_t;

HCCX_API const char* hccx_status_string(hccx_status_t s);
HCCX_API int hccx_abi_version(void);

/* Replaces CodecSpec::fixed_rate's range check (src/codec.cpp:11-17):
 * HCCX_ERR_INVALID_SCHEME when the rate is out of range. */
HCCX_API hccx_status_t hccx_codec_validate(hccx_codec_t codec);

/* Replaces hcc::wire_size_bytes (codec.hpp:63-67, src/codec.cpp:47-61):
 * payload bytes for n values; HCCX_ERR_DATA_DEPENDENT_SIZE for lossless. */
HCCX_API hccx_status_t hccx_wire_size_bytes(hccx_codec_t codec, uint64_t n, uint64_t* bytes);

/* CompressedBuffer::chunk_count (codec.hpp:47): 64-value blocks for
 * fixed-rate, 4-value blocks for zfp-rate, 0 for identity. */
HCCX_API hccx_status_t hccx_chunk_count(hccx_codec_t codec, uint64_t n, uint64_t* count);

/* ---------------------------------------------------------------- codec -- */

/* Device compress (replaces hcc::compress, codec.hpp:53-55 /
 * src/codec_omp.cpp:19-85, for identity / fixed-rate / zfp-rate).
 * d_out must hold hccx_wire_size_bytes() bytes.  d_err (nullable): device
 * word OR-ed with 1 when a live value is NaN/Inf (the reference throws
 * NonFiniteInputError, src/codec_omp.cpp:45); check with hccx_flag_status. */
HCCX_API hccx_status_t hccx_compress(hccx_codec_t codec, const float* d_in, uint64_t n, uint8_t* d_out,
                            uint32_t* d_err, void* stream);

/* Device decompress (replaces hcc::decompress, codec.hpp:57-61 /
 * src/codec_omp.cpp:87-111).  payload_bytes must equal the size law, else
 * HCCX_ERR_CORRUPT_PAYLOAD (src/codec_omp.cpp:94-96). */
HCCX_API hccx_status_t hccx_decompress(hccx_codec_t codec, const uint8_t* d_in, uint64_t payload_bytes,
                              uint64_t n, float* d_out, void* stream);

/* Synchronise `stream`, read the device flag word, clear it, and map it to a
 * status (HCCX_ERR_NONFINITE / HCCX_ERR_TIMEOUT / HCCX_OK). */
HCCX_API hccx_status_t hccx_flag_status(uint32_t* d_err, void* stream);

/* Host-buffer codec: the reference's value API (host vector in, host bytes
 * out) run on `device`, with the host<->device copies pipelined against the
 * kernels in slices.  Same results and errors as hcc::compress/decompress. */
HCCX_API hccx_status_t hccx_compress_host(hccx_codec_t codec, const float* h_in, uint64_t n, uint8_t* h_out,
                                 int device);
HCCX_API hccx_status_t hccx_decompress_host(hccx_codec_t codec, const uint8_t* h_in, uint64_t payload_bytes,
                                   uint64_t n, float* h_out, int device);

/* ------------------------------------------------- lossless predictor -- */
/* hcc::CodecKind::LosslessPredictor on the device (src/codec_kernels.hpp:
 * 165-239 chunk coder, src/codec_serial.cpp:48-66 / :85-107 buffer layout):
 * [ceil(nchunks/8) raw-fallback flag bytes][4096-value chunks].  The size is
 * data-dependent, so these calls synchronise `stream` to report it. */

/* Worst-case payload bytes for n values (every chunk raw): the capacity to
 * pass to hccx_lossless_compress. */
HCCX_API uint64_t hccx_lossless_max_bytes(uint64_t n);
/* Exact payload bytes hcc::compress(LosslessPredictor) would produce
 * (codec_kernels.hpp:203-215 per chunk + flag bytes).  Synchronises. */
HCCX_API hccx_status_t hccx_lossless_size(const float* d_in, uint64_t n, uint64_t* bytes, void* stream);
/* Device compress; *bytes = payload size.  capacity < size ->
 * HCCX_ERR_INVALID_ARGUMENT (nothing written).  Synchronises. */
HCCX_API hccx_status_t hccx_lossless_compress(const float* d_in, uint64_t n, uint8_t* d_out, uint64_t capacity,
                                              uint64_t* bytes, void* stream);
/* Device decompress of `bytes` payload bytes into n values.  A truncated or
 * over-long stream -> HCCX_ERR_CORRUPT_PAYLOAD (codec_serial.cpp:91-104).
 * Synchronises. */
HCCX_API hccx_status_t hccx_lossless_decompress(const uint8_t* d_in, uint64_t bytes, uint64_t n, float* d_out,
                                                void* stream);
/* Host-buffer variants run on `device`. */
HCCX_API hccx_status_t hccx_lossless_compress_host(const float* h_in, uint64_t n, uint8_t* h_out, uint64_t capacity,
                                                   uint64_t* bytes, int device);
HCCX_API hccx_status_t hccx_lossless_decompress_host(const uint8_t* h_in, uint64_t bytes, uint64_t n, float* h_out,
                                                     int device);

/* The communicator's framed LosslessPredictor message (one ring hop, one
 * p2p / broadcast message): [32 B frame: u64 container bytes + the HCC1
 * container header][chunk index: 33 u32 per 4096-value chunk -- byte offset,
 * 64 u16 bit counts of its 64-value blocks][payload byte-identical to
 * hccx_lossless_compress].
 * Neither call synchronises: sizes stay on the device.  frame_decode
 * validates the frame (as hcc::from_bytes) and the index against the
 * payload; a bad message -> HCCX_ERR_CORRUPT_PAYLOAD from hccx_frame_status.
 * fold != 0: d_out = d_out + value (the ring's accumulation).  The encoder's
 * scratch is per device and host thread: one thread's encodes on one device
 * must be stream-ordered (one stream, or events between streams). */
HCCX_API uint64_t hccx_lossless_frame_max_bytes(uint64_t n);
HCCX_API hccx_status_t hccx_lossless_frame_encode(const float* d_in, uint64_t n, uint8_t* d_msg, uint64_t capacity,
                                                  void* stream);
HCCX_API hccx_status_t hccx_lossless_frame_decode(const uint8_t* d_msg, uint64_t capacity, uint64_t n, float* d_out,
                                                  int fold, void* stream);
/* Synchronises `stream`; the first error of frame_decode calls since the
 * last status call (per device and host thread). */
HCCX_API hccx_status_t hccx_frame_status(void* stream);

/* Ring wire bytes (TraceEvent::wire_bytes * p) under LosslessPredictor,
 * which the size law cannot give: every hop's message is sized by the device
 * size pass.  collective: 0 reduce-scatter (d_in[j] = member j's n values;
 * the p(p-1) partial folds of collectives.cpp:34-61), 1 allgather (d_in[j] =
 * member j's n-value shard, each crossing p-1 hops, :94-106), 2 allreduce
 * (both).  Synchronises. */
HCCX_API hccx_status_t hccx_lossless_ring_wire(const float* const* d_in, int p, uint64_t n, int collective,
                                               uint64_t* wire, void* stream);
HCCX_API hccx_status_t hccx_lossless_ring_wire_host(const float* const* h_in, int p, uint64_t n, int collective,
                                                    uint64_t* wire, int device);
/* Per-message payload bytes of the same ring (the reference's cost model
 * charges each hop by its own message, collectives.cpp:53-62, :97-104):
 * collective 0: hop[t*p + j] = bytes member j sends in round t (t < p-1);
 * 1: hop[j] = bytes of shard j (compressed once, forwarded p-1 times);
 * 2: the RS layout, then hop[(p-1)*p + k] = bytes of member k's reduced
 * shard.  hop holds up to p*p entries.  Synchronises. */
HCCX_API hccx_status_t hccx_lossless_ring_hops(const float* const* d_in, int p, uint64_t n, int collective,
                                               uint64_t* hop, void* stream);
HCCX_API hccx_status_t hccx_lossless_ring_hops_host(const float* const* h_in, int p, uint64_t n, int collective,
                                                    uint64_t* hop, int device);

/* ------------------------------------------- single-device ring (group) -- */
/* All p members' buffers live on one device ("virtual ranks"): the value
 * semantics of the reference's all-members-in-one-call collectives
 * (collectives.hpp:23-25) executed by the same ring kernels.  p in [1,16]. */

typedef struct hccx_group* hccx_group_t;

HCCX_API hccx_status_t hccx_group_create(int p, int device, hccx_group_t* out);
HCCX_API hccx_status_t hccx_group_destroy(hccx_group_t g);

/* Replaces hcc::allreduce (collectives.hpp:61-64, src/collectives.cpp:202-248).
 * d_in[j], d_out[j]: member j's n values (d_out[j] may equal d_in[j]).
 * n % p != 0 -> HCCX_ERR_BAD_CHUNKING.  p == 1 copies the input untouched. */
HCCX_API hccx_status_t hccx_group_allreduce(hccx_group_t g, const float* const* d_in, float* const* d_out,
                                   uint64_t n, hccx_codec_t codec, int mode, void* stream);
/* Replaces hcc::ring_reduce_scatter (collectives.hpp:51-55, src/collectives.cpp:154-181).
 * d_shard[j] receives member j's n/p reduced values. */
HCCX_API hccx_status_t hccx_group_reduce_scatter(hccx_group_t g, const float* const* d_in, float* const* d_shard,
                                        uint64_t n, hccx_codec_t codec, void* stream);
/* Replaces hcc::ring_allgather (collectives.hpp:57-59, src/collectives.cpp:183-200).
 * d_out[j] receives p*shard_n values. */
HCCX_API hccx_status_t hccx_group_allgather(hccx_group_t g, const float* const* d_shard, float* const* d_out,
                                   uint64_t shard_n, hccx_codec_t codec, void* stream);
/* Broadcast (NOT in the reference): every member, root
 * included, receives dec(comp(d_in)). */
HCCX_API hccx_status_t hccx_group_broadcast(hccx_group_t g, int root, const float* d_in, float* const* d_out,
                                   uint64_t n, hccx_codec_t codec, void* stream);
/* Replaces hcc::p2p's value path (collectives.hpp:45-48, src/collectives.cpp:130-152):
 * d_out = dec(comp(d_in)). */
HCCX_API hccx_status_t hccx_group_p2p(hccx_group_t g, const float* d_in, float* d_out, uint64_t n,
                             hccx_codec_t codec, void* stream);
/* Host-buffer variants (the reference's value semantics: host vectors in,
 * host vectors out).  Members' buffers are copied to the group's device,
 * the same kernels run, results are copied back; *device_seconds (nullable)
 * receives the device time of the collective itself (CUDA events). */
HCCX_API hccx_status_t hccx_group_allreduce_host(hccx_group_t g, const float* const* h_in, float* const* h_out,
                                                 uint64_t n, hccx_codec_t codec, int mode, double* device_seconds);
HCCX_API hccx_status_t hccx_group_reduce_scatter_host(hccx_group_t g, const float* const* h_in,
                                                      float* const* h_shard, uint64_t n, hccx_codec_t codec,
                                                      double* device_seconds);
HCCX_API hccx_status_t hccx_group_allgather_host(hccx_group_t g, const float* const* h_shard, float* const* h_out,
                                                 uint64_t shard_n, hccx_codec_t codec, double* device_seconds);
HCCX_API hccx_status_t hccx_group_broadcast_host(hccx_group_t g, int root, const float* h_in, float* const* h_out,
                                                 uint64_t n, hccx_codec_t codec, double* device_seconds);
HCCX_API hccx_status_t hccx_group_p2p_host(hccx_group_t g, const float* h_in, float* h_out, uint64_t n,
                                           hccx_codec_t codec, double* device_seconds);

/* Synchronise and report the group's device error flag (see hccx_flag_status). */
HCCX_API hccx_status_t hccx_group_status(hccx_group_t g, void* stream);

/* ------------------------------------ multi-process NVLink communicator -- */
/* One process per GPU.  Each rank allocates a peer-visible window, exports
 * an opaque handle (HCCX_HANDLE_BYTES), the caller all-gathers the handles
 * (e.g. torch.distributed), and every rank connects.  Collectives are ONE
 * persistent kernel per call per rank: compressed chunks are pushed into the
 * next rank's window over NVLink with per-segment flags, and each hop is a
 * fused decompress-add-recompress (same bits as the single-device ring). */

#define HCCX_HANDLE_BYTES 256

typedef struct hccx_comm* hccx_comm_t;

/* max_n: largest per-rank buffer (values) any collective will use. */
HCCX_API hccx_status_t hccx_comm_create(int rank, int nranks, int device, uint64_t max_n, hccx_comm_t* out);
HCCX_API hccx_status_t hccx_comm_export(hccx_comm_t c, void* handle /* HCCX_HANDLE_BYTES */);
HCCX_API hccx_status_t hccx_comm_connect(hccx_comm_t c, const void* handles /* nranks*HCCX_HANDLE_BYTES */);
HCCX_API hccx_status_t hccx_comm_destroy(hccx_comm_t c);

/* Same semantics as the group calls, for this rank's buffer only. */
HCCX_API hccx_status_t hccx_allreduce(hccx_comm_t c, const float* d_in, float* d_out, uint64_t n,
                             hccx_codec_t codec, int mode, void* stream);
HCCX_API hccx_status_t hccx_reduce_scatter(hccx_comm_t c, const float* d_in, float* d_shard, uint64_t n,
                                  hccx_codec_t codec, void* stream);
HCCX_API hccx_status_t hccx_allgather(hccx_comm_t c, const float* d_shard, float* d_out, uint64_t shard_n,
                             hccx_codec_t codec, void* stream);
HCCX_API hccx_status_t hccx_broadcast(hccx_comm_t c, int root, const float* d_in, float* d_out, uint64_t n,
                             hccx_codec_t codec, void* stream);
/* Point-to-point: called by both src and dst (other ranks return at once).
 * src passes d_in, dst passes d_out = dec(comp(src's d_in)). */
HCCX_API hccx_status_t hccx_p2p(hccx_comm_t c, int src, int dst, const float* d_in, float* d_out, uint64_t n,
                       hccx_codec_t codec, void* stream);
/* Synchronise and report this rank's error flag (non-finite, peer timeout). */
HCCX_API hccx_status_t hccx_comm_status(hccx_comm_t c, void* stream);

/* Timeline of CTA 0 of the fused kernel (development / performance
 * analysis: ncu cannot replay a multi-rank kernel).  capacity in 64-bit
 * words: 0 disables, otherwise at least 17408 (the fixed slots: wait-chain
 * log at 4000, role accumulators at 4096, per-CTA times at 8192/16384), else
 * HCCX_ERR_INVALID_ARGUMENT.  Read returns [count, (tag, t_ns) x count]. */
HCCX_API hccx_status_t hccx_comm_trace_enable(hccx_comm_t c, uint64_t capacity);
HCCX_API hccx_status_t hccx_comm_trace_read(hccx_comm_t c, uint64_t* host, uint64_t max_words, uint64_t* words);

/* -------------------------------------- single-process communicator -- */
/* All p members of a communicator in ONE process: the shape of the
 * reference's all-members-in-one-call collectives (collectives.hpp:23-25;
 * SURVEY.md §8(b) "hccx_comm_create(ndev, devices)").  devices[j] is member
 * j's GPU (ring order = member order).  Members on distinct GPUs exchange
 * compressed segments over NVLink through peer access, with the same fused
 * kernel as the multi-process communicator; members sharing a GPU run as
 * virtual ranks of one cooperative launch (bit-identical, used for 1-GPU
 * testing of the NVLink kernel).  Device pointers d_*[j] live on devices[j];
 * streams[j] (nullable array) is member j's stream -- members sharing a GPU
 * run on the stream of the first such member.  p in [1,16].  Semantics and
 * errors as the group calls above. */

typedef struct hccx_mcomm* hccx_mcomm_t;

HCCX_API hccx_status_t hccx_mcomm_create(int nmembers, const int* devices, uint64_t max_n, hccx_mcomm_t* out);
HCCX_API hccx_status_t hccx_mcomm_destroy(hccx_mcomm_t m);
HCCX_API int hccx_mcomm_size(hccx_mcomm_t m);
/* Replaces hcc::allreduce (collectives.hpp:61-64, src/collectives.cpp:202-248). */
HCCX_API hccx_status_t hccx_mcomm_allreduce(hccx_mcomm_t m, const float* const* d_in, float* const* d_out,
                                            uint64_t n, hccx_codec_t codec, int mode, void* const* streams);
/* Replaces hcc::ring_reduce_scatter (collectives.hpp:51-55, src/collectives.cpp:154-181). */
HCCX_API hccx_status_t hccx_mcomm_reduce_scatter(hccx_mcomm_t m, const float* const* d_in, float* const* d_shard,
                                                 uint64_t n, hccx_codec_t codec, void* const* streams);
/* Replaces hcc::ring_allgather (collectives.hpp:57-59, src/collectives.cpp:183-200). */
HCCX_API hccx_status_t hccx_mcomm_allgather(hccx_mcomm_t m, const float* const* d_shard, float* const* d_out,
                                            uint64_t shard_n, hccx_codec_t codec, void* const* streams);
/* Broadcast (NOT in the reference); d_in on devices[root]. */
HCCX_API hccx_status_t hccx_mcomm_broadcast(hccx_mcomm_t m, int root, const float* d_in, float* const* d_out,
                                            uint64_t n, hccx_codec_t codec, void* const* streams);
/* Replaces hcc::p2p (collectives.hpp:45-48, src/collectives.cpp:130-152):
 * d_in on devices[src], d_out on devices[dst] = dec(comp(d_in)). */
HCCX_API hccx_status_t hccx_mcomm_p2p(hccx_mcomm_t m, int src, int dst, const float* d_in, float* d_out,
                                      uint64_t n, hccx_codec_t codec, void* const* streams);
/* Synchronise every member's stream and report the first error flag. */
HCCX_API hccx_status_t hccx_mcomm_status(hccx_mcomm_t m, void* const* streams);
/* Host-buffer variants (the reference's value semantics): device buffers are
 * cached in the communicator; *device_seconds (nullable) = device time of
 * the collective. */
HCCX_API hccx_status_t hccx_mcomm_allreduce_host(hccx_mcomm_t m, const float* const* h_in, float* const* h_out,
                                                 uint64_t n, hccx_codec_t codec, int mode, double* device_seconds);
HCCX_API hccx_status_t hccx_mcomm_reduce_scatter_host(hccx_mcomm_t m, const float* const* h_in,
                                                      float* const* h_shard, uint64_t n, hccx_codec_t codec,
                                                      double* device_seconds);
HCCX_API hccx_status_t hccx_mcomm_allgather_host(hccx_mcomm_t m, const float* const* h_shard, float* const* h_out,
                                                 uint64_t shard_n, hccx_codec_t codec, double* device_seconds);
HCCX_API hccx_status_t hccx_mcomm_broadcast_host(hccx_mcomm_t m, int root, const float* h_in, float* const* h_out,
                                                 uint64_t n, hccx_codec_t codec, double* device_seconds);
HCCX_API hccx_status_t hccx_mcomm_p2p_host(hccx_mcomm_t m, int src, int dst, const float* h_in, float* h_out,
                                           uint64_t n, hccx_codec_t codec, double* device_seconds);

/* Bytes this rank (member) pushed in its last collective: *payload = codec
 * payload bytes (the reference's wire accounting, collectives.cpp:113-126,
 * before the per-rank average), *frame = payload plus message framing.
 * Fixed-size codecs: the size law; LosslessPredictor: the framed,
 * data-dependent messages actually sent (HCC1 container header per message,
 * proj/src/codec.cpp:89-99). */
HCCX_API hccx_status_t hccx_comm_wire_bytes(hccx_comm_t c, uint64_t* payload, uint64_t* frame);
HCCX_API hccx_status_t hccx_mcomm_wire_bytes(hccx_mcomm_t m, int member, uint64_t* payload, uint64_t* frame);
/* Payload bytes of the framed (LosslessPredictor) messages this rank
 * received in its last collective (0 for fixed-size codecs). */
HCCX_API hccx_status_t hccx_comm_recv_bytes(hccx_comm_t c, uint64_t* payload);

/* CUDA devices visible to this process (0 when none). */
HCCX_API int hccx_device_count(void);

/* Kernel launches issued by this library since it was loaded. */
HCCX_API uint64_t hccx_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HCCX_H */
