// comm.cu -- multi-process NVLink communicator (hccx_comm_*): window
// allocation, CUDA-IPC handle export/connect, epochs, and the launch of the
// fused ring kernel (ring_fused.cuh) for every collective.
//
// One process per GPU.  The caller exchanges the exported handles (e.g. with
// torch.distributed all_gather) and connects; after that every collective is
// a single cooperative kernel per rank, no host round trips.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "codec_fixed_rate.cuh"
#include "codec_identity.cuh"
#include "codec_zfp.cuh"
#include "fused_launch.cuh"
#include "hccx.h"
#include "hccx_internal.h"

namespace hccx {

cudaError_t launch_fused_fr_lo(int rate, const FusedParams& p, cudaStream_t s);
cudaError_t launch_fused_fr_hi(int rate, const FusedParams& p, cudaStream_t s);
cudaError_t launch_fused_zfp_a(int rate, const FusedParams& p, cudaStream_t s);
cudaError_t launch_fused_zfp_b(int rate, const FusedParams& p, cudaStream_t s);

int fused_capacity(const void* kernel, int threads, uint32_t smem) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = reinterpret_cast<uint64_t>(kernel) ^ (static_cast<uint64_t>(dev) << 56);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int b = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1) b = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int cap = b * (sms > 0 ? sms : 148);
  cache.emplace(key, cap);
  return cap;
}

static cudaError_t launch_fused(CodecSel c, const FusedParams& p, cudaStream_t s) {
  switch (c.kind) {
    case 0: return launch_fused_codec<IdentityCodec>(p, s);
    case 2: return c.rate <= 16 ? launch_fused_fr_lo(c.rate, p, s) : launch_fused_fr_hi(c.rate, p, s);
    case 3: return c.rate <= 16 ? launch_fused_zfp_a(c.rate, p, s) : launch_fused_zfp_b(c.rate, p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hccx

using namespace hccx;

namespace {

constexpr uint32_t kMagic = 0x48434358u;  // "HCCX"

struct HandleBlob {
  uint32_t magic;
  int32_t rank, nranks;
  uint32_t max_seg;
  uint64_t slot_bytes, win_bytes, chunk_cap;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(HandleBlob) <= HCCX_HANDLE_BYTES, "handle blob too large");

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

constexpr uint64_t kOneShotMaxChunk = 1ull << 21;         // values per chunk the one-shot slots hold
constexpr uint64_t kOneShotBytesPerRank = 4ull << 20;    // one-shot allreduce up to p x this many bytes

uint64_t timeout_ns() {
  const char* e = std::getenv("HCCX_TIMEOUT_MS");
  const uint64_t ms = e ? std::strtoull(e, nullptr, 10) : 20000;
  return (ms ? ms : 20000) * 1000000ull;
}

}  // namespace

struct hccx_comm {
  int rank = 0, p = 0, device = 0;
  uint64_t chunk_cap = 0;   // values per slot (multiple of one segment)
  uint64_t slot_bytes = 0;  // payload capacity per slot (worst codec: 257 B / 64 values)
  uint32_t max_seg = 0;
  uint64_t rs_off = 0, ag_off = 0, pp_off = 0, flag_off = 0, win_bytes = 0;
  uint64_t os_cap = 0;  // one-shot allreduce: values per chunk
  uint64_t os_off = 0, os_ag_off = 0, os_flag_off = 0, os_raw_bytes = 0, os_ag_bytes = 0;
  uint8_t* win = nullptr;
  uint8_t* peers[kMaxRanks] = {};
  bool connected = false;
  uint32_t* d_err = nullptr;
  uint32_t epoch = 0;                  // collectives
  uint32_t last_rs = 0, last_ag = 0;   // epoch of the last collective that used rs / ag slots
  uint32_t send_ep[kMaxRanks] = {};    // p2p / broadcast messages sent to rank d
  uint32_t recv_ep[kMaxRanks] = {};    // ... received from rank s
  uint64_t* d_trace = nullptr;         // optional CTA-0 timeline (hccx_comm_trace_enable)
  uint64_t trace_cap = 0;
};

extern "C" hccx_status_t hccx_comm_create(int rank, int nranks, int device, uint64_t max_n, hccx_comm_t* out) {
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || max_n == 0)
    return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(device);
  hccx_comm* c = new hccx_comm();
  c->rank = rank;
  c->p = nranks;
  c->device = device;
  c->chunk_cap = align_up((max_n + nranks - 1) / nranks, kSegVals);
  c->slot_bytes = align_up((c->chunk_cap / 64) * 257, 256);
  c->max_seg = static_cast<uint32_t>(c->chunk_cap / kSegVals);
  const uint64_t nslots = 3ull * nranks - 1;  // data-flag slots; the acks use kAckIdx per slot
  c->rs_off = 0;
  c->ag_off = c->rs_off + (nranks - 1) * c->slot_bytes;
  c->pp_off = c->ag_off + nranks * c->slot_bytes;
  c->flag_off = c->pp_off + nranks * c->slot_bytes;
  // one-shot region (oneshot.cuh): p-1 raw fp32 slots + p gather slots + flags
  c->os_cap = c->chunk_cap < kOneShotMaxChunk ? c->chunk_cap : kOneShotMaxChunk;
  c->os_raw_bytes = align_up(4 * c->os_cap, 256);
  c->os_ag_bytes = align_up((c->os_cap + 63) / 64 * 257, 256);
  // data flags: 3p-1 slots x max_seg; acks: 4p-1 slots x kAckIdx (ring_fused.cuh flag classes)
  c->os_off = c->flag_off + align_up((nslots * c->max_seg + (nslots + nranks) * kAckIdx) * 4, 256);
  c->os_ag_off = c->os_off + (nranks - 1) * c->os_raw_bytes;
  c->os_flag_off = c->os_ag_off + nranks * c->os_ag_bytes;
  c->win_bytes = c->os_flag_off + align_up(2ull * nranks * kAckIdx * 4, 256);
  if (cudaMalloc(&c->win, c->win_bytes) != cudaSuccess || cudaMalloc(&c->d_err, 4) != cudaSuccess) {
    cudaFree(c->win);
    delete c;
    return HCCX_ERR_CUDA;
  }
  if (cudaMemset(c->win + c->flag_off, 0, c->os_off - c->flag_off) != cudaSuccess ||
      cudaMemset(c->win + c->os_flag_off, 0, c->win_bytes - c->os_flag_off) != cudaSuccess ||
      cudaMemset(c->d_err, 0, 4) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(c->win);
    cudaFree(c->d_err);
    delete c;
    return HCCX_ERR_CUDA;
  }
  c->peers[rank] = c->win;
  *out = c;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_comm_export(hccx_comm_t c, void* handle) {
  if (!c || !handle) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  HandleBlob b{};
  b.magic = kMagic;
  b.rank = c->rank;
  b.nranks = c->p;
  b.max_seg = c->max_seg;
  b.slot_bytes = c->slot_bytes;
  b.win_bytes = c->win_bytes;
  b.chunk_cap = c->chunk_cap;
  if (cudaIpcGetMemHandle(&b.ipc, c->win) != cudaSuccess) return HCCX_ERR_CUDA;
  std::memset(handle, 0, HCCX_HANDLE_BYTES);
  std::memcpy(handle, &b, sizeof(b));
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_comm_connect(hccx_comm_t c, const void* handles) {
  if (!c || !handles) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  const uint8_t* h = static_cast<const uint8_t*>(handles);
  for (int r = 0; r < c->p; ++r) {
    HandleBlob b;
    std::memcpy(&b, h + static_cast<size_t>(r) * HCCX_HANDLE_BYTES, sizeof(b));
    if (b.magic != kMagic || b.rank != r || b.nranks != c->p || b.slot_bytes != c->slot_bytes ||
        b.win_bytes != c->win_bytes || b.max_seg != c->max_seg)
      return HCCX_ERR_INVALID_ARGUMENT;
    if (r == c->rank) continue;
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, b.ipc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HCCX_ERR_CUDA;
    c->peers[r] = static_cast<uint8_t*>(ptr);
  }
  c->connected = true;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_comm_destroy(hccx_comm_t c) {
  if (!c) return HCCX_OK;
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->p; ++r)
    if (r != c->rank && c->peers[r]) cudaIpcCloseMemHandle(c->peers[r]);
  cudaFree(c->win);
  cudaFree(c->d_err);
  delete c;
  return HCCX_OK;
}

namespace {

bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

FusedParams base_params(hccx_comm* c, int op, uint64_t n_chunk, const float* in, float* out) {
  FusedParams P{};
  for (int r = 0; r < c->p; ++r) P.win[r] = c->peers[r];
  P.rank = c->rank;
  P.p = c->p;
  P.op = op;
  P.n_chunk = n_chunk;
  P.slot_bytes = c->slot_bytes;
  P.rs_off = c->rs_off;
  P.ag_off = c->ag_off;
  P.pp_off = c->pp_off;
  P.flag_off = c->flag_off;
  P.max_seg = c->max_seg;
  P.in = in;
  P.out = out;
  P.err = c->d_err;
  P.timeout_ns = timeout_ns();
  static const int dbg = [] {
    const char* e = std::getenv("HCCX_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  P.debug = dbg;
  static const uint32_t step_segs = [] {
    const char* e = std::getenv("HCCX_STEP_SEGS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? static_cast<uint32_t>(v) : 0u;  // 0: chosen per launch (fused_launch.cuh)
  }();
  P.step_segs = step_segs;
  static const uint32_t first_segs = [] {
    const char* e = std::getenv("HCCX_FIRST_SEGS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? static_cast<uint32_t>(v) : 0u;  // 0: same as the step size
  }();
  P.first_segs = first_segs;
  // Allgather (and the allreduce's gather half) as a forwarding ring once a
  // chunk is large: the owner pushing to all p-1 peers at once makes that
  // phase NVLink-bound (measured p=4: ring wins at 64 MiB chunks, direct at
  // 16 MiB); HCCX_AG_RING_BYTES sets the chunk size threshold.
  static const uint64_t ring_from = [] {
    const char* e = std::getenv("HCCX_AG_RING_BYTES");
    return e ? std::strtoull(e, nullptr, 10) : (32ull << 20);
  }();
  P.ag_ring = 4 * n_chunk >= ring_from ? 1 : 0;
  P.os_off = c->os_off;
  P.os_ag_off = c->os_ag_off;
  P.os_flag_off = c->os_flag_off;
  P.os_raw_bytes = c->os_raw_bytes;
  P.os_ag_bytes = c->os_ag_bytes;
  P.trace = c->d_trace;
  P.trace_cap = c->trace_cap;
  // chunk offsets are multiples of n_chunk floats: aligned iff n_chunk % 8 == 0
  P.vec_ok = (aligned32(in) && aligned32(out) && (n_chunk % 8 == 0)) ? 1 : 0;
  return P;
}

hccx_status_t check_comm(hccx_comm* c, hccx_codec_t codec) {
  if (!c || !c->connected) return HCCX_ERR_INVALID_ARGUMENT;
  return check_codec(codec);
}

// Allreduce algorithm choice: the two-round one-shot path up to
// HCCX_ONESHOT_BYTES (bytes per rank, default below; 0 disables it), the
// fused ring above.  Both give the reference's bits.
bool use_oneshot(const hccx_comm* c, uint64_t n) {
  // default: 4 MiB per rank per peer count (16 MiB at p = 4, measured
  // crossover; the ring's 2(p-1) dependent rounds grow with p while the
  // one-shot path keeps two)
  static const int64_t limit = [] {
    const char* e = std::getenv("HCCX_ONESHOT_BYTES");
    return e ? static_cast<int64_t>(std::strtoull(e, nullptr, 10)) : int64_t{-1};
  }();
  const uint64_t lim = limit >= 0 ? static_cast<uint64_t>(limit) : kOneShotBytesPerRank * c->p;
  return 4 * n <= lim && n / c->p <= c->os_cap;
}

hccx_status_t run(hccx_comm* c, hccx_codec_t codec, const FusedParams& P, cudaStream_t s) {
  if (cudaSuccess != launch_fused(sel_of(codec), P, s)) return HCCX_ERR_CUDA;
  return cuda_status(cudaGetLastError());
}

}  // namespace

extern "C" hccx_status_t hccx_allreduce(hccx_comm_t c, const float* d_in, float* d_out, uint64_t n,
                                        hccx_codec_t codec, int mode, void* stream) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (n / c->p > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->p == 1 || n == 0) {
    if (n && d_out != d_in) return cuda_status(cudaMemcpyAsync(d_out, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFAllReduce, n / c->p, d_in, d_out);
  P.epoch = ++c->epoch;
  if (use_oneshot(c, n)) {
    P.op = kFOneShotAllReduce;  // own slots and flags: the ring's slot epochs are untouched
  } else {
    P.prev_rs = c->last_rs;
    P.prev_ag = c->last_ag;
    c->last_rs = c->last_ag = P.epoch;
  }
  StepParams tmp{};
  set_divisor(tmp, mode, c->p);
  P.div_mode = tmp.div_mode;
  P.recip = tmp.recip;
  P.divisor = tmp.divisor;
  return run(c, codec, P, s);
}

extern "C" hccx_status_t hccx_reduce_scatter(hccx_comm_t c, const float* d_in, float* d_shard, uint64_t n,
                                             hccx_codec_t codec, void* stream) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (n / c->p > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->p == 1 || n == 0) {
    if (n) return cuda_status(cudaMemcpyAsync(d_shard, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFReduceScatter, n / c->p, d_in, d_shard);
  P.vec_ok = P.vec_ok && aligned32(d_shard);
  P.epoch = ++c->epoch;
  P.prev_rs = c->last_rs;
  c->last_rs = P.epoch;
  return run(c, codec, P, s);
}

extern "C" hccx_status_t hccx_allgather(hccx_comm_t c, const float* d_shard, float* d_out, uint64_t shard_n,
                                        hccx_codec_t codec, void* stream) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  if (shard_n > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->p == 1 || shard_n == 0) {
    if (shard_n) return cuda_status(cudaMemcpyAsync(d_out, d_shard, 4 * shard_n, cudaMemcpyDeviceToDevice, s));
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFAllGather, shard_n, d_shard, d_out);
  P.epoch = ++c->epoch;
  P.prev_ag = c->last_ag;
  c->last_ag = P.epoch;
  return run(c, codec, P, s);
}

// Broadcast / p2p messages larger than one slot go in passes of whole
// 256-value groups: the codec is blockwise from the buffer start, so the
// concatenated passes carry exactly the bits of one message.
static hccx_status_t pp_passes(hccx_comm* c, int op, int root, int dst, const float* d_in, float* d_out,
                               uint64_t n, hccx_codec_t codec, cudaStream_t s) {
  const uint64_t pass = c->chunk_cap;  // values (multiple of 2048)
  for (uint64_t off = 0; off < n; off += pass) {
    const uint64_t m = (n - off) < pass ? (n - off) : pass;
    FusedParams P = base_params(c, op, m, d_in ? d_in + off : nullptr, d_out ? d_out + off : nullptr);
    P.root = root;
    P.dst = dst;
    if (c->rank == root) {
      for (int d = 0; d < c->p; ++d)
        if (d != root && (op == kFBroadcast || d == dst)) P.pp_epoch[d] = ++c->send_ep[d];
    } else {
      P.pp_epoch[root] = ++c->recv_ep[root];
    }
    hccx_status_t st = run(c, codec, P, s);
    if (st != HCCX_OK) return st;
  }
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_broadcast(hccx_comm_t c, int root, const float* d_in, float* d_out, uint64_t n,
                                        hccx_codec_t codec, void* stream) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  if (root < 0 || root >= c->p) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return HCCX_OK;
  if (c->p == 1) {
    if (d_out != d_in) return cuda_status(cudaMemcpyAsync(d_out, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
    return HCCX_OK;
  }
  return pp_passes(c, kFBroadcast, root, -1, c->rank == root ? d_in : nullptr, d_out, n, codec, s);
}

extern "C" hccx_status_t hccx_p2p(hccx_comm_t c, int src, int dst, const float* d_in, float* d_out, uint64_t n,
                                  hccx_codec_t codec, void* stream) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  if (src < 0 || src >= c->p || dst < 0 || dst >= c->p || src == dst) return HCCX_ERR_INVALID_ARGUMENT;
  if (c->rank != src && c->rank != dst) return HCCX_OK;
  DeviceGuard guard(c->device);
  if (n == 0) return HCCX_OK;
  return pp_passes(c, kFP2P, src, dst, c->rank == src ? d_in : nullptr, c->rank == dst ? d_out : nullptr, n, codec,
                   static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_comm_status(hccx_comm_t c, void* stream) {
  if (!c) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  return read_flag(c->d_err, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_comm_trace_enable(hccx_comm_t c, uint64_t capacity) {
  if (!c) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaFree(c->d_trace);
  c->d_trace = nullptr;
  c->trace_cap = 0;
  if (capacity == 0) return HCCX_OK;
  if (cudaMalloc(&c->d_trace, capacity * 8) != cudaSuccess) return HCCX_ERR_CUDA;
  c->trace_cap = capacity;
  return cuda_status(cudaMemset(c->d_trace, 0, capacity * 8));
}

extern "C" hccx_status_t hccx_comm_trace_read(hccx_comm_t c, uint64_t* host, uint64_t max_words, uint64_t* words) {
  if (!c || !host || !words) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  *words = 0;
  if (!c->d_trace) return HCCX_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return HCCX_ERR_CUDA;
  const uint64_t n = max_words < c->trace_cap ? max_words : c->trace_cap;
  if (cudaMemcpy(host, c->d_trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return HCCX_ERR_CUDA;
  *words = n;
  return cuda_status(cudaMemset(c->d_trace, 0, c->trace_cap * 8));
}
