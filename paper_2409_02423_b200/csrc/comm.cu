// comm.cu -- multi-process NVLink communicator (hccx_comm_*): window
// allocation, CUDA-IPC handle export/connect, epochs, and the launch of the
// fused ring kernel (ring_fused.cuh) for every collective.
//
// One process per GPU.  The caller exchanges the exported handles (e.g. with
// torch.distributed all_gather) and connects; after that every collective is
// a single cooperative kernel per rank, no host round trips.
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "codec_fixed_rate.cuh"
#include "codec_identity.cuh"
#include "codec_zfp.cuh"
#include "fused_launch.cuh"
#include "hccx.h"
#include "hccx_internal.h"
#include "comm_internal.h"

namespace hccx {

cudaError_t launch_fused_fr_lo(int rate, const FusedParams* p, int nv, cudaStream_t s);
cudaError_t launch_fused_fr_hi(int rate, const FusedParams* p, int nv, cudaStream_t s);
cudaError_t launch_fused_zfp_a(int rate, const FusedParams* p, int nv, cudaStream_t s);
cudaError_t launch_fused_zfp_b(int rate, const FusedParams* p, int nv, cudaStream_t s);

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

// One launch for the nv ranks p[0..nv) living on the current device.
static cudaError_t launch_fused(CodecSel c, const FusedParams* p, int nv, cudaStream_t s) {
  switch (c.kind) {
    case 0: return launch_fused_codec<IdentityCodec>(p, nv, s);
    case 2: return c.rate <= 16 ? launch_fused_fr_lo(c.rate, p, nv, s) : launch_fused_fr_hi(c.rate, p, nv, s);
    case 3: return c.rate <= 16 ? launch_fused_zfp_a(c.rate, p, nv, s) : launch_fused_zfp_b(c.rate, p, nv, s);
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
constexpr uint64_t kOneShotBytesPerRank = 8ull << 20;    // one-shot allreduce up to p x this many bytes

uint64_t timeout_ns() {
  const char* e = std::getenv("HCCX_TIMEOUT_MS");
  const uint64_t ms = e ? std::strtoull(e, nullptr, 10) : 20000;
  return (ms ? ms : 20000) * 1000000ull;
}

}  // namespace

namespace hccx {
uint64_t comm_timeout_ns() { return timeout_ns(); }
hccx_status_t ll_collective(hccx_comm* const* comms, int nr, int op, const float* const* in, float* const* out,
                            uint64_t n, int mode, int root, int dst, const cudaStream_t* streams);
}  // namespace hccx


extern "C" hccx_status_t hccx_comm_create(int rank, int nranks, int device, uint64_t max_n, hccx_comm_t* out) {
  HCCX_NVTX("hccx_comm_create");
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || max_n == 0)
    return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(device);
  hccx_comm* c = new hccx_comm();
  c->rank = rank;
  c->p = nranks;
  c->device = device;
  c->chunk_cap = align_up((max_n + nranks - 1) / nranks, kSegVals);
  // worst fixed-size codec (257 B / 64 values) or a framed LosslessPredictor
  // message (lossless_msg.h: frame + chunk index + 4 B per value + flag
  // bytes), whichever is larger
  c->slot_bytes = align_up(std::max((c->chunk_cap / 64) * 257 + kFrameBytes, msg_max_bytes(c->chunk_cap)), 256);
  c->max_seg = static_cast<uint32_t>(c->chunk_cap / kSegVals);
  const uint64_t nslots = 3ull * nranks - 1;  // data-flag slots; the acks use kAckIdx per slot
  c->rs_off = 0;
  c->ag_off = c->rs_off + (nranks - 1) * c->slot_bytes;
  c->pp_off = c->ag_off + nranks * c->slot_bytes;
  c->flag_off = c->pp_off + nranks * c->slot_bytes;
  // one-shot region (oneshot.cuh): p-1 raw fp32 slots + p gather slots + flags
  c->os_cap = c->chunk_cap < kOneShotMaxChunk ? c->chunk_cap : kOneShotMaxChunk;
  // flag mode: raw fp32 / payload bytes; pair mode (flag-in-data): 8 bytes
  // per raw value / payload word -- separate regions (oneshot.cuh)
  c->os_raw_bytes = align_up(4 * c->os_cap, 256);
  c->os_ag_bytes = align_up((c->os_cap + 63) / 64 * 257, 256);
  c->os_ll_raw_bytes = align_up(8 * c->os_cap, 256);
  c->os_ll_ag_bytes = align_up(2 * ((c->os_cap + 63) / 64 * 257 + 4), 256);
  // data flags: 3p-1 slots x max_seg; acks: 4p-1 slots x kAckIdx (ring_fused.cuh flag classes)
  c->os_off = c->flag_off + align_up((nslots * c->max_seg + (nslots + nranks) * kAckIdx) * 4, 256);
  c->os_ag_off = c->os_off + (nranks - 1) * c->os_raw_bytes;
  c->os_flag_off = c->os_ag_off + nranks * c->os_ag_bytes;
  c->os_ll_off = c->os_flag_off + align_up(2ull * nranks * kAckIdx * 4, 256);
  c->os_ll_ag_off = c->os_ll_off + (nranks - 1) * c->os_ll_raw_bytes;
  // everything from os_flag_off on is zeroed: flags, and pair epochs (epochs start at 1)
  c->win_bytes = c->os_ll_ag_off + nranks * c->os_ll_ag_bytes;
  if (cudaMalloc(&c->win, c->win_bytes) != cudaSuccess || cudaMalloc(&c->d_err, 4) != cudaSuccess) {
    cudaFree(c->win);
    delete c;
    return HCCX_CUDA_FAIL;
  }
  if (cudaMemset(c->win + c->flag_off, 0, c->os_off - c->flag_off) != cudaSuccess ||
      cudaMemset(c->win + c->os_flag_off, 0, c->win_bytes - c->os_flag_off) != cudaSuccess ||
      cudaMemset(c->d_err, 0, 4) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(c->win);
    cudaFree(c->d_err);
    delete c;
    return HCCX_CUDA_FAIL;
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
  if (cudaIpcGetMemHandle(&b.ipc, c->win) != cudaSuccess) return HCCX_CUDA_FAIL;
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
    if (cudaIpcOpenMemHandle(&ptr, b.ipc, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return HCCX_CUDA_FAIL;
    c->peers[r] = static_cast<uint8_t*>(ptr);
  }
  c->connected = true;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_comm_destroy(hccx_comm_t c) {
  if (!c) return HCCX_OK;
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  if (c->ipc)
    for (int r = 0; r < c->p; ++r)
      if (r != c->rank && c->peers[r]) cudaIpcCloseMemHandle(c->peers[r]);
  cudaFree(c->win);
  cudaFree(c->d_err);
  c->ll_msg.release();
  cudaFree(c->ll_acct);
  cudaFree(c->ll_work);
  cudaFree(c->ll_stage);
  cudaFree(c->d_trace);
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
  P.max_grid = c->max_grid;
  const char* dbg = std::getenv("HCCX_DEBUG");  // per call: A/B of development knobs in one process
  P.debug = dbg ? std::atoi(dbg) : 0;
  // development knobs, read per call (A/B in one process; every rank must agree)
  const char* ss = std::getenv("HCCX_STEP_SEGS");  // 0/unset: chosen per launch (fused_launch.cuh)
  P.step_segs = ss && std::atoi(ss) > 0 ? static_cast<uint32_t>(std::atoi(ss)) : 0u;
  const char* fs = std::getenv("HCCX_FIRST_SEGS");  // 0/unset: same as the step size
  P.first_segs = fs && std::atoi(fs) > 0 ? static_cast<uint32_t>(std::atoi(fs)) : 0u;
  // Allgather (and the allreduce's gather half) as a forwarding ring once a
  // chunk is large: the owner pushing to all p-1 peers at once makes that
  // phase NVLink-bound (measured p=4: ring wins at 64 MiB chunks, direct at
  // 16 MiB); HCCX_AG_RING_BYTES sets the chunk size threshold.
  // (read per call, like HCCX_ONESHOT_BYTES, so tests can steer one process
  // through both modes; every rank must see the same value)
  const char* ring_env = std::getenv("HCCX_AG_RING_BYTES");
  const uint64_t ring_from = ring_env ? std::strtoull(ring_env, nullptr, 10) : (32ull << 20);
  P.ag_ring = 4 * n_chunk >= ring_from ? 1 : 0;
  P.os_off = c->os_off;
  P.os_ag_off = c->os_ag_off;
  P.os_flag_off = c->os_flag_off;
  P.os_raw_bytes = c->os_raw_bytes;
  P.os_ag_bytes = c->os_ag_bytes;
  P.os_ll_off = c->os_ll_off;
  P.os_ll_ag_off = c->os_ll_ag_off;
  P.os_ll_raw_bytes = c->os_ll_raw_bytes;
  P.os_ll_ag_bytes = c->os_ll_ag_bytes;
  P.trace = c->d_trace;
  P.trace_cap = c->trace_cap;
  // chunk offsets are multiples of n_chunk floats: aligned iff n_chunk % 8 == 0
  P.vec_ok = (aligned32(in) && aligned32(out) && (n_chunk % 8 == 0)) ? 1 : 0;
  return P;
}

// Slot geometry key: the codec fixes the bytes per segment, the chunk size
// fixes the grid (hence which CTA reads which segment).
uint64_t geo_key(hccx_codec_t codec, uint64_t n_chunk) {
  return (static_cast<uint64_t>(codec.kind & 0xff) << 56) | (static_cast<uint64_t>(codec.rate_bits & 0xff) << 48) |
         (n_chunk & ((1ull << 48) - 1));
}

// Bit `cls` of P.credit_all when slot class `cls`'s geometry changed.
void note_geo(uint64_t& last, uint64_t key, int cls, FusedParams& P) {
  if (last != key) P.credit_all |= 1u << cls;
  last = key;
}

hccx_status_t check_comm(hccx_comm* c, hccx_codec_t codec) {
  if (!c || !c->connected) return HCCX_ERR_INVALID_ARGUMENT;
  return check_codec(codec);
}

// Allreduce algorithm choice: the two-round one-shot path up to
// HCCX_ONESHOT_BYTES (bytes per rank, default below; 0 disables it), the
// fused ring above.  Both give the reference's bits.
// 0: fused ring; 1: one-shot, flag mode; 2: one-shot, pair (LL) mode.
int use_oneshot(const hccx_comm* c, uint64_t n) {
  // defaults: one-shot up to 8 MiB per peer (the one-shot slots' capacity;
  // measured tools/nvl_small.py: at 32 MiB one-shot 96 us vs ring 103 us at
  // p = 4, 61 vs 62 us at p = 2 -- the ring's 2(p-1) dependent rounds cost
  // more than the raw bytes below that), pair mode up to 2 MiB per peer (p =
  // 4: pairs 28 us vs flags 29 us at 4 MiB, 79 vs 59 us at 16 MiB)
  const char* e = std::getenv("HCCX_ONESHOT_BYTES");
  const int64_t limit = e ? static_cast<int64_t>(std::strtoull(e, nullptr, 10)) : int64_t{-1};
  const uint64_t lim = limit >= 0 ? static_cast<uint64_t>(limit) : kOneShotBytesPerRank * c->p;
  if (!(4 * n <= lim && n / c->p <= c->os_cap)) return 0;
  const char* l = std::getenv("HCCX_LL_BYTES");
  const uint64_t ll = l ? std::strtoull(l, nullptr, 10) : (2ull << 20) * c->p;
  return 4 * n <= ll ? 2 : 1;
}

// One rank's share of a collective: a device-to-device copy (p == 1 and
// other degenerate cases) and/or a sequence of fused launches (one per
// pass).  Planning advances the communicator's epochs exactly as the
// collective will; every rank plans the same sequence.
struct RankWork {
  const void* copy_src = nullptr;
  void* copy_dst = nullptr;
  uint64_t copy_bytes = 0;
  std::vector<FusedParams> launches;
};

void plan_copy(RankWork& w, const void* src, void* dst, uint64_t bytes) {
  if (bytes && src != dst) {
    w.copy_src = src;
    w.copy_dst = dst;
    w.copy_bytes = bytes;
  }
}

hccx_status_t plan_allreduce(hccx_comm* c, const float* d_in, float* d_out, uint64_t n, hccx_codec_t codec,
                             int mode, RankWork& w) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  c->last_payload = c->last_frame = 0;
  if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (n / c->p > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  if (c->p == 1 || n == 0) {
    plan_copy(w, d_in, d_out, 4 * n);
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFAllReduce, n / c->p, d_in, d_out);
  P.epoch = ++c->epoch;
  if (const int os = use_oneshot(c, n)) {
    P.op = kFOneShotAllReduce;  // own slots and flags: the ring's slot epochs are untouched
    P.os_ll = os == 2 ? 1 : 0;
  } else {
    P.prev_rs = c->last_rs;
    P.prev_ag = c->last_ag;
    c->last_rs = c->last_ag = P.epoch;
    const uint64_t key = geo_key(codec, n / c->p);
    note_geo(c->geo_rs, key, 0, P);
    note_geo(c->geo_ag, key, 1, P);
  }
  {
    const uint64_t W = payload_bytes(sel_of(codec), n / c->p);
    c->last_payload = c->last_frame = P.op == kFOneShotAllReduce ? (P.os_ll ? 2 : 1) * (c->p - 1) * (4 * (n / c->p) + W)
                                                                  : 2ull * (c->p - 1) * W;
  }
  StepParams tmp{};
  set_divisor(tmp, mode, c->p);
  P.div_mode = tmp.div_mode;
  P.recip = tmp.recip;
  P.divisor = tmp.divisor;
  w.launches.push_back(P);
  return HCCX_OK;
}

hccx_status_t plan_reduce_scatter(hccx_comm* c, const float* d_in, float* d_shard, uint64_t n, hccx_codec_t codec,
                                  RankWork& w) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  c->last_payload = c->last_frame = 0;
  if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (n / c->p > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  if (c->p == 1 || n == 0) {
    plan_copy(w, d_in, d_shard, 4 * n);
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFReduceScatter, n / c->p, d_in, d_shard);
  P.vec_ok = P.vec_ok && aligned32(d_shard);
  P.epoch = ++c->epoch;
  P.prev_rs = c->last_rs;
  c->last_rs = P.epoch;
  note_geo(c->geo_rs, geo_key(codec, n / c->p), 0, P);
  c->last_payload = c->last_frame = (c->p - 1) * payload_bytes(sel_of(codec), n / c->p);
  w.launches.push_back(P);
  return HCCX_OK;
}

hccx_status_t plan_allgather(hccx_comm* c, const float* d_shard, float* d_out, uint64_t shard_n, hccx_codec_t codec,
                             RankWork& w) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  c->last_payload = c->last_frame = 0;
  if (shard_n > c->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
  if (c->p == 1 || shard_n == 0) {
    plan_copy(w, d_shard, d_out, 4 * shard_n);
    return HCCX_OK;
  }
  FusedParams P = base_params(c, kFAllGather, shard_n, d_shard, d_out);
  P.epoch = ++c->epoch;
  P.prev_ag = c->last_ag;
  c->last_ag = P.epoch;
  note_geo(c->geo_ag, geo_key(codec, shard_n), 1, P);
  c->last_payload = c->last_frame = (c->p - 1) * payload_bytes(sel_of(codec), shard_n);
  w.launches.push_back(P);
  return HCCX_OK;
}

// Broadcast / p2p messages larger than one slot go in passes of whole
// 256-value groups: the codec is blockwise from the buffer start, so the
// concatenated passes carry exactly the bits of one message.
void plan_pp_passes(hccx_comm* c, int op, int root, int dst, const float* d_in, float* d_out, uint64_t n,
                    hccx_codec_t codec, RankWork& w) {
  const uint64_t pass = c->chunk_cap;  // values (multiple of one segment)
  c->last_payload = c->last_frame = 0;
  for (uint64_t off = 0; off < n; off += pass) {
    const uint64_t m = (n - off) < pass ? (n - off) : pass;
    FusedParams P = base_params(c, op, m, d_in ? d_in + off : nullptr, d_out ? d_out + off : nullptr);
    P.root = root;
    P.dst = dst;
    if (c->rank == root) {
      const uint64_t key = geo_key(codec, m);
      for (int d = 0; d < c->p; ++d)
        if (d != root && (op == kFBroadcast || d == dst)) {
          P.pp_epoch[d] = ++c->send_ep[d];
          note_geo(c->geo_pp[d], key, 2, P);
          c->last_payload += payload_bytes(sel_of(codec), m);
          c->last_frame = c->last_payload;
        }
    } else {
      P.pp_epoch[root] = ++c->recv_ep[root];
    }
    w.launches.push_back(P);
  }
}

hccx_status_t plan_broadcast(hccx_comm* c, int root, const float* d_in, float* d_out, uint64_t n,
                             hccx_codec_t codec, RankWork& w) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  c->last_payload = c->last_frame = 0;
  if (root < 0 || root >= c->p) return HCCX_ERR_INVALID_ARGUMENT;
  if (n == 0) return HCCX_OK;
  if (c->p == 1) {
    plan_copy(w, d_in, d_out, 4 * n);
    return HCCX_OK;
  }
  plan_pp_passes(c, kFBroadcast, root, -1, c->rank == root ? d_in : nullptr, d_out, n, codec, w);
  return HCCX_OK;
}

hccx_status_t plan_p2p(hccx_comm* c, int src, int dst, const float* d_in, float* d_out, uint64_t n,
                       hccx_codec_t codec, RankWork& w) {
  hccx_status_t st = check_comm(c, codec);
  if (st != HCCX_OK) return st;
  c->last_payload = c->last_frame = 0;
  if (src < 0 || src >= c->p || dst < 0 || dst >= c->p || src == dst) return HCCX_ERR_INVALID_ARGUMENT;
  if (c->rank != src && c->rank != dst) return HCCX_OK;
  if (n == 0) return HCCX_OK;
  plan_pp_passes(c, kFP2P, src, dst, c->rank == src ? d_in : nullptr, c->rank == dst ? d_out : nullptr, n, codec,
                 w);
  return HCCX_OK;
}

// Run one rank's work on its own device and stream (multi-process comms).
hccx_status_t exec_rank(hccx_comm* c, hccx_codec_t codec, const RankWork& w, cudaStream_t s) {
  DeviceGuard guard(c->device);
  if (w.copy_bytes &&
      cudaMemcpyAsync(w.copy_dst, w.copy_src, w.copy_bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return HCCX_CUDA_FAIL;
  for (const FusedParams& P : w.launches)
    if (launch_fused(sel_of(codec), &P, 1, s) != cudaSuccess) return HCCX_CUDA_FAIL;
  return HCCX_STATUS(cudaGetLastError());
}

}  // namespace

extern "C" hccx_status_t hccx_allreduce(hccx_comm_t c, const float* d_in, float* d_out, uint64_t n,
                                        hccx_codec_t codec, int mode, void* stream) {
  HCCX_NVTX("hccx_allreduce");
  if (c && codec.kind == HCCX_CODEC_LOSSLESS) {
    if (!c->connected) return HCCX_ERR_INVALID_ARGUMENT;
    if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return ll_collective(&c, 1, 0, &d_in, &d_out, n, mode, 0, 0, &s);
  }
  RankWork w;
  hccx_status_t st = plan_allreduce(c, d_in, d_out, n, codec, mode, w);
  return st != HCCX_OK ? st : exec_rank(c, codec, w, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_reduce_scatter(hccx_comm_t c, const float* d_in, float* d_shard, uint64_t n,
                                             hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_reduce_scatter");
  if (c && codec.kind == HCCX_CODEC_LOSSLESS) {
    if (!c->connected) return HCCX_ERR_INVALID_ARGUMENT;
    if (n % static_cast<uint64_t>(c->p) != 0) return HCCX_ERR_BAD_CHUNKING;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return ll_collective(&c, 1, 1, &d_in, &d_shard, n, 0, 0, 0, &s);
  }
  RankWork w;
  hccx_status_t st = plan_reduce_scatter(c, d_in, d_shard, n, codec, w);
  return st != HCCX_OK ? st : exec_rank(c, codec, w, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_allgather(hccx_comm_t c, const float* d_shard, float* d_out, uint64_t shard_n,
                                        hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_allgather");
  if (c && codec.kind == HCCX_CODEC_LOSSLESS) {
    if (!c->connected) return HCCX_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return ll_collective(&c, 1, 2, &d_shard, &d_out, shard_n, 0, 0, 0, &s);
  }
  RankWork w;
  hccx_status_t st = plan_allgather(c, d_shard, d_out, shard_n, codec, w);
  return st != HCCX_OK ? st : exec_rank(c, codec, w, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_broadcast(hccx_comm_t c, int root, const float* d_in, float* d_out, uint64_t n,
                                        hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_broadcast");
  if (c && codec.kind == HCCX_CODEC_LOSSLESS) {
    if (!c->connected || root < 0 || root >= c->p) return HCCX_ERR_INVALID_ARGUMENT;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const float* src = c->rank == root ? d_in : nullptr;
    return ll_collective(&c, 1, 3, &src, &d_out, n, 0, root, -1, &s);
  }
  RankWork w;
  hccx_status_t st = plan_broadcast(c, root, d_in, d_out, n, codec, w);
  return st != HCCX_OK ? st : exec_rank(c, codec, w, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_p2p(hccx_comm_t c, int src, int dst, const float* d_in, float* d_out, uint64_t n,
                                  hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_p2p");
  if (c && codec.kind == HCCX_CODEC_LOSSLESS) {
    if (!c->connected || src < 0 || src >= c->p || dst < 0 || dst >= c->p || src == dst)
      return HCCX_ERR_INVALID_ARGUMENT;
    if (c->rank != src && c->rank != dst) return HCCX_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const float* in = c->rank == src ? d_in : nullptr;
    float* out = c->rank == dst ? d_out : nullptr;
    return ll_collective(&c, 1, 4, &in, &out, n, 0, src, dst, &s);
  }
  RankWork w;
  hccx_status_t st = plan_p2p(c, src, dst, d_in, d_out, n, codec, w);
  return st != HCCX_OK ? st : exec_rank(c, codec, w, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_comm_status(hccx_comm_t c, void* stream) {
  if (!c) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  return read_flag(c->d_err, static_cast<cudaStream_t>(stream));
}

extern "C" hccx_status_t hccx_comm_trace_enable(hccx_comm_t c, uint64_t capacity) {
  if (!c) return HCCX_ERR_INVALID_ARGUMENT;
  if (capacity != 0 && capacity < kTraceMinWords) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  cudaFree(c->d_trace);
  c->d_trace = nullptr;
  c->trace_cap = 0;
  if (capacity == 0) return HCCX_OK;
  if (cudaMalloc(&c->d_trace, capacity * 8) != cudaSuccess) return HCCX_CUDA_FAIL;
  c->trace_cap = capacity;
  return HCCX_STATUS(cudaMemset(c->d_trace, 0, capacity * 8));
}

extern "C" hccx_status_t hccx_comm_trace_read(hccx_comm_t c, uint64_t* host, uint64_t max_words, uint64_t* words) {
  if (!c || !host || !words) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(c->device);
  *words = 0;
  if (!c->d_trace) return HCCX_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return HCCX_CUDA_FAIL;
  const uint64_t n = max_words < c->trace_cap ? max_words : c->trace_cap;
  if (cudaMemcpy(host, c->d_trace, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return HCCX_CUDA_FAIL;
  *words = n;
  return HCCX_STATUS(cudaMemset(c->d_trace, 0, c->trace_cap * 8));
}

// ===================================================== single process ====
// hccx_mcomm: every member of the communicator in this process, on the
// devices the caller lists (SURVEY.md §8(b) hccx_comm_create(ndev, devices)).
// Members on distinct GPUs talk over NVLink through peer access (the same
// windows and kernel as the multi-process comm, mapped with
// cudaDeviceEnablePeerAccess instead of CUDA IPC); members sharing a GPU are
// virtual ranks of one cooperative launch (ring_fused_vkernel).  This is the
// shape of the reference's all-members-in-one-call API
// (proj/include/hcc/collectives.hpp:23-25).

struct hccx_mcomm {
  int p = 0;
  std::vector<int> devices;         // member -> device
  std::vector<hccx_comm*> members;  // one window per member
  std::vector<int> dev_list;        // distinct devices, first-use order
  // cached device buffers of the host-buffer entry points, per member
  std::vector<float*> hin, hout;
  uint64_t hcap = 0;
};

namespace {

hccx_status_t mcomm_exec(hccx_mcomm* m, hccx_codec_t codec, std::vector<RankWork>& work, void* const* streams) {
  auto stream_of = [&](int j) { return streams ? static_cast<cudaStream_t>(streams[j]) : cudaStream_t{}; };
  size_t passes = 0;
  for (int j = 0; j < m->p; ++j) {
    if (work[j].copy_bytes) {
      DeviceGuard guard(m->devices[j]);
      if (cudaMemcpyAsync(work[j].copy_dst, work[j].copy_src, work[j].copy_bytes, cudaMemcpyDeviceToDevice,
                          stream_of(j)) != cudaSuccess)
        return HCCX_CUDA_FAIL;
    }
    passes = work[j].launches.size() > passes ? work[j].launches.size() : passes;
  }
  // Pass by pass, one launch per device covering its members (every rank of
  // a pass must be resident at once: distinct devices run concurrently, the
  // virtual ranks of one device share a cooperative grid).
  for (size_t ps = 0; ps < passes; ++ps) {
    for (int dev : m->dev_list) {
      FusedParams P[kMaxRanks];
      int nv = 0, first = -1;
      for (int j = 0; j < m->p; ++j)
        if (m->devices[j] == dev && ps < work[j].launches.size()) {
          if (first < 0) first = j;
          P[nv++] = work[j].launches[ps];
        }
      if (!nv) continue;
      DeviceGuard guard(dev);
      if (launch_fused(sel_of(codec), P, nv, stream_of(first)) != cudaSuccess) return HCCX_CUDA_FAIL;
    }
  }
  return HCCX_STATUS(cudaGetLastError());
}

std::vector<cudaStream_t> mstreams(hccx_mcomm* m, void* const* streams) {
  std::vector<cudaStream_t> out(m->p, nullptr);
  if (streams)
    for (int j = 0; j < m->p; ++j) out[j] = static_cast<cudaStream_t>(streams[j]);
  return out;
}

hccx_status_t mcomm_check(hccx_mcomm* m, hccx_codec_t codec) {
  if (!m) return HCCX_ERR_INVALID_ARGUMENT;
  return check_codec(codec);
}

}  // namespace

extern "C" hccx_status_t hccx_mcomm_create(int nmembers, const int* devices, uint64_t max_n, hccx_mcomm_t* out) {
  HCCX_NVTX("hccx_mcomm_create");
  if (!out || !devices || nmembers < 1 || nmembers > kMaxRanks || max_n == 0) return HCCX_ERR_INVALID_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) return HCCX_CUDA_FAIL;
  for (int j = 0; j < nmembers; ++j)
    if (devices[j] < 0 || devices[j] >= ndev) return HCCX_ERR_INVALID_ARGUMENT;
  hccx_mcomm* m = new hccx_mcomm();
  m->p = nmembers;
  m->devices.assign(devices, devices + nmembers);
  for (int d : m->devices)
    if (std::find(m->dev_list.begin(), m->dev_list.end(), d) == m->dev_list.end()) m->dev_list.push_back(d);
  // peer access between every pair of distinct devices
  for (int a : m->dev_list)
    for (int b : m->dev_list) {
      if (a == b) continue;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, a, b) != cudaSuccess || !ok) {
        delete m;
        return HCCX_ERR_UNSUPPORTED;
      }
      DeviceGuard guard(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        delete m;
        return HCCX_CUDA_FAIL;
      }
    }
  // every rank uses the same CTAs per rank: the smallest share of a device
  uint32_t max_grid = kAckIdx;
  for (int dev : m->dev_list) {
    int sms = 0, nv = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int d : m->devices) nv += d == dev;
    const uint32_t g = static_cast<uint32_t>((sms > 0 ? sms : 148) / nv);
    max_grid = g < max_grid ? g : max_grid;
  }
  for (int j = 0; j < nmembers; ++j) {
    hccx_comm_t c = nullptr;
    const hccx_status_t st = hccx_comm_create(j, nmembers, devices[j], max_n, &c);
    if (st != HCCX_OK) {
      hccx_mcomm_destroy(m);
      return st;
    }
    c->ipc = false;
    c->max_grid = max_grid < 1 ? 1 : max_grid;
    m->members.push_back(c);
  }
  for (hccx_comm* c : m->members) {
    for (int r = 0; r < nmembers; ++r) c->peers[r] = m->members[r]->win;
    c->connected = true;
  }
  *out = m;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_mcomm_destroy(hccx_mcomm_t m) {
  if (!m) return HCCX_OK;
  for (size_t j = 0; j < m->members.size(); ++j) {
    DeviceGuard guard(m->devices[j]);
    if (j < m->hin.size()) cudaFree(m->hin[j]);
    if (j < m->hout.size()) cudaFree(m->hout[j]);
    hccx_comm_destroy(m->members[j]);
  }
  delete m;
  return HCCX_OK;
}

extern "C" int hccx_mcomm_size(hccx_mcomm_t m) { return m ? m->p : 0; }

extern "C" hccx_status_t hccx_mcomm_allreduce(hccx_mcomm_t m, const float* const* d_in, float* const* d_out,
                                              uint64_t n, hccx_codec_t codec, int mode, void* const* streams) {
  HCCX_NVTX("hccx_mcomm_allreduce");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(m->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (codec.kind == HCCX_CODEC_LOSSLESS)
    return ll_collective(m->members.data(), m->p, 0, d_in, d_out, n, mode, 0, 0, mstreams(m, streams).data());
  std::vector<RankWork> w(m->p);
  for (int j = 0; j < m->p; ++j)
    if ((st = plan_allreduce(m->members[j], d_in[j], d_out[j], n, codec, mode, w[j])) != HCCX_OK) return st;
  return mcomm_exec(m, codec, w, streams);
}

extern "C" hccx_status_t hccx_mcomm_reduce_scatter(hccx_mcomm_t m, const float* const* d_in, float* const* d_shard,
                                                   uint64_t n, hccx_codec_t codec, void* const* streams) {
  HCCX_NVTX("hccx_mcomm_reduce_scatter");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(m->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  if (codec.kind == HCCX_CODEC_LOSSLESS)
    return ll_collective(m->members.data(), m->p, 1, d_in, d_shard, n, 0, 0, 0, mstreams(m, streams).data());
  std::vector<RankWork> w(m->p);
  for (int j = 0; j < m->p; ++j)
    if ((st = plan_reduce_scatter(m->members[j], d_in[j], d_shard[j], n, codec, w[j])) != HCCX_OK) return st;
  return mcomm_exec(m, codec, w, streams);
}

extern "C" hccx_status_t hccx_mcomm_allgather(hccx_mcomm_t m, const float* const* d_shard, float* const* d_out,
                                              uint64_t shard_n, hccx_codec_t codec, void* const* streams) {
  HCCX_NVTX("hccx_mcomm_allgather");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (codec.kind == HCCX_CODEC_LOSSLESS)
    return ll_collective(m->members.data(), m->p, 2, d_shard, d_out, shard_n, 0, 0, 0, mstreams(m, streams).data());
  std::vector<RankWork> w(m->p);
  for (int j = 0; j < m->p; ++j)
    if ((st = plan_allgather(m->members[j], d_shard[j], d_out[j], shard_n, codec, w[j])) != HCCX_OK) return st;
  return mcomm_exec(m, codec, w, streams);
}

extern "C" hccx_status_t hccx_mcomm_broadcast(hccx_mcomm_t m, int root, const float* d_in, float* const* d_out,
                                              uint64_t n, hccx_codec_t codec, void* const* streams) {
  HCCX_NVTX("hccx_mcomm_broadcast");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (root < 0 || root >= m->p) return HCCX_ERR_INVALID_ARGUMENT;
  if (codec.kind == HCCX_CODEC_LOSSLESS) {
    std::vector<const float*> ins(m->p, nullptr);
    ins[root] = d_in;
    return ll_collective(m->members.data(), m->p, 3, ins.data(), d_out, n, 0, root, -1, mstreams(m, streams).data());
  }
  std::vector<RankWork> w(m->p);
  for (int j = 0; j < m->p; ++j)
    if ((st = plan_broadcast(m->members[j], root, j == root ? d_in : nullptr, d_out[j], n, codec, w[j])) != HCCX_OK)
      return st;
  return mcomm_exec(m, codec, w, streams);
}

extern "C" hccx_status_t hccx_mcomm_p2p(hccx_mcomm_t m, int src, int dst, const float* d_in, float* d_out,
                                        uint64_t n, hccx_codec_t codec, void* const* streams) {
  HCCX_NVTX("hccx_mcomm_p2p");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (src < 0 || src >= m->p || dst < 0 || dst >= m->p || src == dst) return HCCX_ERR_INVALID_ARGUMENT;
  if (codec.kind == HCCX_CODEC_LOSSLESS) {
    hccx_comm* two[2] = {m->members[src], m->members[dst]};
    const float* ins[2] = {d_in, nullptr};
    float* outs[2] = {nullptr, d_out};
    const auto all = mstreams(m, streams);
    const cudaStream_t ss[2] = {all[src], all[dst]};
    return ll_collective(two, 2, 4, ins, outs, n, 0, src, dst, ss);
  }
  std::vector<RankWork> w(m->p);
  for (int j : {src, dst})
    if ((st = plan_p2p(m->members[j], src, dst, d_in, d_out, n, codec, w[j])) != HCCX_OK) return st;
  return mcomm_exec(m, codec, w, streams);
}

extern "C" hccx_status_t hccx_mcomm_status(hccx_mcomm_t m, void* const* streams) {
  if (!m) return HCCX_ERR_INVALID_ARGUMENT;
  hccx_status_t first = HCCX_OK;
  for (int j = 0; j < m->p; ++j) {
    DeviceGuard guard(m->devices[j]);
    const hccx_status_t st =
        read_flag(m->members[j]->d_err, streams ? static_cast<cudaStream_t>(streams[j]) : cudaStream_t{});
    if (first == HCCX_OK) first = st;
  }
  return first;
}

// ------------------------------------------ host-buffer mcomm variants ----
// The reference's value API (host vectors in, host vectors out): member j's
// buffer is copied to its device (cached device buffers, grown on demand),
// the collective runs, results are copied back.  *device_seconds (nullable)
// receives the device time of the collective (events on member 0's device,
// all devices synchronised).

namespace {

hccx_status_t mcomm_bufs(hccx_mcomm* m, uint64_t in_n, uint64_t out_n) {
  const uint64_t need = in_n > out_n ? in_n : out_n;
  if (m->hin.size() == static_cast<size_t>(m->p) && m->hcap >= need) return HCCX_OK;
  for (int j = 0; j < m->p; ++j) {
    DeviceGuard guard(m->devices[j]);
    if (j < static_cast<int>(m->hin.size())) {
      cudaFree(m->hin[j]);
      cudaFree(m->hout[j]);
    }
  }
  m->hin.assign(m->p, nullptr);
  m->hout.assign(m->p, nullptr);
  m->hcap = 0;
  uint64_t cap = need < 1024 ? 1024 : need;
  for (int j = 0; j < m->p; ++j) {
    DeviceGuard guard(m->devices[j]);
    if (cudaMalloc(&m->hin[j], 4 * cap) != cudaSuccess || cudaMalloc(&m->hout[j], 4 * cap) != cudaSuccess)
      return HCCX_CUDA_FAIL;
  }
  m->hcap = cap;
  return HCCX_OK;
}

template <class F>
hccx_status_t mcomm_host_run(hccx_mcomm* m, const float* const* h_in, uint64_t in_n, int only_in,
                             float* const* h_out, uint64_t out_n, const std::vector<char>& out_mask, double* secs,
                             F&& body) {
  hccx_status_t st = mcomm_bufs(m, in_n, out_n);
  if (st != HCCX_OK) return st;
  for (int j = 0; j < m->p; ++j) {
    if (only_in >= 0 && j != only_in) continue;
    DeviceGuard guard(m->devices[j]);
    const float* src = only_in >= 0 ? h_in[0] : h_in[j];
    if (in_n && cudaMemcpy(m->hin[j], src, 4 * in_n, cudaMemcpyHostToDevice) != cudaSuccess) return HCCX_CUDA_FAIL;
  }
  for (int dev : m->dev_list) {
    DeviceGuard guard(dev);
    if (cudaDeviceSynchronize() != cudaSuccess) return HCCX_CUDA_FAIL;
  }
  cudaEvent_t a = nullptr, b = nullptr;
  {
    DeviceGuard guard(m->devices[0]);
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return HCCX_CUDA_FAIL;
    cudaEventRecord(a, nullptr);
  }
  st = body();
  float ms = 0.0f;
  {
    // every device's work is complete before member 0's end event
    for (int dev : m->dev_list) {
      DeviceGuard guard(dev);
      cudaDeviceSynchronize();
    }
    DeviceGuard guard(m->devices[0]);
    cudaEventRecord(b, nullptr);
    if (cudaEventSynchronize(b) == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  if (secs) *secs = ms * 1e-3;
  if (st == HCCX_OK) st = hccx_mcomm_status(m, nullptr);
  if (st != HCCX_OK) return st;
  for (int j = 0; j < m->p; ++j) {
    if (!out_mask[j] || !out_n) continue;
    DeviceGuard guard(m->devices[j]);
    if (cudaMemcpy(h_out[j], m->hout[j], 4 * out_n, cudaMemcpyDeviceToHost) != cudaSuccess) return HCCX_CUDA_FAIL;
  }
  return HCCX_OK;
}

}  // namespace

extern "C" hccx_status_t hccx_mcomm_allreduce_host(hccx_mcomm_t m, const float* const* h_in, float* const* h_out,
                                                   uint64_t n, hccx_codec_t codec, int mode, double* secs) {
  HCCX_NVTX("hccx_mcomm_allreduce_host");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(m->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  return mcomm_host_run(m, h_in, n, -1, h_out, n, std::vector<char>(m->p, 1), secs, [&] {
    return hccx_mcomm_allreduce(m, m->hin.data(), m->hout.data(), n, codec, mode, nullptr);
  });
}

extern "C" hccx_status_t hccx_mcomm_reduce_scatter_host(hccx_mcomm_t m, const float* const* h_in,
                                                        float* const* h_shard, uint64_t n, hccx_codec_t codec,
                                                        double* secs) {
  HCCX_NVTX("hccx_mcomm_reduce_scatter_host");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(m->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  return mcomm_host_run(m, h_in, n, -1, h_shard, m->p == 1 ? n : n / m->p, std::vector<char>(m->p, 1), secs, [&] {
    return hccx_mcomm_reduce_scatter(m, m->hin.data(), m->hout.data(), n, codec, nullptr);
  });
}

extern "C" hccx_status_t hccx_mcomm_allgather_host(hccx_mcomm_t m, const float* const* h_shard, float* const* h_out,
                                                   uint64_t shard_n, hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_mcomm_allgather_host");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  return mcomm_host_run(m, h_shard, shard_n, -1, h_out, shard_n * m->p, std::vector<char>(m->p, 1), secs, [&] {
    return hccx_mcomm_allgather(m, m->hin.data(), m->hout.data(), shard_n, codec, nullptr);
  });
}

extern "C" hccx_status_t hccx_mcomm_broadcast_host(hccx_mcomm_t m, int root, const float* h_in, float* const* h_out,
                                                   uint64_t n, hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_mcomm_broadcast_host");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (root < 0 || root >= m->p) return HCCX_ERR_INVALID_ARGUMENT;
  const float* const hin[1] = {h_in};
  return mcomm_host_run(m, hin, n, root, h_out, n, std::vector<char>(m->p, 1), secs, [&] {
    return hccx_mcomm_broadcast(m, root, m->hin[root], m->hout.data(), n, codec, nullptr);
  });
}

extern "C" hccx_status_t hccx_mcomm_p2p_host(hccx_mcomm_t m, int src, int dst, const float* h_in, float* h_out,
                                             uint64_t n, hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_mcomm_p2p_host");
  hccx_status_t st = mcomm_check(m, codec);
  if (st != HCCX_OK) return st;
  if (src < 0 || src >= m->p || dst < 0 || dst >= m->p || src == dst) return HCCX_ERR_INVALID_ARGUMENT;
  const float* const hin[1] = {h_in};
  std::vector<float*> outs(m->p, nullptr);
  outs[dst] = h_out;
  std::vector<char> mask(m->p, 0);
  mask[dst] = 1;
  return mcomm_host_run(m, hin, n, src, outs.data(), n, mask, secs, [&] {
    return hccx_mcomm_p2p(m, src, dst, m->hin[src], m->hout[dst], n, codec, nullptr);
  });
}

extern "C" hccx_status_t hccx_comm_wire_bytes(hccx_comm_t c, uint64_t* payload, uint64_t* frame) {
  if (!c || !payload || !frame) return HCCX_ERR_INVALID_ARGUMENT;
  *payload = c->last_payload;
  *frame = c->last_frame;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_mcomm_wire_bytes(hccx_mcomm_t m, int member, uint64_t* payload, uint64_t* frame) {
  if (!m || member < 0 || member >= m->p) return HCCX_ERR_INVALID_ARGUMENT;
  return hccx_comm_wire_bytes(m->members[member], payload, frame);
}

extern "C" hccx_status_t hccx_comm_recv_bytes(hccx_comm_t c, uint64_t* payload) {
  if (!c || !payload) return HCCX_ERR_INVALID_ARGUMENT;
  *payload = c->last_recv;
  return HCCX_OK;
}
