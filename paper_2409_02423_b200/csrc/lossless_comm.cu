// lossless_comm.cu -- LosslessPredictor collectives over the NVLink
// communicator: the compressed bytes themselves go on the wire.
//
// The reference's MZHybrid scheme sends TP / PP / ZeRO traffic through the
// LosslessPredictor (proj/src/parallel3d.cpp:63-69): every ring hop carries
// compress(partial) (proj/src/collectives.cpp:44), whose size is data
// dependent.  Here each hop is a framed message in the receiver's slot
// (lossless_msg.h: frame + HCC1 header, a chunk index, the payload
// byte-identical to hcc::compress).  The sender encodes straight into the
// peer's slot (the emit kernel's stores cross NVLink; the frame's size is
// written by a kernel from the device-side scan) and publishes the slot's
// data flag with a system-scope fence + store; the receiver waits for the
// flag on the device, validates the frame like hcc::from_bytes
// (codec.cpp:101-121: magic, kind, lengths -> CorruptPayloadError) and
// decodes warp-per-chunk from the index, folding into its accumulator
// (acc = acc + dec, collectives.cpp:50), then acks the slot.  No stage
// waits on the host: sizes, errors and the byte accounting stay on the
// device until the collective's one synchronisation at the end (broadcast
// and p2p also read the message size once, to cut it into slot fragments).
// A single-process communicator enqueues every member's stage before any
// member's next stage.  Values are exact (the codec is lossless), so results
// equal the identity ring's bit for bit; the traced wire bytes are the
// payload bytes actually pushed.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "comm_internal.h"
#include "device_common.cuh"
#include "hccx.h"
#include "hccx_internal.h"
#include "lossless_msg.h"

namespace hccx {

namespace {

__global__ void ll_signal_kernel(uint32_t* flags, uint32_t count, uint32_t value) {
  if (threadIdx.x == 0) fence_acq_rel_sys();  // every prior write of this stream (payload, frame) before the flags
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) st_relaxed_sys(flags + i, value);
}

__global__ void ll_wait_kernel(const uint32_t* flags, uint32_t count, uint32_t epoch, uint32_t* err,
                               uint64_t timeout_ns) {
  for (uint32_t i = threadIdx.x; i < count; i += blockDim.x) {
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0;
    while (static_cast<int32_t>(ld_acquire_sys(flags + i) - epoch) < 0) {
      __nanosleep(64);
      if ((++spins & 255u) == 0) {
        if (ldg_u32_coherent(err) & kErrTimeout) return;
        if (globaltimer_ns() - t0 > timeout_ns) {
          atomicOr(err, kErrTimeout);
          return;
        }
      }
    }
  }
}

__global__ void ll_scale_kernel(float* x, uint64_t n, int div_mode, float recip, float divisor) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] = div_mode == 1 ? __fmul_rn(x[i], recip) : __fdiv_rn(x[i], divisor);
}

uint32_t* host_flag(const hccx_comm* c, int rank, int cls, int slot, uint32_t idx) {
  uint32_t* f = reinterpret_cast<uint32_t*>(c->peers[rank] + c->flag_off);
  const int p = c->p;
  if (cls < 3) {
    const int base[3] = {0, p - 1, 2 * p - 1};
    return f + static_cast<uint64_t>(base[cls] + slot) * c->max_seg + idx;
  }
  const int base[4] = {0, p - 1, 2 * p - 1, 3 * p - 1};
  return f + static_cast<uint64_t>(3 * p - 1) * c->max_seg + static_cast<uint64_t>(base[cls - 3] + slot) * kAckIdx +
         idx;
}

uint8_t* host_slot(const hccx_comm* c, int rank, int cls, int slot) {
  const uint64_t off = cls == 0 ? c->rs_off : (cls == 1 ? c->ag_off : c->pp_off);
  return c->peers[rank] + off + static_cast<uint64_t>(slot) * c->slot_bytes;
}

hccx_status_t ensure(float*& buf, uint64_t& cap, uint64_t n) {
  if (n <= cap && buf) return HCCX_OK;
  cudaFree(buf);
  buf = nullptr;
  cap = 0;
  if (cudaMalloc(&buf, 4 * (n ? n : 1)) != cudaSuccess) return HCCX_CUDA_FAIL;
  cap = n;
  return HCCX_OK;
}

hccx_status_t launched() { return HCCX_STATUS(cudaGetLastError()); }

// One framed message: encode `m` values into slot (cls, slot) of `dst`.
hccx_status_t send_frame(hccx_comm* c, const float* src, uint64_t m, int dst, int cls, int slot, cudaStream_t s) {
  return msg_encode(src, m, host_slot(c, dst, cls, slot), c->ll_msg, c->ll_acct, s);
}

// One thread per flag (up to kAckIdx = 1024): an ack or credit touches every
// index of a slot, and serial system-scope accesses would cost ~1 us each.
unsigned flag_threads(uint32_t count) { return count < 32 ? 32u : (count > 1024 ? 1024u : (count + 31) / 32 * 32); }

hccx_status_t signal(hccx_comm* c, int rank, int cls, int slot, uint32_t count, uint32_t value, cudaStream_t s) {
  ll_signal_kernel<<<1, flag_threads(count), 0, s>>>(host_flag(c, rank, cls, slot, 0), count, value);
  count_launch();
  return launched();
}

hccx_status_t wait(hccx_comm* c, int cls, int slot, uint32_t count, uint32_t epoch, cudaStream_t s) {
  ll_wait_kernel<<<1, flag_threads(count), 0, s>>>(host_flag(c, c->rank, cls, slot, 0), count, epoch, c->d_err,
                                                   comm_timeout_ns());
  count_launch();
  return launched();
}

// Receive side: wait for the slot's data flag, validate and decode the
// message into `out` (fold: out = out + value).
hccx_status_t recv_frame(hccx_comm* c, int cls, int slot, uint32_t epoch, uint64_t m, float* out, bool fold,
                         cudaStream_t s) {
  const hccx_status_t st = wait(c, cls, slot, 1, epoch, s);
  if (st != HCCX_OK) return st;
  return msg_decode(host_slot(c, c->rank, cls, slot), c->slot_bytes, m, out, fold, c->d_err, c->ll_acct + 2, s);
}

// Consumption ack of slot (cls, slot) in `rank`'s window: every index, so
// fused-kernel senders (which wait on their own CTA's index, or on all of
// them after a geometry change) see it too.
hccx_status_t ack(hccx_comm* c, int rank, int cls, int slot, uint32_t epoch, cudaStream_t s) {
  return signal(c, rank, cls, slot, kAckIdx, epoch, s);
}

hccx_status_t credit(hccx_comm* c, int cls, int slot, uint32_t need, cudaStream_t s) {
  return wait(c, cls, slot, kAckIdx, need, s);
}

}  // namespace

// ---------------------------------------------------------------------------
// Per-rank stage machine of one lossless collective.  Ops: 0 allreduce,
// 1 reduce-scatter, 2 allgather, 3 broadcast, 4 p2p.

struct LLRank {
  hccx_comm* c = nullptr;
  cudaStream_t s = nullptr;
  int op = 0, mode = 0, root = 0, dst = 0;
  uint64_t n = 0, chunk = 0;
  const float* in = nullptr;
  float* out = nullptr;
  float* work = nullptr;
  uint32_t epoch = 0, prev_rs = 0, prev_ag = 0;
  // broadcast / p2p: one message = the whole compressed container, carried
  // in slot-sized fragments (each fragment one pp epoch)
  bool pp_root = false, pp_recv = false;
  bool single = false;      // the whole message fits one slot: no staging, no host size read
  uint64_t msg_bytes = 0;   // frame + payload (root: after compress; receiver: after fragment 0)
  uint32_t nfrag = 0;
  uint32_t frag_send[kMaxRanks] = {};  // root: epoch of the current fragment per destination
  uint32_t frag_recv = 0;              // receiver: epoch of the current fragment
};

hccx_status_t ll_setup(LLRank& r, hccx_comm* c, int op, const float* in, float* out, uint64_t n, int mode, int root,
                       int dst, cudaStream_t s) {
  r = LLRank{};
  r.c = c;
  r.s = s;
  r.op = op;
  r.in = in;
  r.out = out;
  r.n = n;
  r.mode = mode;
  r.root = root;
  r.dst = dst;
  c->last_payload = c->last_frame = c->last_recv = 0;
  const int p = c->p;
  // the lossless geometry differs from every fused-kernel geometry: the next
  // fused use of these slots waits for every receiver CTA's ack
  const uint64_t lossless_key = 1ull << 62;
  if (op <= 2) {
    r.chunk = op == 2 ? n : n / p;
    r.epoch = ++c->epoch;
    if (op != 2) {
      r.prev_rs = c->last_rs;
      c->last_rs = r.epoch;
      c->geo_rs = lossless_key;
    }
    if (op != 1) {
      r.prev_ag = c->last_ag;
      c->last_ag = r.epoch;
      c->geo_ag = lossless_key;
    }
  } else {
    r.chunk = n;
    r.pp_root = c->rank == root;
    r.pp_recv = !r.pp_root && (op == 3 || c->rank == dst);
    r.single = msg_max_bytes(n) <= c->slot_bytes;
    if (r.pp_root)
      for (int d = 0; d < p; ++d)
        if (d != root && (op == 3 || d == dst)) c->geo_pp[d] = lossless_key;
  }
  DeviceGuard guard(c->device);
  if (op == 0 || op == 1) {  // the ring folds into a work copy of the input
    float* w = out;
    if (op == 1) {
      if (ensure(c->ll_work, c->ll_work_cap, n) != HCCX_OK) return HCCX_CUDA_FAIL;
      w = c->ll_work;
    }
    if (w != in && cudaMemcpyAsync(w, in, 4 * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return HCCX_CUDA_FAIL;
    r.work = w;
  }
  if (!c->ll_acct && cudaMalloc(&c->ll_acct, 4 * sizeof(unsigned long long)) != cudaSuccess) return HCCX_CUDA_FAIL;
  if (cudaMemsetAsync(c->ll_acct, 0, 4 * sizeof(unsigned long long), s) != cudaSuccess) return HCCX_CUDA_FAIL;
  if (op >= 3 && (r.pp_root || r.pp_recv)) {  // message staging (root) / reassembly (receiver)
    const uint64_t need = msg_max_bytes(n);
    if (need > c->ll_stage_cap) {
      cudaFree(c->ll_stage);
      c->ll_stage = nullptr;
      c->ll_stage_cap = 0;
      if (cudaMalloc(&c->ll_stage, need) != cudaSuccess) return HCCX_CUDA_FAIL;
      c->ll_stage_cap = need;
    }
  }
  return HCCX_OK;
}

// Reduce-scatter round t (collectives.cpp:34-52): send this rank's partial
// of chunk (j-1-t) to the right neighbour's rs[t].
hccx_status_t ll_rs_send(LLRank& r, int t) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  const int p = c->p, j = c->rank, right = (j + 1) % p;
  hccx_status_t st = credit(c, 3, t, r.prev_rs, r.s);
  if (st != HCCX_OK) return st;
  const int ch = ((j - 1 - t) % p + p) % p;
  st = send_frame(c, r.work + static_cast<uint64_t>(ch) * r.chunk, r.chunk, right, 0, t, r.s);
  if (st != HCCX_OK) return st;
  return signal(c, right, 0, t, 1, r.epoch, r.s);
}

// ... and its receive: acc(chunk j-2-t) = acc + dec(msg) in the decoder,
// then ack the left neighbour.
hccx_status_t ll_rs_recv(LLRank& r, int t) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  const int p = c->p, j = c->rank, left = (j + p - 1) % p;
  const int ch = ((j - 2 - t) % p + p) % p;
  hccx_status_t st = recv_frame(c, 0, t, r.epoch, r.chunk, r.work + static_cast<uint64_t>(ch) * r.chunk, true, r.s);
  if (st != HCCX_OK) return st;
  return ack(c, left, 3, t, r.epoch, r.s);
}

// Allgather (collectives.cpp:77-107): the owner encodes its shard once
// into its own (otherwise unused) ag[j] slot and one kernel copies the
// message into every peer's ag[j] slot -- each shard's payload crosses the
// wire p-1 times.
hccx_status_t ll_ag_send(LLRank& r) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  const int p = c->p, j = c->rank;
  const float* shard = r.op == 2 ? r.in : r.work + static_cast<uint64_t>(j) * r.chunk;
  for (int q = 1; q < p; ++q) {
    const hccx_status_t st = credit(c, 4, (j + q) % p, r.prev_ag, r.s);
    if (st != HCCX_OK) return st;
  }
  uint8_t* own = host_slot(c, j, 1, j);
  hccx_status_t st = msg_encode(shard, r.chunk, own, c->ll_msg, nullptr, r.s);  // local staging: not on the wire
  if (st != HCCX_OK) return st;
  uint8_t* dsts[kMaxRanks] = {};
  for (int q = 1; q < p; ++q) dsts[q - 1] = host_slot(c, (j + q) % p, 1, j);
  if ((st = msg_copy(own, r.chunk, dsts, p - 1, c->ll_acct, r.s)) != HCCX_OK) return st;
  for (int q = 1; q < p; ++q)
    if ((st = signal(c, (j + q) % p, 1, j, 1, r.epoch, r.s)) != HCCX_OK) return st;
  // the owner's own chunk: dec(comp(shard)) == shard
  float* mine = r.out + static_cast<uint64_t>(j) * r.chunk;
  if (mine != shard && cudaMemcpyAsync(mine, shard, 4 * r.chunk, cudaMemcpyDeviceToDevice, r.s) != cudaSuccess)
    return HCCX_CUDA_FAIL;
  return HCCX_OK;
}

hccx_status_t ll_ag_recv(LLRank& r) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  const int p = c->p, j = c->rank, left = (j + p - 1) % p;
  for (int q = 1; q < p; ++q) {
    const int i = (j - q + p) % p;
    hccx_status_t st = recv_frame(c, 1, i, r.epoch, r.chunk, r.out + static_cast<uint64_t>(i) * r.chunk, false, r.s);
    if (st != HCCX_OK) return st;
    // ack to the owner (direct-gather credit) and to the left neighbour
    // (ring-gather credit), like the fused kernel's gather receives
    if ((st = ack(c, i, 4, j, r.epoch, r.s)) != HCCX_OK) return st;
    if ((st = ack(c, left, 6, i, r.epoch, r.s)) != HCCX_OK) return st;
  }
  return HCCX_OK;
}

// Broadcast / p2p (no reference counterpart for broadcast, SURVEY.md §8
// a10; p2p: collectives.cpp:130-152).  The root compresses the whole
// message once into its staging buffer -- the reference's single
// container, so the bytes on the wire are exactly its payload -- and sends
// it in slot-sized fragments; every receiver reassembles, then decodes.
hccx_status_t ll_pp_prepare(LLRank& r) {
  hccx_comm* c = r.c;
  if (!r.pp_root || r.n == 0) return HCCX_OK;
  DeviceGuard guard(c->device);
  if (r.single) {  // one fragment; a broadcast encodes once and copies (size read on the device)
    r.nfrag = 1;
    return r.op == 3 ? msg_encode(r.in, r.n, c->ll_stage, c->ll_msg, nullptr, r.s) : HCCX_OK;
  }
  hccx_status_t st = msg_encode(r.in, r.n, c->ll_stage, c->ll_msg, nullptr, r.s);
  if (st != HCCX_OK) return st;
  uint64_t container = 0;  // the message size decides the fragment count
  if (cudaMemcpyAsync(&container, c->ll_stage, 8, cudaMemcpyDeviceToHost, r.s) != cudaSuccess ||
      cudaStreamSynchronize(r.s) != cudaSuccess)
    return HCCX_CUDA_FAIL;
  r.msg_bytes = kMsgHeaderBytes + msg_index_bytes(r.n) + container - 18;
  r.nfrag = static_cast<uint32_t>((r.msg_bytes + c->slot_bytes - 1) / c->slot_bytes);
  return HCCX_OK;
}

// Fragment f: returns HCCX_OK and sets *active when this rank had work.
hccx_status_t ll_pp_send_frag(LLRank& r, uint32_t f, bool* active) {
  hccx_comm* c = r.c;
  if (!r.pp_root || f >= r.nfrag) return HCCX_OK;
  *active = true;
  DeviceGuard guard(c->device);
  const int p = c->p, j = c->rank;
  if (r.single) {
    uint8_t* dsts[kMaxRanks] = {};
    int nd = 0;
    hccx_status_t st = HCCX_OK;
    for (int d = 0; d < p; ++d) {
      if (d == j || !(r.op == 3 || d == r.dst)) continue;
      r.frag_send[d] = ++c->send_ep[d];
      if ((st = credit(c, 5, d, r.frag_send[d] - 1, r.s)) != HCCX_OK) return st;
      dsts[nd++] = host_slot(c, d, 2, j);
    }
    st = r.op == 3 ? msg_copy(c->ll_stage, r.n, dsts, nd, c->ll_acct, r.s)
                   : msg_encode(r.in, r.n, dsts[0], c->ll_msg, c->ll_acct, r.s);  // straight into the peer's slot
    if (st != HCCX_OK) return st;
    for (int d = 0; d < p; ++d)
      if (d != j && (r.op == 3 || d == r.dst) && (st = signal(c, d, 2, j, 1, r.frag_send[d], r.s)) != HCCX_OK)
        return st;
    return HCCX_OK;
  }
  const uint64_t off = static_cast<uint64_t>(f) * c->slot_bytes;
  const uint64_t len = r.msg_bytes - off < c->slot_bytes ? r.msg_bytes - off : c->slot_bytes;
  for (int d = 0; d < p; ++d) {
    if (d == j || !(r.op == 3 || d == r.dst)) continue;
    r.frag_send[d] = ++c->send_ep[d];
    hccx_status_t st = credit(c, 5, d, r.frag_send[d] - 1, r.s);
    if (st != HCCX_OK) return st;
    if (cudaMemcpyAsync(host_slot(c, d, 2, j), c->ll_stage + off, len, cudaMemcpyDeviceToDevice, r.s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    if ((st = signal(c, d, 2, j, 1, r.frag_send[d], r.s)) != HCCX_OK) return st;
    c->last_frame += len;
    const uint64_t lead = kMsgHeaderBytes + msg_index_bytes(r.n);  // frame + index before the payload
    const uint64_t hdr_part = off < lead ? (lead - off < len ? lead - off : len) : 0;
    c->last_payload += len - hdr_part;
  }
  return HCCX_OK;
}

hccx_status_t ll_pp_recv_frag(LLRank& r, uint32_t f, bool* active) {
  hccx_comm* c = r.c;
  if (!r.pp_recv || r.n == 0 || (f > 0 && f >= r.nfrag)) return HCCX_OK;
  *active = true;
  DeviceGuard guard(c->device);
  r.frag_recv = ++c->recv_ep[r.root];
  hccx_status_t st = wait(c, 2, r.root, 1, r.frag_recv, r.s);
  if (st != HCCX_OK) return st;
  if (r.single) {  // decode straight from the slot, then free it
    r.nfrag = 1;
    st = msg_decode(host_slot(c, c->rank, 2, r.root), c->slot_bytes, r.n, r.out, false, c->d_err, c->ll_acct + 2, r.s);
    return st != HCCX_OK ? st : ack(c, r.root, 5, c->rank, r.frag_recv, r.s);
  }
  const uint64_t off = static_cast<uint64_t>(f) * c->slot_bytes;
  if (f == 0) {  // the frame: how many fragments follow (hcc::from_bytes checks)
    uint8_t h[26];
    uint32_t err = 0;
    if (cudaMemcpyAsync(h, host_slot(c, c->rank, 2, r.root), 26, cudaMemcpyDeviceToHost, r.s) != cudaSuccess ||
        cudaMemcpyAsync(&err, c->d_err, 4, cudaMemcpyDeviceToHost, r.s) != cudaSuccess ||
        cudaStreamSynchronize(r.s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    if (err & kErrTimeout) return HCCX_ERR_TIMEOUT;
    uint64_t container = 0, n = 0;
    uint32_t chunks = 0;
    for (int i = 0; i < 8; ++i) container |= static_cast<uint64_t>(h[i]) << (8 * i);
    for (int i = 0; i < 8; ++i) n |= static_cast<uint64_t>(h[14 + i]) << (8 * i);
    for (int i = 0; i < 4; ++i) chunks |= static_cast<uint32_t>(h[22 + i]) << (8 * i);
    r.msg_bytes = kMsgHeaderBytes + msg_index_bytes(r.n) + container - 18;
    if (container < 18 || r.msg_bytes + 16 > c->ll_stage_cap || std::memcmp(h + 8, "HCC1", 4) != 0 ||
        h[12] != HCCX_CODEC_LOSSLESS || n != r.n || chunks != msg_chunks(r.n))
      return HCCX_ERR_CORRUPT_PAYLOAD;
    r.nfrag = static_cast<uint32_t>((r.msg_bytes + c->slot_bytes - 1) / c->slot_bytes);
  }
  const uint64_t len = r.msg_bytes - off < c->slot_bytes ? r.msg_bytes - off : c->slot_bytes;
  if (cudaMemcpyAsync(c->ll_stage + off, host_slot(c, c->rank, 2, r.root), len, cudaMemcpyDeviceToDevice, r.s) !=
      cudaSuccess)
    return HCCX_CUDA_FAIL;
  return ack(c, r.root, 5, c->rank, r.frag_recv, r.s);
}

hccx_status_t ll_pp_complete(LLRank& r) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  if (r.pp_recv && r.n && !r.single)
    return msg_decode(c->ll_stage, c->ll_stage_cap, r.n, r.out, false, c->d_err, c->ll_acct + 2, r.s);
  if (r.pp_root && r.op == 3 && r.out && r.out != r.in && r.n &&
      cudaMemcpyAsync(r.out, r.in, 4 * r.n, cudaMemcpyDeviceToDevice, r.s) != cudaSuccess)
    return HCCX_CUDA_FAIL;
  return HCCX_OK;
}

hccx_status_t ll_finish(LLRank& r, const StepParams& div) {
  hccx_comm* c = r.c;
  DeviceGuard guard(c->device);
  if (r.op == 1) {  // reduce-scatter: this rank's reduced chunk
    if (cudaMemcpyAsync(r.out, r.work + static_cast<uint64_t>(c->rank) * r.chunk, 4 * r.chunk,
                        cudaMemcpyDeviceToDevice, r.s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
  }
  if (r.op == 0 && div.div_mode != 0) {  // Average: IEEE v / float(p) after the gather (collectives.cpp:234-239)
    ll_scale_kernel<<<148 * 4, 256, 0, r.s>>>(r.out, r.n, div.div_mode, div.recip, div.divisor);
    count_launch();
    return launched();
  }
  return HCCX_OK;
}

// The collective's one host synchronisation: device-side byte accounting
// and error flags (timeouts, corrupt messages) of every rank.
hccx_status_t ll_settle(std::vector<LLRank>& ranks, hccx_status_t st) {
  for (LLRank& r : ranks) {
    hccx_comm* c = r.c;
    if (!c || !c->ll_acct) continue;
    DeviceGuard guard(c->device);
    unsigned long long a[4] = {};
    if (cudaMemcpyAsync(a, c->ll_acct, sizeof a, cudaMemcpyDeviceToHost, r.s) != cudaSuccess) {
      if (st == HCCX_OK) st = HCCX_ERR_CUDA;
      continue;
    }
    const hccx_status_t fl = read_flag(c->d_err, r.s);  // synchronises the stream first
    c->last_payload += a[0];
    c->last_frame += a[1];
    c->last_recv += a[2];
    if (st == HCCX_OK) st = fl;
  }
  return st;
}

// Runs the stages of every rank in `ranks` in lockstep (one rank for a
// multi-process communicator, all members for a single-process one).
hccx_status_t ll_run(std::vector<LLRank>& ranks, const StepParams& div) {
  if (ranks.empty()) return HCCX_OK;
  const LLRank& r0 = ranks[0];
  const int p = r0.c->p;
  hccx_status_t st = HCCX_OK;
  // HCCX_LL_PROFILE: per-stage device time on the first rank's stream and
  // host enqueue time, printed to stderr (development aid)
  static const bool prof = std::getenv("HCCX_LL_PROFILE") != nullptr;
  std::vector<cudaEvent_t> evs;
  std::vector<std::chrono::steady_clock::time_point> hts;
  std::vector<const char*> names;
  const char* stage = "start";
  auto mark = [&](const char* name) {
    if (!prof) return;
    DeviceGuard guard(r0.c->device);
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, r0.s);
    evs.push_back(e);
    hts.push_back(std::chrono::steady_clock::now());
    names.push_back(name);
  };
  mark("start");
  auto all = [&](auto&& fn) {
    for (LLRank& r : ranks)
      if ((st = fn(r)) != HCCX_OK) return false;
    mark(stage);
    return true;
  };
  struct Report {
    std::vector<cudaEvent_t>& evs;
    std::vector<std::chrono::steady_clock::time_point>& hts;
    std::vector<const char*>& names;
    int dev;
    ~Report() {
      if (evs.empty()) return;
      DeviceGuard guard(dev);
      cudaEventSynchronize(evs.back());
      for (size_t i = 1; i < evs.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, evs[i - 1], evs[i]);
        std::fprintf(stderr, "hccx ll stage %-10s device %8.1f us  host %8.1f us\n", names[i], ms * 1e3,
                     std::chrono::duration<double, std::micro>(hts[i] - hts[i - 1]).count());
      }
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
    }
  } report{evs, hts, names, r0.c->device};
  if (r0.op == 0 || r0.op == 1) {
    for (int t = 0; t < p - 1; ++t) {
      stage = "rs_send";
      if (!all([&](LLRank& r) { return ll_rs_send(r, t); })) return st;
      stage = "rs_recv";
      if (!all([&](LLRank& r) { return ll_rs_recv(r, t); })) return st;
    }
  }
  if (r0.op == 0 || r0.op == 2) {
    stage = "ag_send";
    if (!all([&](LLRank& r) { return ll_ag_send(r); })) return st;
    stage = "ag_recv";
    if (!all([&](LLRank& r) { return ll_ag_recv(r); })) return st;
  }
  if (r0.op == 3 || r0.op == 4) {
    stage = "pp_prep";
    if (!all([&](LLRank& r) { return ll_pp_prepare(r); })) return st;
    for (uint32_t f = 0;; ++f) {  // every rank's fragment f before anyone's fragment f+1
      bool active = false;
      stage = "pp_send";
      if (!all([&](LLRank& r) { return ll_pp_send_frag(r, f, &active); })) return st;
      stage = "pp_recv";
      if (!all([&](LLRank& r) { return ll_pp_recv_frag(r, f, &active); })) return st;
      if (!active) break;
    }
    stage = "pp_done";
    if (!all([&](LLRank& r) { return ll_pp_complete(r); })) return st;
  }
  stage = "finish";
  all([&](LLRank& r) { return ll_finish(r, div); });
  return st;
}

}  // namespace hccx

namespace hccx {

// Entry for the communicators (comm.cu): one LosslessPredictor collective
// for the ranks `comms[0..nr)` (one rank: multi-process; all members: a
// single-process communicator).  op 0 allreduce, 1 reduce-scatter,
// 2 allgather (n = shard values), 3 broadcast, 4 p2p.  Synchronous: the
// codec's sizes are read on the host.
hccx_status_t ll_collective(hccx_comm* const* comms, int nr, int op, const float* const* in, float* const* out,
                            uint64_t n, int mode, int root, int dst, const cudaStream_t* streams) {
  if (nr < 1) return HCCX_OK;
  const int p = comms[0]->p;
  for (int k = 0; k < nr; ++k) {
    hccx_comm* c = comms[k];
    DeviceGuard guard(c->device);
    c->last_payload = c->last_frame = c->last_recv = 0;
  }
  StepParams div{};
  set_divisor(div, mode, p);
  if (op <= 2) {
    if (p == 1 || n == 0) {
      for (int k = 0; k < nr; ++k) {
        DeviceGuard guard(comms[k]->device);
        if (n && out[k] != in[k] &&
            cudaMemcpyAsync(out[k], in[k], 4 * n, cudaMemcpyDeviceToDevice, streams[k]) != cudaSuccess)
          return HCCX_CUDA_FAIL;
      }
      return HCCX_OK;
    }
    const uint64_t chunk = op == 2 ? n : n / p;
    if (chunk > comms[0]->chunk_cap) return HCCX_ERR_INVALID_ARGUMENT;
    std::vector<LLRank> ranks(nr);
    for (int k = 0; k < nr; ++k) {
      const hccx_status_t st = ll_setup(ranks[k], comms[k], op, in[k], out[k], n, mode, root, dst, streams[k]);
      if (st != HCCX_OK) return st;
    }
    return ll_settle(ranks, ll_run(ranks, div));
  }
  // broadcast / p2p: one message in fragments (ll_pp_*)
  std::vector<LLRank> ranks(nr);
  for (int k = 0; k < nr; ++k) {
    const hccx_status_t st = ll_setup(ranks[k], comms[k], op, in[k], out[k], n, mode, root, dst, streams[k]);
    if (st != HCCX_OK) return st;
  }
  return ll_settle(ranks, ll_run(ranks, div));
}

}  // namespace hccx
