// ring_fused.cuh -- the NVLink engine: ONE persistent kernel per collective
// per rank, moving only compressed chunks between GPUs.
//
// Every rank owns a window (cudaMalloc'd; mapped by every peer over
// NVLink/NVSwitch through CUDA IPC, or through peer access in a
// single-process communicator) holding inbox slots and per-step flags:
//   rs[t]   t = 0..p-2   message of ring round t from the left neighbour
//   ag[i]   i = 0..p-1   compressed final shard C_i of rank i (allgather)
//   pp[i]   i = 0..p-1   point-to-point / broadcast message from rank i
// A "segment" is kSegGroups = 24 warp groups (6,144 values) of a chunk, one
// group per compute warp; CTA b of the cooperative grid (G CTAs per rank,
// one per SM) owns segments b, b+G, b+2G, ... in every phase, so rank j's
// CTA b only ever waits on CTA b of its peers: a per-segment wavefront
// pipeline with no grid-wide barrier.  The virtual-rank kernel runs several
// ranks' CTA sets in one cooperative grid on one GPU (same device code).
//
// Ring schedule (identical bits to proj/src/collectives.cpp:27-111):
//   phase 0     encode local chunk (j-1) mod p -> push to rs[0] of rank j+1
//   phase t     wait rs[t-1]; fused decompress-add-recompress with local
//               chunk (j-1-t) mod p -> push to rs[t] of rank j+1
//   final       wait rs[p-2]; add local chunk j ->
//                 allreduce: encode C_j, push it into ag[j] (right neighbour
//                            for the forwarding ring, every peer for the
//                            direct gather), write dec(C_j) (/p) to out chunk j
//                 reduce-scatter: write the fp32 sum to the shard
//   gather      wait ag[i], decode (/p) to out chunk i, forward the payload
//               bytes unchanged (ring mode)
// Roles per CTA: 24 compute warps; a producer warp (waits for the step's
// inbound flag, streams inbox payload + local fp32 into a shared-memory
// stage ring with cp.async.bulk); a pusher warp (hands each encoded segment
// to the TMA engine as one cp.async.bulk store per destination window and
// recycles the tile once read); a signaller warp (after the step's bulk
// writes complete: one fence.acq_rel.sys per batch of ready events, then
// relaxed system-scope flag / ack stores).  Waits are bounded
// (%globaltimer); a timeout raises kErrTimeout instead of hanging the GPU.
#pragma once
#include "step_kernel.cuh"

namespace hccx {

constexpr int kMaxRanks = 16;

// Role timing accumulators, per-warp progress words (timeout wait chains)
// and their clock reads cost ~10% of the kernel's issue slots: compiled in
// only for analysis builds (make EXTRA=-DHCCX_FUSED_PROFILE=1 OUT=...;
// tools/nvl_trace.py reads them).  CTA-0 event timelines stay runtime-gated.
#ifndef HCCX_FUSED_PROFILE
#define HCCX_FUSED_PROFILE 0
#endif
__device__ __forceinline__ uint64_t prof_clock() {
  if constexpr (HCCX_FUSED_PROFILE) return clock64();
  return 0;
}
#define HCCX_PROG(stmt)                    \
  do {                                     \
    if constexpr (HCCX_FUSED_PROFILE) {    \
      stmt;                                \
    }                                      \
  } while (0)
// Compute warps per CTA of the fused kernel.  One CTA per SM with 24
// compute warps working through the same segments: with three 8-warp CTAs
// per SM the warp scheduler's age priority starved the SM's third CTA, which
// then finished ~30 us after the others while running alone latency-bound.
#ifndef HCCX_FUSED_COMPUTE
#define HCCX_FUSED_COMPUTE 24
#endif
constexpr int kFusedWarps = HCCX_FUSED_COMPUTE;
constexpr int kFCtasPerSm = 24 / kFusedWarps;
constexpr int kSegGroups = kFusedWarps;  // groups per segment (one per compute warp)
constexpr uint32_t kSegVals = kSegGroups * kGroupVals;

enum FusedOp : int {
  kFAllReduce = 0,
  kFReduceScatter = 1,
  kFAllGather = 2,
  kFBroadcast = 3,
  kFP2P = 4,
  kFOneShotAllReduce = 5  // small-message allreduce (oneshot.cuh)
};

struct FusedParams {
  uint8_t* win[kMaxRanks];  // every rank's window (own included), mapped in this process
  int rank, p, op;
  int root, dst;            // broadcast root / p2p (src = root, dst)
  uint64_t n_chunk;         // values per chunk (allreduce/RS: n/p; AG: shard; bcast/p2p: message)
  uint64_t slot_bytes;      // slot stride in the window
  uint64_t rs_off, ag_off, pp_off, flag_off;
  uint32_t max_seg;         // flags per slot
  const float* in;
  float* out;
  uint32_t epoch;           // collective epoch (allreduce / reduce-scatter / allgather)
  uint32_t prev_rs, prev_ag;  // epoch of the previous use of the rs / ag slots (ack to wait for)
  uint32_t pp_epoch[kMaxRanks];  // broadcast / p2p: per-destination (send) or per-source (receive)
  int vec_ok;               // in/out chunk pointers 32-byte aligned
  int div_mode;
  float recip, divisor;
  uint32_t* err;
  uint64_t timeout_ns;
  uint64_t* trace;  // optional event log (hccx_comm_trace_enable): [0] = count, then (tag, t_ns) pairs
  uint64_t trace_cap;
  uint64_t os_off, os_ag_off, os_flag_off;  // one-shot region: raw slots, gather slots, flags
  uint64_t os_raw_bytes, os_ag_bytes;       // one-shot slot strides
  int os_ll;                                // one-shot transport: 1 pairs (LL), 0 flags
  uint64_t os_ll_off, os_ll_ag_off;         // pair-mode regions: raw pairs, gather pairs
  uint64_t os_ll_raw_bytes, os_ll_ag_bytes;
  int ag_ring;         // allgather as a forwarding ring (1) or direct owner pushes (0)
  uint32_t first_segs;  // segments in the first step of every phase
  uint32_t step_segs;  // segments per published step (one release + flag per destination)
  uint32_t credit_all;  // bit c: slot class c (0 rs, 1 ag, 2 pp) changed geometry since its last use
  uint32_t ack_span;    // consumption-ack indices covering every CTA of any grid this communicator launches
  uint32_t max_grid;    // CTAs per rank cap shared by all ranks (0: the device's co-resident capacity)
  int debug;  // development knobs (HCCX_DEBUG): 16 = warp-store pushes, 32 = synchronous tile release, 64 = log launches,
            // 512 = lazy step publication, 256 = one system fence per signalled event
};

// Parameters of the virtual-rank kernels: nv ranks, G CTAs each.
struct VParams {
  FusedParams r[kMaxRanks];
  uint32_t G;
};

// Flag classes in every window:
//   0 rs[t]      data ready, written by the left neighbour      (p-1 slots x max_seg)
//   1 ag[i]      data ready, written by rank i                  (p x max_seg)
//   2 pp[i]      data ready, written by rank i                  (p x max_seg)
//   3 ack_rs[t]  rs[t] of the RIGHT neighbour consumed           (p-1 x kAckIdx)
//   4 ack_ag[r]  receiver r consumed our shard in its ag slot   (p x kAckIdx)
//   5 ack_pp[r]  receiver r consumed our pp message              (p x kAckIdx)
//   6 ack_agl[i] RIGHT neighbour consumed its ag slot i          (p x kAckIdx)
// A receiver acks every consumed ag slot both ways (to the shard's owner in
// class 4, to its left neighbour in class 6), so the direct allgather (owner
// pushes to everyone) and the ring allgather (left neighbour forwards) can
// alternate between calls: each checks the credit its own writer needs.
// Acks are per CTA index, not per segment: after a receiver CTA b (grid G)
// has consumed all of its segments of a slot it acks every index b, b+G, ...
// below kAckIdx, so each call acks the whole index space whatever its grid.
// A sender CTA waits once per slot per call on its own index's ack of the
// slot's previous use before overwriting it -- back-to-back collectives
// never race a slow receiver.
constexpr uint64_t kTraceMinWords = 16384 + 1024;  // fixed trace slots (timeouts 4000.., accumulators 4096..)
constexpr uint32_t kAckIdx = 1024;  // >= any co-resident grid of the fused kernel (148 SMs x CTAs per SM)

__device__ __forceinline__ uint32_t* flag_ptr(const FusedParams& P, int rank, int cls, int slot, uint32_t idx) {
  const int p = P.p;
  uint32_t* f = reinterpret_cast<uint32_t*>(P.win[rank] + P.flag_off);
  if (cls < 3) {
    const int base[3] = {0, p - 1, 2 * p - 1};
    return f + static_cast<uint64_t>(base[cls] + slot) * P.max_seg + idx;
  }
  const int base[4] = {0, p - 1, 2 * p - 1, 3 * p - 1};
  return f + static_cast<uint64_t>(3 * p - 1) * P.max_seg + static_cast<uint64_t>(base[cls - 3] + slot) * kAckIdx +
         idx;
}

__device__ __forceinline__ uint8_t* slot_ptr(const FusedParams& P, int rank, int slot_class, int slot) {
  const uint64_t off = slot_class == 0 ? P.rs_off : (slot_class == 1 ? P.ag_off : P.pp_off);
  return P.win[rank] + off + static_cast<uint64_t>(slot) * P.slot_bytes;
}

// Thread 0 spins until *flag >= epoch (wrap-safe) or the timeout expires.
// Expired waits are logged (trace words 4000..4090: cta << 32 | who) so the
// wait chain of a stalled collective can be read back.
__device__ __forceinline__ void trace_timeout(const FusedParams& P, uint32_t who, const uint32_t* prog = nullptr) {
  if (!P.trace || P.trace_cap < kTraceMinWords) return;  // hccx_comm_trace_enable enforces the minimum
  unsigned long long* t = reinterpret_cast<unsigned long long*>(P.trace);
  const unsigned long long i = atomicAdd(t + 4000, 1ull);
  if (i < 90) t[4001 + i] = (static_cast<unsigned long long>(blockIdx.x) << 32) | who;
  if (atomicCAS(t + 4095, 0ull, (static_cast<unsigned long long>(blockIdx.x) << 32) | who) == 0ull && prog) {
    for (int w = 0; w < 10; ++w) t[4200 + w] = prog[w];
  }
}

// Once any wait of this rank has timed out (err word), later waits return at
// once, so a dead peer costs one timeout, not one per segment.
__device__ __forceinline__ void spin_ge(const FusedParams& P, const uint32_t* flag, uint32_t epoch,
                                        uint32_t who = 0x600u) {
  if (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) >= 0) return;
  if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t spins = 0;
  while (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) < 0) {
    __nanosleep(32);
    if ((++spins & 1023u) == 0) {
      if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return;
      if (globaltimer_ns() - t0 > P.timeout_ns) {
        if (P.err) atomicOr(P.err, kErrTimeout);
        trace_timeout(P, who | (epoch << 12));
        return;
      }
    }
  }
}

// Bounded mbarrier wait for the fused kernel: a pipeline that stops making
// progress (a bug, or a peer that died mid-collective) turns into
// kErrTimeout + an identifying trace word instead of a hung GPU.
__device__ __forceinline__ void mbar_wait_to(const FusedParams& P, uint64_t* bar, uint32_t parity, uint32_t who,
                                             const uint32_t* prog = nullptr) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  if (ok) return;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t spins = 0;; ++spins) {
    // suspended in hardware until the phase completes (or ~20 us pass): a
    // waiting role warp takes no issue slots from the compute warps
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(20000u)
        : "memory");
    if (ok) return;
    if ((spins & 15u) == 15u) {
      if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return;
      if (globaltimer_ns() - t0 > P.timeout_ns) {
        if (P.err) atomicOr(P.err, kErrTimeout);
        trace_timeout(P, who, prog);
        return;
      }
    }
  }
}

// Publish a step.  The pushes of every thread precede this thread's
// release store through the CTA barrier (cumulativity of st.release at
// system scope), so no separate sc fence is needed; the remote reader
// pairs it with ld.acquire.sys.
__device__ __forceinline__ void signal(uint32_t* flag, uint32_t epoch) { st_release_sys(flag, epoch); }

// ---------------------------------------------------------------------------
// Warp-specialised fused kernel.
//
// One CTA per SM: kFCompute (24) compute warps + a producer, a pusher and a
// signaller warp.  The collective is a list of *phases* (ring rounds,
// allgather receives, ...; see phase_of) that every role walks in the same
// order.  The producer's elected lane waits for each step's inbound-data
// flag, then streams every segment's inputs (inbox payload and/or local
// fp32) into a per-phase carved (up to kFMaxStages deep) shared-memory ring
// with cp.async.bulk (completing on the stage's "full" mbarrier).  Compute
// warps decode / add / encode one group each per segment straight from
// shared memory, release the stage ("empty" mbarrier) and stage the encoded
// segment in a tile; the pusher hands tiles to the TMA engine (bulk stores
// into the peer's window); the signaller publishes completed steps and
// consumption acks with system-scope releases.  HBM latency is hidden
// behind several segments of prefetch per CTA.
// Partial segments (and unaligned buffers / non-word codecs) are read
// directly from global memory instead ("direct" stages).
// ---------------------------------------------------------------------------

constexpr int kFMaxStages = 8;                      // input ring depth cap (mbarrier pairs)
constexpr uint32_t kFArena = 6144u * kFusedWarps;    // input ring bytes, carved per phase
constexpr int kFMaxTiles = 8;                        // output (push) ring depth cap
constexpr uint32_t kFTileBudget = 2176u * kFusedWarps;  // output ring bytes
#ifndef HCCX_READS_IN_FLIGHT
#define HCCX_READS_IN_FLIGHT 4
#endif
#ifndef HCCX_PREFETCH_SEGS
#define HCCX_PREFETCH_SEGS 4
#endif
constexpr int kFReadsInFlight = HCCX_READS_IN_FLIGHT;  // bulk pushes whose smem read may be pending
constexpr uint32_t kFPrefetch = HCCX_PREFETCH_SEGS;  // L2 prefetch distance (segments)
constexpr int kFCompute = kFusedWarps;               // compute warps
constexpr int kFThreads2 = (kFCompute + 3) * 32;     // + producer, pusher and signaller warps
constexpr uint32_t kFGenBytes = kFCompute * kStageBytes;

// Output tiles hold one encoded segment (one group per compute warp) each;
// their size follows the codec (6 KiB at r8 with 24 warps), so the ring is as
// deep as the budget allows.
template <class Codec>
struct TileGeom {
  static constexpr uint32_t kBytes = (kSegGroups * Codec::kGroupBytes + 127u) / 128u * 128u;
  static constexpr int kFit = static_cast<int>(kFTileBudget / kBytes);
  static constexpr int kTiles = kFit > kFMaxTiles ? kFMaxTiles : (kFit < 2 ? 2 : kFit);
};

template <class Codec>
struct FusedSmem2 {
  uint8_t arena[kFArena];
  uint8_t tile[TileGeom<Codec>::kTiles][TileGeom<Codec>::kBytes];
  uint8_t gen[kFGenBytes];
  uint64_t full[kFMaxStages];
  uint64_t empty[kFMaxStages];
  uint64_t tfull[kFMaxTiles];
  uint64_t tempty[kFMaxTiles];
  uint32_t direct[kFMaxStages];
  uint32_t prog[kFCompute + 3];  // debug: per-warp progress word (phase << 20 | segment << 4 | state)
  uint32_t sig_events;           // pusher -> signaller: events completed (release/acquire, CTA scope)
};

enum PhaseKind : int { kPhEnc = 0, kPhDar = 1, kPhFinAr = 2, kPhFinRs = 3, kPhDec = 4 };

struct Phase {
  int kind;
  const uint8_t* pay;   // inbox slot (local window)
  const float* vals;    // local fp32 input chunk
  float* out;           // fp32 output chunk (or nullptr)
  bool div;             // apply the Average divisor to `out`
  int wait_cls, wait_slot;  // data flags to wait for (-1: none)
  uint32_t wait_ep;
  int push_cls, push_slot;  // destination slot (-1: no push)
  int push_mode;            // 0 right neighbour, 1 every peer, 2 P.dst
  int credit_cls;           // ack class to wait on before pushing (-1: none)
  uint32_t credit_ep;       // (pp: per destination, see credit_for)
  int ack_rank, ack_cls, ack_slot;  // consumption ack at phase end (-1: none)
  int ack2_rank, ack2_cls, ack2_slot;  // second ack (ag slots: owner and left neighbour)
  uint32_t ack_ep;
};

// Per-phase input stage geometry: A = the phase's primary input of one
// segment (fp32 for Enc, payload otherwise), B = local fp32 for the adds.
struct StageGeom {
  uint32_t a, b, stride;
  int n;
};

// HCCX_UNIFORM_STAGES: one stage geometry (the largest phase's) for the
// whole collective, so the input ring runs on across phase boundaries
// without draining; otherwise the arena is re-carved per phase.
#ifndef HCCX_UNIFORM_STAGES
#define HCCX_UNIFORM_STAGES 0
#endif
constexpr bool kFUniform = HCCX_UNIFORM_STAGES != 0;
#ifndef HCCX_ROTATE
#define HCCX_ROTATE 0
#endif
constexpr bool kFRotate = HCCX_ROTATE != 0;

template <class Codec>
__device__ __forceinline__ StageGeom stage_geom(int kind) {
  StageGeom g;
  g.a = kind == kPhEnc ? kSegVals * 4u : (kSegGroups * Codec::kGroupBytes + 127u) / 128u * 128u;
  g.b = (kind == kPhDar || kind == kPhFinAr || kind == kPhFinRs) ? kSegVals * 4u : 0u;
  g.stride = g.a + g.b;
  if constexpr (kFUniform) {
    const uint32_t pay = (kSegGroups * Codec::kGroupBytes + 127u) / 128u * 128u;
    const uint32_t big = pay + kSegVals * 4u;  // Dar / Fin (>= Enc's fp32 segment)
    g.stride = big > kSegVals * 4u ? big : kSegVals * 4u;
  }
  const uint32_t fit = kFArena / g.stride;
  g.n = static_cast<int>(fit < kFMaxStages ? fit : kFMaxStages);
  return g;
}

__device__ __forceinline__ int nphases(const FusedParams& P) {
  switch (P.op) {
    case kFAllReduce: return 2 * P.p - 1;
    case kFReduceScatter: return P.p;
    case kFAllGather: return P.p;
    default: return 1;  // broadcast / p2p: one phase per participant
  }
}

// Allgather receive k (1..p-1): shard i = j-k is in our ag slot i; decode it
// into `out`.  Ring mode (P.ag_ring): it came from the left neighbour and,
// unless the right neighbour owns it, is forwarded unchanged into the right
// neighbour's ag slot i.  Direct mode: its owner wrote it.  Every rank thus pushes (p-1)W bytes per allgather,
// one W per phase, instead of (p-1)W at once from the owner (which made the
// owner's last reduce-scatter phase NVLink-bound).  Consumption is acked to
// the left neighbour (the writer) per slot; the credit for slot i waits on
// the right neighbour's ack.
__device__ __forceinline__ void ring_ag_hop(const FusedParams& P, Phase& f, int k, float* out, bool div) {
  const int p = P.p, j = P.rank;
  const int i = (j - k + p) % p;
  f.kind = kPhDec;
  f.pay = P.win[j] + P.ag_off + static_cast<uint64_t>(i) * P.slot_bytes;
  f.out = out;
  f.div = div;
  f.wait_cls = 1;
  f.wait_slot = i;
  f.wait_ep = P.epoch;
  f.ack_rank = i;  // both acks, whatever the mode (see flag classes)
  f.ack_cls = 4;
  f.ack_slot = j;
  f.ack_ep = P.epoch;
  f.ack2_rank = (j + p - 1) % p;
  f.ack2_cls = 6;
  f.ack2_slot = i;
  if (P.ag_ring && k < p - 1) {
    f.push_cls = 1;
    f.push_slot = i;
    f.push_mode = 0;
    f.credit_cls = 6;
    f.credit_ep = P.prev_ag;
  }
}

__device__ __forceinline__ Phase phase_of(const FusedParams& P, int ph) {
  const int p = P.p, j = P.rank;
  const uint64_t c = P.n_chunk;
  auto cin = [&](int ch) { return P.in + static_cast<uint64_t>(((ch % p) + p) % p) * c; };
  auto cout = [&](int ch) { return P.out + static_cast<uint64_t>(((ch % p) + p) % p) * c; };
  Phase f;
  f.kind = kPhEnc;
  f.pay = nullptr;
  f.vals = nullptr;
  f.out = nullptr;
  f.div = false;
  f.wait_cls = -1;
  f.wait_slot = 0;
  f.wait_ep = 0;
  f.push_cls = -1;
  f.push_slot = 0;
  f.push_mode = 0;
  f.credit_cls = -1;
  f.credit_ep = 0;
  f.ack_rank = -1;
  f.ack_cls = 0;
  f.ack_slot = 0;
  f.ack_ep = 0;
  f.ack2_rank = -1;
  f.ack2_cls = 0;
  f.ack2_slot = 0;
  const int left = (j + p - 1) % p;
  if (P.op == kFAllReduce || P.op == kFReduceScatter) {
    if (ph < p) {
      const int t = ph;
      f.vals = cin(j - 1 - t);
      if (t > 0) {
        f.pay = P.win[j] + P.rs_off + static_cast<uint64_t>(t - 1) * P.slot_bytes;
        f.wait_cls = 0;
        f.wait_slot = t - 1;
        f.wait_ep = P.epoch;
        f.ack_rank = left;
        f.ack_cls = 3;
        f.ack_slot = t - 1;
        f.ack_ep = P.epoch;
      }
      if (t < p - 1) {
        f.kind = t == 0 ? kPhEnc : kPhDar;
        f.push_cls = 0;
        f.push_slot = t;
        f.push_mode = 0;
        f.credit_cls = 3;
        f.credit_ep = P.prev_rs;
      } else if (P.op == kFAllReduce) {
        f.kind = kPhFinAr;
        f.out = cout(j);
        f.div = true;
        f.push_cls = 1;  // own shard into ag slot j: the right neighbour (ring) or everyone (direct)
        f.push_slot = j;
        f.push_mode = P.ag_ring ? 0 : 1;
        f.credit_cls = P.ag_ring ? 6 : 4;
        f.credit_ep = P.prev_ag;
      } else {
        f.kind = kPhFinRs;
        f.out = P.out;
      }
    } else {
      ring_ag_hop(P, f, ph - p + 1, cout((j - (ph - p + 1) + p) % p), true);
    }
  } else if (P.op == kFAllGather) {
    if (ph == 0) {
      f.kind = kPhEnc;
      f.vals = P.in;
      f.out = P.out + static_cast<uint64_t>(j) * c;
      f.push_cls = 1;
      f.push_slot = j;
      f.push_mode = P.ag_ring ? 0 : 1;
      f.credit_cls = P.ag_ring ? 6 : 4;
      f.credit_ep = P.prev_ag;
    } else {
      ring_ag_hop(P, f, ph, P.out + static_cast<uint64_t>((j - ph + p) % p) * c, false);
    }
  } else {  // broadcast / p2p
    if (j == P.root) {
      f.kind = kPhEnc;
      f.vals = P.in;
      f.out = P.op == kFBroadcast ? P.out : nullptr;
      f.push_cls = 2;
      f.push_slot = j;
      f.push_mode = P.op == kFP2P ? 2 : 1;
      f.credit_cls = 5;
    } else {
      const int i = P.root;
      f.kind = kPhDec;
      f.pay = P.win[j] + P.pp_off + static_cast<uint64_t>(i) * P.slot_bytes;
      f.out = P.out;
      f.wait_cls = 2;
      f.wait_slot = i;
      f.wait_ep = P.pp_epoch[i];
      f.ack_rank = i;
      f.ack_cls = 5;
      f.ack_slot = j;
      f.ack_ep = P.pp_epoch[i];
    }
  }
  return f;
}

// Event log for CTA 0 (timeline of one CTA; ncu cannot replay a multi-rank
// kernel).  tag = (event << 32) | (phase << 16) | segment.
__device__ __forceinline__ void trace_ev(const FusedParams& P, uint32_t cta, uint32_t ev, uint32_t ph, uint32_t seg) {
  if (P.trace == nullptr || cta != 0) return;
  const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(P.trace), 1ull);
  if (2 * i + 2 < 4000 && 2 * i + 2 < P.trace_cap) {
    P.trace[1 + 2 * i] = (static_cast<uint64_t>(ev) << 32) | (static_cast<uint64_t>(ph) << 16) | seg;
    P.trace[2 + 2 * i] = globaltimer_ns();
  }
}

// Cycle accumulators for CTA 0 (written once at the end, slots 1..): a
// breakdown of where each role's time goes without per-event round trips.
__device__ __forceinline__ void trace_acc(const FusedParams& P, uint32_t cta, uint32_t slot, uint64_t cycles) {
  if (P.trace == nullptr || cta != 0 || 4096 + slot >= P.trace_cap) return;
  atomicAdd(reinterpret_cast<unsigned long long*>(P.trace) + 4096 + slot, static_cast<unsigned long long>(cycles));
}

__device__ __forceinline__ uint32_t push_epoch(const FusedParams& P, int push_cls, int d) {
  return push_cls == 2 ? P.pp_epoch[d] : P.epoch;
}


template <class Codec>
__device__ __forceinline__ void compute_group(const FusedParams& P, const Phase& f, uint64_t g, bool direct,
                                              const uint8_t* sa, const uint8_t* sb, uint8_t* tile_g, uint8_t* gen,
                                              int lane, uint32_t& bad) {
  const uint64_t base = g * kGroupVals;
  const uint32_t live = static_cast<uint32_t>(P.n_chunk - base < kGroupVals ? P.n_chunk - base : kGroupVals);
  const bool vec = P.vec_ok != 0;
  typename Codec::Lane s;
  float v[8];
  // ---- inputs
  if (f.kind == kPhEnc) {
    if (direct)
      load_vals<false>(f.vals, base, live, vec, lane, v);
    else
      ld_vals<2>(reinterpret_cast<const float*>(sa) + 8 * lane, v);
  } else {
    bool loaded = false;
    if constexpr (Codec::kFastPath) {
      if (!direct) {
        typename Codec::Raw raw;
        Codec::template load_raw<2>(raw, reinterpret_cast<const uint32_t*>(sa), lane);
        Codec::assemble(s, raw, lane);
        loaded = true;
      }
    }
    if (!loaded) group_load<Codec, false>(s, f.pay + g * Codec::kGroupBytes, live, true, gen, lane);
    Codec::decode(s, v);
    if (f.kind != kPhDec) {
      float loc[8];
      if (direct)
        load_vals<false>(f.vals, base, live, vec, lane, loc);
      else
        ld_vals<2>(reinterpret_cast<const float*>(sb) + 8 * lane, loc);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], loc[i]);
    }
  }
  // ---- outputs
  if (f.kind == kPhDec || f.kind == kPhFinRs) {
    if (f.kind == kPhDec && f.push_cls >= 0) {  // ring allgather: forward the payload bytes unchanged
      const uint32_t* src = reinterpret_cast<const uint32_t*>(direct ? f.pay + g * Codec::kGroupBytes : sa);
      uint32_t* dst = reinterpret_cast<uint32_t*>(tile_g);
      for (uint32_t w = static_cast<uint32_t>(lane); w < Codec::kGroupBytes / 4; w += 32) dst[w] = src[w];
    }
    if (f.div) apply_div(v, P.div_mode, P.recip, P.divisor);
    store_vals(f.out, base, live, vec, lane, v);
    return;
  }
  Codec::encode(v, s, bad, lane_live(live, lane));
  bool done = false;
  if constexpr (Codec::kFastPath) {
    if (live == kGroupVals && (reinterpret_cast<uintptr_t>(tile_g) & (Codec::kKind == 0 ? 31u : 3u)) == 0) {
      Codec::store_fast_generic(s, reinterpret_cast<uint32_t*>(tile_g), lane);
      done = true;
    }
  }
  if (!done) Codec::to_stage(s, tile_g, lane);
  if (f.out) {
    Codec::decode(s, v);
    if (f.div) apply_div(v, P.div_mode, P.recip, P.divisor);
    store_vals(f.out, base, live, vec, lane, v);
  }
}

static_assert(kFusedWarps == 8 || kFusedWarps == 12 || kFusedWarps == 24, "CTAs per SM = 24 / compute warps");

// The kernel body for one rank's CTA `cta` of `G`: the real kernel runs one
// rank per launch (cta = blockIdx.x); the virtual-rank kernel below splits
// one cooperative grid into several ranks on the same device (single-process
// communicators and the 1-GPU tests of this exact code).
template <class Codec>
__device__ __forceinline__ void ring_fused_body(const FusedParams& P, const uint32_t cta, const uint32_t G) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  FusedSmem2<Codec>& S = *reinterpret_cast<FusedSmem2<Codec>*>(smem_raw);
  constexpr int kT = TileGeom<Codec>::kTiles;
  // Compute needs tile (s mod kT) back before segment s; the pusher frees
  // tiles up to seq - kRd after segment seq-1, so kRd must stay below kT.
  constexpr int kRd = kFReadsInFlight < kT - 1 ? kFReadsInFlight : kT - 1;
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const int p = P.p, j = P.rank;
  const uint64_t c = P.n_chunk;
  const uint64_t ngroups = (c + kGroupVals - 1) / kGroupVals;
  const uint32_t nseg = static_cast<uint32_t>((ngroups + kSegGroups - 1) / kSegGroups);
  const uint64_t GB = Codec::kGroupBytes;
  const uint64_t wire = Codec::wire_bytes(c);
  // Segment set of this CTA: set, set + G, ... (acks and credits are per
  // set).  HCCX_ROTATE: the set index is rotated by rank, so a segment's
  // chain around the ring passes through different CTA indices (SMs) on
  // different ranks instead of CTA b everywhere.
  const uint32_t set = kFRotate ? (cta + static_cast<uint32_t>(j) * ((G + p - 1) / p)) % G : cta;
  const uint32_t myseg = nseg > set ? (nseg - set + G - 1) / G : 0;
  const int nph = nphases(P);
  // TMA needs whole 16B-multiple segments at 16B-aligned addresses: word
  // codecs with 32B-aligned fp32 chunks (payload segments are 8*GB bytes,
  // a multiple of 16, at 256B-aligned slot offsets).
  const bool tma_ok = Codec::kFastPath && P.vec_ok;
  auto seg_of = [&](uint32_t k) { return set + k * G; };
  auto seg_full = [&](uint32_t sg) { return (static_cast<uint64_t>(sg) + 1) * kSegVals <= c; };
  // Step boundaries within a phase: a short first step (P.first_segs) so the
  // neighbour's next phase can start early, then P.step_segs per step.
  auto step_end = [&](uint32_t k0) { return min(k0 == 0 ? P.first_segs : k0 + P.step_segs, myseg); };

  if (threadIdx.x == 0) {
    for (int st = 0; st < kFMaxStages; ++st) {
      mbar_init(&S.full[st], 1);
      mbar_init(&S.empty[st], kFCompute);
    }
    for (int tt = 0; tt < kT; ++tt) {
      mbar_init(&S.tfull[tt], kFCompute);
      mbar_init(&S.tempty[tt], 1);
    }
    S.sig_events = 0;
    fence_mbar_init();
  }
  Codec::kernel_init();
  __syncthreads();
  if (P.trace && threadIdx.x == 0 && 16384 + cta < P.trace_cap) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    P.trace[8192 + 2 * cta] = globaltimer_ns();
    P.trace[16384 + cta] = smid;
  }

  if (warp == kFCompute) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint64_t c_empty = 0, c_flag = 0, c_total = prof_clock();
      uint32_t pu = 0;  // per-barrier fill parity
      int st = 0;
      for (int ph = 0; ph < nph; ++ph) {
        const Phase f = phase_of(P, ph);
        const StageGeom sg_ = stage_geom<Codec>(f.kind);
        if constexpr (!kFUniform) {
          // the arena is re-carved for this phase: every earlier fill must be consumed
          for (int b = 0; b < kFMaxStages; ++b) mbar_wait_to(P, &S.empty[b], ((pu >> b) & 1u) ^ 1u, 0x100u | b, S.prog);
          st = 0;
        }
        for (uint32_t k0 = 0, k1; k0 < myseg; k0 = k1) {
          k1 = step_end(k0);
          if (f.wait_cls >= 0) {
            const uint64_t t0 = prof_clock();
            spin_ge(P, flag_ptr(P, j, f.wait_cls, f.wait_slot, seg_of(k0)), f.wait_ep, 0x700u | (ph << 4) | f.wait_cls);
            asm volatile("fence.proxy.async.global;" ::: "memory");
            c_flag += prof_clock() - t0;
            trace_ev(P, cta, 1, ph, k0);
          }
          for (uint32_t k = k0; k < k1; ++k) {
            const uint32_t sg = seg_of(k);
            // L2 prefetch kFPrefetch segments ahead (same step), so the
            // bulk load issued when the stage frees up hits L2
            if (tma_ok && k + kFPrefetch < k1) {
              const uint32_t sp = seg_of(k + kFPrefetch);
              if (seg_full(sp)) {
                if (f.kind == kPhEnc) {
                  bulk_prefetch_l2(f.vals + static_cast<uint64_t>(sp) * kSegVals, kSegVals * 4u);
                } else {
                  bulk_prefetch_l2(f.pay + static_cast<uint64_t>(sp) * kSegGroups * GB,
                                   static_cast<uint32_t>(kSegGroups * GB));
                  if (f.kind != kPhDec) bulk_prefetch_l2(f.vals + static_cast<uint64_t>(sp) * kSegVals, kSegVals * 4u);
                }
              }
            }
            HCCX_PROG(S.prog[kFCompute] = (ph << 20) | (k << 4) | 3u);
            const uint64_t t1 = prof_clock();
            mbar_wait_to(P, &S.empty[st], ((pu >> st) & 1u) ^ 1u, 0x200u | st, S.prog);
            c_empty += prof_clock() - t1;
            pu ^= 1u << st;
            const bool full_seg = tma_ok && seg_full(sg);
            S.direct[st] = full_seg ? 0u : 1u;
            uint8_t* base = S.arena + st * sg_.stride;
            if (full_seg) {
              const uint32_t a_bytes = f.kind == kPhEnc ? kSegVals * 4u : static_cast<uint32_t>(kSegGroups * GB);
              mbar_arrive_expect_tx(&S.full[st], a_bytes + sg_.b);
              if (f.kind == kPhEnc)
                bulk_g2s(base, f.vals + static_cast<uint64_t>(sg) * kSegVals, a_bytes, &S.full[st]);
              else
                bulk_g2s(base, f.pay + static_cast<uint64_t>(sg) * kSegGroups * GB, a_bytes, &S.full[st]);
              if (sg_.b) bulk_g2s(base + sg_.a, f.vals + static_cast<uint64_t>(sg) * kSegVals, sg_.b, &S.full[st]);
            } else {
              mbar_arrive(&S.full[st]);  // consumers read this segment from global memory
            }
            if (++st == sg_.n) st = 0;
          }
        }
      }
      trace_acc(P, cta, 0, prof_clock() - c_total);
      trace_acc(P, cta, 1, c_empty);
      trace_acc(P, cta, 2, c_flag);
    }
    return;
  }

  if (warp == kFCompute + 1) {
    // -------------------------------------------------------------- pusher
    // Takes each computed segment from the tile ring, hands it to the TMA
    // engine (one bulk store per destination window), recycles the tile
    // once the engine has read it, and publishes every step with one
    // release store per destination after its bulk writes completed.
    // Control flow is uniform across the warp: lane 0 alone waits on and
    // arrives at mbarriers, spins on credits and writes flags; the other
    // lanes only join the 16-byte store loops.  Every lane passes exactly
    // the same sequence of __syncwarp() calls (divergent lane-0 blocks plus
    // __syncwarp at different sites let lanes drift a segment apart).
    int tt = 0;
    uint32_t tbit = 0;
    uint32_t seq = 0, released = 0;  // segments seen / tiles handed back (ring order)
    uint64_t c_tfull = 0, c_read = 0, c_pub = 0, c_credit = 0, c_issue = 0, c_total = prof_clock();
    uint32_t events = 0;  // signaller events issued (lane 0)
    // Lazy publication (lane 0): a finished step's event is queued with the
    // bulk-group count at its end and handed to the signaller once those
    // groups have completed -- checked kLazy groups later (by then they are
    // done, so the wait is free) or whenever the pusher would otherwise
    // block (waiting for a tile or a credit): the TMA engine keeps pushing
    // across step boundaries instead of draining at every step.  Events
    // (step publications and phase-end acks) stay in the signaller's order.
    constexpr int kLazy = 3;
    constexpr int kPend = 8;
    uint32_t pend_g[kPend];  // group count at the step's end; ~0u = ack event (no bulk dependency)
    int pend_head = 0, pend_n = 0;
    uint32_t groups = 0;     // bulk groups committed (one per pushed segment)
    auto release_upto = [&](uint32_t upto) {
      for (; released < upto; ++released) mbar_arrive(&S.tempty[released % kT]);
    };
    auto emit = [&](bool drain) {  // lane 0
      bool waited_all = false;
      while (pend_n) {
        const uint32_t g = pend_g[pend_head];
        if (g != ~0u) {
          if (groups - g >= static_cast<uint32_t>(kLazy)) {
            asm volatile("cp.async.bulk.wait_group %0;" ::"n"(kLazy) : "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
          } else if (drain) {
            if (!waited_all) bulk_wait_all();
            waited_all = true;
          } else {
            break;
          }
        }
        st_release_cta_shared(&S.sig_events, ++events);
        pend_head = (pend_head + 1) % kPend;
        --pend_n;
      }
    };
    auto enqueue = [&](uint32_t g) {  // lane 0
      if (pend_n == kPend) emit(true);
      pend_g[(pend_head + pend_n) % kPend] = g;
      ++pend_n;
    };
    for (int ph = 0; ph < nph; ++ph) {
      const Phase f = phase_of(P, ph);
      const bool push = f.push_cls >= 0;
      const uint64_t tc = prof_clock();
      if (push) {  // credit: previous use of the destination slot(s) consumed
        // Same slot geometry as the previous use (codec, chunk size, hence
        // grid and segment bytes): this CTA's segments were read by the
        // receiver CTA with our index, whose ack we wait for.  Geometry
        // changed (P.credit_all): the byte ranges we are about to overwrite
        // were read by arbitrary receiver CTAs, so wait for all of them --
        // receiver CTA r of a grid G' acked indices r, r+G', ..., so indices
        // [0, ack_span) cover every CTA of any grid <= ack_span.
        if (lane == 0) emit(true);  // never hold a publication across a wait on a peer
        __syncwarp();
        const bool all = ((P.credit_all >> f.push_cls) & 1u) != 0;
        for (int q = 1; q < p; ++q) {
          const int d = (j + q) % p;
          if (f.push_mode == 0 && d != (j + 1) % p) continue;
          if (f.push_mode == 2 && d != P.dst) continue;
          const uint32_t need = f.push_cls == 2 ? P.pp_epoch[d] - 1u : f.credit_ep;
          const uint32_t* fl = flag_ptr(P, j, f.credit_cls, f.push_mode == 0 ? f.push_slot : d, 0);
          if (all) {
            for (uint32_t k = lane; k < P.ack_span; k += 32) spin_ge(P, fl + k, need, 0x900u | (ph << 4) | f.credit_cls);
          } else if (lane == 0) {
            spin_ge(P, fl + set, need, 0x800u | (ph << 4) | f.credit_cls);
          }
        }
      }
      __syncwarp();
      c_credit += prof_clock() - tc;
      for (uint32_t k0 = 0, k1; k0 < myseg; k0 = k1) {
        k1 = step_end(k0);
        for (uint32_t k = k0; k < k1; ++k) {
          const uint32_t sg = seg_of(k);
          if (lane == 0) {
            HCCX_PROG(S.prog[kFCompute + 1] = (ph << 20) | (k << 4) | 2u);
            const uint64_t t0 = prof_clock();
            // about to wait for compute: publish what has completed first
            if (pend_n && !mbar_test(&S.tfull[tt], tbit)) emit(true);
            mbar_wait_to(P, &S.tfull[tt], tbit, 0x300u | tt, S.prog);
            c_tfull += prof_clock() - t0;
          }
          __syncwarp();  // the tile is complete for every lane
          bool bulk_issued = false;
          if (push) {
            const uint64_t soff = static_cast<uint64_t>(sg) * kSegGroups * GB;
            const uint64_t rem = wire - soff;
            const uint32_t nb = static_cast<uint32_t>(rem < kSegGroups * GB ? rem : kSegGroups * GB);
            // TMA bulk push (one instruction per destination); HCCX_DEBUG
            // bit 16 selects the warp's 16-byte stores instead.
            if ((nb & 15u) == 0 && !(P.debug & 16)) {
              if (lane == 0) {
                const uint64_t ti = prof_clock();
                // the tile was written through the generic proxy; the bulk
                // copy reads it through the async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                for (int q = 1; q < p; ++q) {
                  const int d = (j + q) % p;
                  if (f.push_mode == 0 && q != 1) break;
                  if (f.push_mode == 2 && d != P.dst) continue;
                  bulk_s2g(slot_ptr(P, d, f.push_cls, f.push_slot) + soff, S.tile[tt], nb);
                }
                bulk_commit();
                ++groups;
                c_issue += prof_clock() - ti;
                trace_ev(P, cta, 3, ph, k);
              }
              bulk_issued = true;
            } else {
              for (int q = 1; q < p; ++q) {
                const int d = (j + q) % p;
                if (f.push_mode == 0 && q != 1) break;
                if (f.push_mode == 2 && d != P.dst) continue;
                uint8_t* dst = slot_ptr(P, d, f.push_cls, f.push_slot) + soff;
                const uint32_t n16 = (nb & 15u) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0 ? nb >> 4 : 0;
                for (uint32_t i = lane; i < n16; i += 32)
                  reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(S.tile[tt])[i];
                for (uint32_t b = (n16 << 4) + lane; b < nb; b += 32) dst[b] = S.tile[tt][b];
              }
            }
          }
          ++seq;
          __syncwarp();  // every lane's reads of the tile are done
          if (lane == 0) {
            const uint64_t t1 = prof_clock();
            if (bulk_issued && !(P.debug & 32)) {
              bulk_wait_read<kRd>();  // hand tiles back once the TMA engine has read them
              release_upto(seq > static_cast<uint32_t>(kRd) ? seq - kRd : 0);
            } else {
              if (bulk_issued) bulk_wait_read<0>();
              release_upto(seq);
            }
            if (pend_n) emit(false);
            c_read += prof_clock() - t1;
          }
          if (++tt == kT) {
            tt = 0;
            tbit ^= 1u;
          }
        }
        if (push) {  // the step is issued: its publication follows once its groups complete
          const uint64_t t2 = prof_clock();
          if (lane == 0) {
            // (warp-copied segments commit no group: their lanes' stores
            // are ordered before lane 0's event release by __syncwarp)
            // Eager by default: measured at p = 4 (tools/nvl_ab.py), lazy
            // publication cost 6% -- consumers saw the flags later than the
            // drain at the step end costs the pusher.  HCCX_DEBUG bit 512:
            // lazy (development).
            enqueue(groups);
            if (!(P.debug & 512)) emit(true);
          }
          c_pub += prof_clock() - t2;
          __syncwarp();
        }
      }
      // every segment of the phase has been computed (tfull) -> its inbox
      // inputs are consumed: the signaller acknowledges them
      if (f.ack_rank >= 0 && lane == 0) enqueue(~0u);
      __syncwarp();
    }
    if (lane == 0) {
      emit(true);
      bulk_wait_all();
      release_upto(seq);
      trace_acc(P, cta, 8, prof_clock() - c_total);
      trace_acc(P, cta, 9, c_tfull);
      trace_acc(P, cta, 10, c_read);
      trace_acc(P, cta, 11, c_pub);
      trace_acc(P, cta, 12, c_credit);
      trace_acc(P, cta, 13, c_issue);
      if (P.trace && 8192 + 2 * cta + 1 < P.trace_cap) P.trace[8193 + 2 * cta] = globaltimer_ns();
    }
    return;
  }

  if (warp == kFCompute + 2) {
    // ----------------------------------------------------------- signaller
    // Publishes the pusher's completed steps (one flag store per
    // destination) and the phase-end consumption acks.  Walks the same
    // (phase, step) event sequence as the pusher; event e is ready once
    // S.sig_events >= e (the pusher's release.cta after the step's bulk
    // writes completed).  A system-scope fence costs microseconds while
    // NVLink writes are in flight, so events are published in batches: one
    // acquire of the ready count, one fence.acq_rel.sys by every lane, then
    // relaxed system-scope stores for every event up to that count --
    // causality order carries the data writes to the remote acquirer.
    uint32_t events = 0, ready = 0;
    uint64_t c_sig = 0, c_ack = 0;
    auto need = [&](uint32_t ev) {  // make event ev publishable (fenced)
      if (P.debug & 256) ready = 0;  // development: one fence per event (no batching)
      if (ev <= ready) return;
      if (lane == 0) {
        const uint64_t t0 = globaltimer_ns();
        uint32_t r;
        for (uint32_t spins = 0; (r = ld_acquire_cta_shared(&S.sig_events)) < ev; ++spins) {
          __nanosleep(64);  // leave the issue slots to the compute warps
          if ((spins & 255u) == 255u) {
            if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) break;
            if (globaltimer_ns() - t0 > P.timeout_ns) {
              if (P.err) atomicOr(P.err, kErrTimeout);
              trace_timeout(P, 0xa00u, S.prog);
              break;
            }
          }
        }
        ready = r < ev ? ev : r;
      }
      __syncwarp();
      ready = __shfl_sync(kFull, ready, 0);
      fence_acq_rel_sys();
    };
    for (int ph = 0; ph < nph; ++ph) {
      const Phase f = phase_of(P, ph);
      if (f.push_cls >= 0) {
        for (uint32_t k0 = 0; k0 < myseg; k0 = step_end(k0)) {
          const uint64_t ts = prof_clock();
          need(++events);
          if (lane < p - 1) {
            const int d = (j + 1 + lane) % p;
            const bool tgt =
                f.push_mode == 1 || (f.push_mode == 0 && lane == 0) || (f.push_mode == 2 && d == P.dst);
            if (tgt) st_relaxed_sys(flag_ptr(P, d, f.push_cls, f.push_slot, seg_of(k0)), push_epoch(P, f.push_cls, d));
          }
          __syncwarp();
          c_sig += prof_clock() - ts;
          if (lane == 0) trace_ev(P, cta, 5, ph, k0);
        }
      }
      if (f.ack_rank >= 0) {
        const uint64_t ta = prof_clock();
        need(++events);
        for (uint32_t kk = set + lane * G; kk < kAckIdx; kk += G * 32) {
          st_relaxed_sys(flag_ptr(P, f.ack_rank, f.ack_cls, f.ack_slot, 0) + kk, f.ack_ep);
          if (f.ack2_rank >= 0) st_relaxed_sys(flag_ptr(P, f.ack2_rank, f.ack2_cls, f.ack2_slot, 0) + kk, f.ack_ep);
        }
        c_ack += prof_clock() - ta;
        __syncwarp();
      }
    }
    if (lane == 0) {
      trace_acc(P, cta, 14, c_ack);
      trace_acc(P, cta, 15, c_sig);
    }
    return;
  }

  // -------------------------------------------------------------- compute
  uint32_t bad = 0;
  uint32_t cu = 0;  // per-barrier consume parity
  int tt = 0;
  uint32_t tbit = 0;
  uint8_t* gen = S.gen + warp * kStageBytes;
  uint64_t c_full = 0, c_tile = 0, c_comp = 0, c_total = prof_clock();
  int st = 0;
  for (int ph = 0; ph < nph; ++ph) {
    const Phase f = phase_of(P, ph);
    const StageGeom sg_ = stage_geom<Codec>(f.kind);
    if constexpr (!kFUniform) st = 0;
    for (uint32_t k = 0; k < myseg; ++k) {
      const uint32_t sg = seg_of(k);
      if (lane == 0) HCCX_PROG(S.prog[warp] = (ph << 20) | (k << 4) | 1u);
      const uint64_t t0 = prof_clock();
      mbar_wait_to(P, &S.full[st], (cu >> st) & 1u, 0x400u | st, S.prog);
      cu ^= 1u << st;
      if (lane == 0) HCCX_PROG(S.prog[warp] = (ph << 20) | (k << 4) | 2u);
      const uint64_t t1 = prof_clock();
      mbar_wait_to(P, &S.tempty[tt], tbit ^ 1u, 0x500u | tt, S.prog);
      const uint64_t t2 = prof_clock();
      c_full += t1 - t0;
      c_tile += t2 - t1;
      const bool direct = S.direct[st] != 0;
      const uint64_t g = static_cast<uint64_t>(sg) * kSegGroups + warp;
      const uint8_t* base = S.arena + st * sg_.stride;
      const uint8_t* sa = base + (f.kind == kPhEnc ? warp * 1024u : warp * static_cast<uint32_t>(GB));
      const uint8_t* sb = base + sg_.a + warp * 1024u;
      if (g < ngroups) compute_group<Codec>(P, f, g, direct, sa, sb, S.tile[tt] + warp * GB, gen, lane, bad);
      __syncwarp();
      c_comp += prof_clock() - t2;
      if (warp == 0 && lane == 0) trace_ev(P, cta, 2, ph, k);
      if (lane == 0) HCCX_PROG(S.prog[warp] = (ph << 20) | (k << 4) | 3u);
      if (lane == 0) {
        mbar_arrive(&S.empty[st]);
        mbar_arrive(&S.tfull[tt]);
      }
      if (++st == sg_.n) st = 0;
      if (++tt == kT) {
        tt = 0;
        tbit ^= 1u;
      }
    }
  }
  if (lane == 0 && warp == 0) {
    trace_acc(P, cta, 16, prof_clock() - c_total);
    trace_acc(P, cta, 17, c_full);
    trace_acc(P, cta, 18, c_tile);
    trace_acc(P, cta, 19, c_comp);
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

template <class Codec>
__global__ void __launch_bounds__(kFThreads2, kFCtasPerSm) ring_fused_kernel(const __grid_constant__ FusedParams P) {
  pdl_wait_and_release();  // see oneshot_allreduce_kernel
  ring_fused_body<Codec>(P, blockIdx.x, gridDim.x);
}

// Virtual ranks: several ranks of one communicator on this device share one
// cooperative grid of nv x G CTAs (all co-resident, so every flag wait can
// be satisfied); rank v's parameters are V.r[v] (a large kernel parameter,
// up to 16 x sizeof(FusedParams), passed by value: graph-capturable).
template <class Codec>
__global__ void __launch_bounds__(kFThreads2, kFCtasPerSm) ring_fused_vkernel(const __grid_constant__ VParams V) {
  const uint32_t v = blockIdx.x / V.G;
  ring_fused_body<Codec>(V.r[v], blockIdx.x - v * V.G, V.G);
}

}  // namespace hccx
