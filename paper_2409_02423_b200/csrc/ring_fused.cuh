// ring_fused.cuh -- the multi-process NVLink engine: ONE persistent kernel per
// collective per rank, moving only compressed chunks between GPUs.
//
// Every rank owns a window (cudaMalloc'd, exported with CUDA IPC, mapped by
// every peer over NVLink/NVSwitch) holding inbox slots and per-segment flags:
//   rs[t]   t = 0..p-2   message of ring round t from the left neighbour
//   ag[i]   i = 0..p-1   compressed final shard C_i of rank i (allgather)
//   pp[i]   i = 0..p-1   point-to-point / broadcast message from rank i
// A "segment" is a tile of 8 warp groups (2048 values) of a chunk; CTA b of
// the cooperative grid owns segments b, b+G, b+2G, ... in every round, so
// rank j's CTA b only ever waits on rank (j-1)'s CTA b: a per-segment
// wavefront pipeline with no grid-wide barrier.
//
// Ring schedule (identical bits to proj/src/collectives.cpp:27-111):
//   round 0     encode local chunk (j-1) mod p -> push to rs[0] of rank j+1
//   round t     wait rs[t-1]; fused decompress-add-recompress with local
//               chunk (j-1-t) mod p -> push to rs[t] of rank j+1
//   final       wait rs[p-2]; add local chunk j ->
//                 allreduce: encode C_j, push to ag[j] of every peer, write
//                            dec(C_j) (/p) to out chunk j
//                 reduce-scatter: write the fp32 sum to the shard
//   allgather   wait ag[i] of every peer i, decode (/p) to out chunk i
// A segment's compressed bytes are assembled in shared memory and pushed to
// the peer with 16-byte stores; then one thread fences (system scope) and
// release-stores the epoch into the peer's flag.  Waits are bounded
// (%globaltimer); a timeout raises kErrTimeout instead of hanging the GPU.
#pragma once
#include "step_kernel.cuh"

namespace hccx {

constexpr int kMaxRanks = 16;
constexpr int kFusedWarps = 8;
constexpr int kFusedThreads = kFusedWarps * 32;
constexpr int kSegGroups = kFusedWarps;  // groups per segment
constexpr uint32_t kSegVals = kSegGroups * kGroupVals;
constexpr uint32_t kStepSegs = 16;  // segments per published step (one fence + flag)

enum FusedOp : int { kFAllReduce = 0, kFReduceScatter = 1, kFAllGather = 2, kFBroadcast = 3, kFP2P = 4 };

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
};

struct FusedSmem {
  uint8_t tile[kSegGroups * 1040];  // >= 8 x largest group (1028 B), 16B multiple
  uint8_t stage[kFusedWarps][kStageBytes];
};

// Flag classes in every window:
//   0 rs[t]      data ready, written by the left neighbour      (p-1 slots x max_seg)
//   1 ag[i]      data ready, written by rank i                  (p x max_seg)
//   2 pp[i]      data ready, written by rank i                  (p x max_seg)
//   3 ack_rs[t]  rs[t] of the RIGHT neighbour consumed           (p-1 x kAckIdx)
//   4 ack_ag[r]  receiver r consumed our shard in its ag slot   (p x kAckIdx)
//   5 ack_pp[r]  receiver r consumed our pp message              (p x kAckIdx)
// Acks are per CTA index, not per segment: after a receiver CTA b (grid G)
// has consumed all of its segments of a slot it acks every index b, b+G, ...
// below kAckIdx, so each call acks the whole index space whatever its grid.
// A sender CTA waits once per slot per call on its own index's ack of the
// slot's previous use before overwriting it -- back-to-back collectives
// never race a slow receiver.
constexpr uint32_t kAckIdx = 2048;  // > any co-resident grid (148 SMs x 8 CTAs)

__device__ __forceinline__ uint32_t* flag_ptr(const FusedParams& P, int rank, int cls, int slot, uint32_t idx) {
  const int p = P.p;
  uint32_t* f = reinterpret_cast<uint32_t*>(P.win[rank] + P.flag_off);
  if (cls < 3) {
    const int base[3] = {0, p - 1, 2 * p - 1};
    return f + static_cast<uint64_t>(base[cls] + slot) * P.max_seg + idx;
  }
  const int base[3] = {0, p - 1, 2 * p - 1};
  return f + static_cast<uint64_t>(3 * p - 1) * P.max_seg + static_cast<uint64_t>(base[cls - 3] + slot) * kAckIdx +
         idx;
}

__device__ __forceinline__ uint8_t* slot_ptr(const FusedParams& P, int rank, int slot_class, int slot) {
  const uint64_t off = slot_class == 0 ? P.rs_off : (slot_class == 1 ? P.ag_off : P.pp_off);
  return P.win[rank] + off + static_cast<uint64_t>(slot) * P.slot_bytes;
}

// Thread 0 spins until *flag >= epoch (wrap-safe) or the timeout expires.
// Once any wait of this rank has timed out (err word), later waits return at
// once, so a dead peer costs one timeout, not one per segment.
__device__ __forceinline__ void spin_ge(const FusedParams& P, const uint32_t* flag, uint32_t epoch) {
  if (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) >= 0) return;
  if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return;
  const uint64_t t0 = globaltimer_ns();
  uint32_t spins = 0;
  while (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) < 0) {
    if ((++spins & 1023u) == 0) {
      if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return;
      if (globaltimer_ns() - t0 > P.timeout_ns) {
        if (P.err) atomicOr(P.err, kErrTimeout);
        return;
      }
    }
  }
}

// The CTA barrier publishes thread 0's acquire to every warp.
__device__ __forceinline__ void seg_wait(const FusedParams& P, const uint32_t* flag, uint32_t epoch) {
  if (threadIdx.x == 0) spin_ge(P, flag, epoch);
  __syncthreads();
}

// Push `nbytes` of the staged tile to `dst` (peer memory) with 16-byte stores.
__device__ __forceinline__ void push_tile(const uint8_t* tile, uint8_t* dst, uint32_t nbytes) {
  const uint32_t n16 = nbytes >> 4;
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(tile)[i];
    for (uint32_t b = (n16 << 4) + threadIdx.x; b < nbytes; b += blockDim.x) dst[b] = tile[b];
  } else {
    for (uint32_t b = threadIdx.x; b < nbytes; b += blockDim.x) dst[b] = tile[b];
  }
}

__device__ __forceinline__ void signal(uint32_t* flag, uint32_t epoch) {
  __threadfence_system();
  st_release_sys(flag, epoch);
}

// Consumption ack for this CTA's indices (see kAckIdx).  Call after a CTA
// barrier that follows the last read of the slot.
__device__ __forceinline__ void ack_all(uint32_t* flags, uint32_t epoch) {
  for (uint32_t k = blockIdx.x + threadIdx.x * gridDim.x; k < kAckIdx; k += gridDim.x * blockDim.x)
    st_release_sys(flags + k, epoch);
}

// One warp's group of a segment.
//   kEnc  : values (src_vals [+ local]) -> encoded group written into the
//           shared tile at `tile_g`; optional decoded copy -> out_vals
//   !kEnc : payload (src_pay, local memory) decoded [+ local] -> out_vals
template <class Codec, bool kEnc, bool kAdd>
__device__ __forceinline__ void fused_group(const FusedParams& P, const uint8_t* src_pay, const float* src_vals,
                                            const float* local, float* out_vals, bool out_is_sum,
                                            uint8_t* tile_g, uint64_t g, uint8_t* sm, int lane, uint32_t& bad) {
  const uint64_t base = g * kGroupVals;
  const uint32_t live = static_cast<uint32_t>(P.n_chunk - base < kGroupVals ? P.n_chunk - base : kGroupVals);
  const bool full = live == kGroupVals;
  const bool vec = P.vec_ok != 0;
  typename Codec::Lane s;
  float v[8];
  if (src_pay) {
    group_load<Codec, false>(s, src_pay + g * Codec::kGroupBytes, live, true, sm, lane);
    Codec::decode(s, v);
  } else {
    load_vals<false>(src_vals, base, live, vec, lane, v);
  }
  if constexpr (kAdd) {
    float loc[8];
    load_vals<false>(local, base, live, vec, lane, loc);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], loc[i]);
  }
  if constexpr (kEnc) {
    Codec::encode(v, s, bad, lane_live(live, lane));
    bool done = false;
    if constexpr (Codec::kFastPath) {
      if (full && (reinterpret_cast<uintptr_t>(tile_g) & (Codec::kKind == 0 ? 31u : 3u)) == 0) {
        Codec::store_fast_generic(s, reinterpret_cast<uint32_t*>(tile_g), lane);
        done = true;
      }
    }
    if (!done) Codec::to_stage(s, tile_g, lane);
    if (out_vals) {
      Codec::decode(s, v);
      apply_div(v, P.div_mode, P.recip, P.divisor);
      store_vals(out_vals, base, live, vec, lane, v);
    }
  } else {
    if (!out_is_sum) apply_div(v, P.div_mode, P.recip, P.divisor);
    store_vals(out_vals, base, live, vec, lane, v);
  }
}

template <class Codec>
__global__ void __launch_bounds__(kFusedThreads) ring_fused_kernel(const __grid_constant__ FusedParams P) {
  __shared__ __align__(16) FusedSmem S;
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const int p = P.p, j = P.rank;
  const uint64_t c = P.n_chunk;
  const uint64_t ngroups = (c + kGroupVals - 1) / kGroupVals;
  const uint32_t nseg = static_cast<uint32_t>((ngroups + kSegGroups - 1) / kSegGroups);
  const uint64_t GB = Codec::kGroupBytes;
  const uint64_t wire = Codec::wire_bytes(c);
  uint8_t* tile = S.tile;
  uint8_t* sm = S.stage[warp];
  uint32_t bad = 0;
  auto chunk_in = [&](int ch) { return P.in + static_cast<uint64_t>(((ch % p) + p) % p) * c; };
  auto chunk_out = [&](int ch) { return P.out + static_cast<uint64_t>(((ch % p) + p) % p) * c; };
  auto seg_bytes = [&](uint32_t sg) {
    const uint64_t start = static_cast<uint64_t>(sg) * kSegGroups * GB;
    const uint64_t rem = wire - start;
    return static_cast<uint32_t>(rem < kSegGroups * GB ? rem : kSegGroups * GB);
  };
  const int right = (j + 1) % p, left = (j + p - 1) % p;

  // This CTA's segments are sg = blockIdx.x + k*G, k < myseg.  They are
  // processed in steps of kStepSegs segments; a step is published with ONE
  // system-scope fence + flag (indexed by the step's first segment), which
  // amortises the fence over up to kStepSegs x 8 groups.
  const uint32_t G = gridDim.x;
  const uint32_t myseg = nseg > blockIdx.x ? (nseg - blockIdx.x + G - 1) / G : 0;
  auto seg_of = [&](uint32_t k) { return blockIdx.x + k * G; };

  if (P.op == kFAllReduce || P.op == kFReduceScatter) {
    const bool ar = P.op == kFAllReduce;
    for (int t = 0; t < p; ++t) {  // t = p-1 is the final receive
      const bool last = t == p - 1;
      const bool push = !(last && !ar);
      // credit for the slot(s) this round pushes into (previous use consumed)
      if (threadIdx.x == 0) {
        if (!last) spin_ge(P, flag_ptr(P, j, 3, t, blockIdx.x), P.prev_rs);
        if (last && ar)
          for (int q = 1; q < p; ++q) spin_ge(P, flag_ptr(P, j, 4, (j + q) % p, blockIdx.x), P.prev_ag);
      }
      const uint8_t* rx = t > 0 ? slot_ptr(P, j, 0, t - 1) : nullptr;
      const float* local = chunk_in(j - 1 - t);
      for (uint32_t k0 = 0; k0 < myseg; k0 += kStepSegs) {
        const uint32_t k1 = min(k0 + kStepSegs, myseg);
        if (threadIdx.x == 0 && t > 0) spin_ge(P, flag_ptr(P, j, 0, t - 1, seg_of(k0)), P.epoch);
        __syncthreads();
        for (uint32_t k = k0; k < k1; ++k) {
          const uint32_t sg = seg_of(k);
          const uint64_t g = static_cast<uint64_t>(sg) * kSegGroups + warp;
          if (g < ngroups) {
            if (!push) {
              fused_group<Codec, false, true>(P, rx, nullptr, local, P.out, true, nullptr, g, sm, lane, bad);
            } else {
              uint8_t* tg = tile + warp * GB;
              float* ov = last ? chunk_out(j) : nullptr;
              if (t == 0)
                fused_group<Codec, true, false>(P, nullptr, local, nullptr, ov, false, tg, g, sm, lane, bad);
              else
                fused_group<Codec, true, true>(P, rx, nullptr, local, ov, false, tg, g, sm, lane, bad);
            }
          }
          if (!push) continue;  // reduce-scatter final: fp32 shard, nothing to push
          __syncthreads();
          const uint64_t soff = static_cast<uint64_t>(sg) * kSegGroups * GB;
          const uint32_t nb = seg_bytes(sg);
          if (!last)
            push_tile(tile, slot_ptr(P, right, 0, t) + soff, nb);
          else
            for (int q = 1; q < p; ++q) push_tile(tile, slot_ptr(P, (j + q) % p, 1, j) + soff, nb);
          __syncthreads();
        }
        if (push) {
          if (!last) {
            if (threadIdx.x == 0) signal(flag_ptr(P, right, 0, t, seg_of(k0)), P.epoch);
          } else if (threadIdx.x < p - 1) {
            signal(flag_ptr(P, (j + 1 + threadIdx.x) % p, 1, j, seg_of(k0)), P.epoch);
          }
        }
      }
      if (t > 0) {
        __syncthreads();
        ack_all(flag_ptr(P, left, 3, t - 1, 0), P.epoch);
      }
    }
    if (ar) {
      for (int q = 1; q < p; ++q) {
        const int i = (j - q + p) % p;
        for (uint32_t k0 = 0; k0 < myseg; k0 += kStepSegs) {
          const uint32_t k1 = min(k0 + kStepSegs, myseg);
          seg_wait(P, flag_ptr(P, j, 1, i, seg_of(k0)), P.epoch);
          for (uint32_t k = k0; k < k1; ++k) {
            const uint64_t g = static_cast<uint64_t>(seg_of(k)) * kSegGroups + warp;
            if (g < ngroups)
              fused_group<Codec, false, false>(P, slot_ptr(P, j, 1, i), nullptr, nullptr, chunk_out(i), false,
                                               nullptr, g, sm, lane, bad);
          }
        }
        __syncthreads();
        ack_all(flag_ptr(P, i, 4, j, 0), P.epoch);
      }
    }
  } else {
    // allgather: every rank is an origin (its shard, ag slots); broadcast /
    // p2p: the root is the origin (pp slots, pairwise epochs).
    const bool ag = P.op == kFAllGather;
    const int cls = ag ? 1 : 2;
    const bool origin = ag || j == P.root;
    float* own_out = ag ? P.out + static_cast<uint64_t>(j) * c : (P.op == kFBroadcast ? P.out : nullptr);
    if (origin) {
      if (threadIdx.x == 0) {
        for (int q = 1; q < p; ++q) {
          const int d = (j + q) % p;
          if (P.op == kFP2P && d != P.dst) continue;
          spin_ge(P, flag_ptr(P, j, ag ? 4 : 5, d, blockIdx.x), ag ? P.prev_ag : P.pp_epoch[d] - 1u);
        }
      }
      __syncthreads();
      for (uint32_t k0 = 0; k0 < myseg; k0 += kStepSegs) {
        const uint32_t k1 = min(k0 + kStepSegs, myseg);
        for (uint32_t k = k0; k < k1; ++k) {
          const uint32_t sg = seg_of(k);
          const uint64_t g = static_cast<uint64_t>(sg) * kSegGroups + warp;
          if (g < ngroups)
            fused_group<Codec, true, false>(P, nullptr, P.in, nullptr, own_out, false, tile + warp * GB, g, sm,
                                            lane, bad);
          __syncthreads();
          const uint64_t soff = static_cast<uint64_t>(sg) * kSegGroups * GB;
          const uint32_t nb = seg_bytes(sg);
          if (P.op == kFP2P)
            push_tile(tile, slot_ptr(P, P.dst, cls, j) + soff, nb);
          else
            for (int q = 1; q < p; ++q) push_tile(tile, slot_ptr(P, (j + q) % p, cls, j) + soff, nb);
          __syncthreads();
        }
        if (P.op == kFP2P) {
          if (threadIdx.x == 0) signal(flag_ptr(P, P.dst, cls, j, seg_of(k0)), P.pp_epoch[P.dst]);
        } else if (threadIdx.x < p - 1) {
          const int d = (j + 1 + threadIdx.x) % p;
          signal(flag_ptr(P, d, cls, j, seg_of(k0)), ag ? P.epoch : P.pp_epoch[d]);
        }
      }
    }
    for (int q = 1; q < p; ++q) {
      const int i = (j - q + p) % p;
      if (!ag && i != P.root) continue;
      if (P.op == kFP2P && j != P.dst) continue;
      const uint32_t ep = ag ? P.epoch : P.pp_epoch[i];
      float* dst = ag ? P.out + static_cast<uint64_t>(i) * c : P.out;
      for (uint32_t k0 = 0; k0 < myseg; k0 += kStepSegs) {
        const uint32_t k1 = min(k0 + kStepSegs, myseg);
        seg_wait(P, flag_ptr(P, j, cls, i, seg_of(k0)), ep);
        for (uint32_t k = k0; k < k1; ++k) {
          const uint64_t g = static_cast<uint64_t>(seg_of(k)) * kSegGroups + warp;
          if (g < ngroups)
            fused_group<Codec, false, false>(P, slot_ptr(P, j, cls, i), nullptr, nullptr, dst, true, nullptr, g,
                                             sm, lane, bad);
        }
      }
      __syncthreads();
      ack_all(flag_ptr(P, i, ag ? 4 : 5, j, 0), ep);
    }
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

}  // namespace hccx
