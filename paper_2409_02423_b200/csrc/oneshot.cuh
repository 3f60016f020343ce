// oneshot.cuh -- latency path of the NVLink allreduce for small messages.
//
// The ring (ring_fused.cuh) needs 2(p-1) dependent cross-GPU rounds, each a
// push + system-scope release + remote acquire, so a 4 KiB allreduce costs
// tens of microseconds at p = 4.  The one-shot path keeps the reference's
// arithmetic bit for bit (src/collectives.cpp:27-66 fold, :69-111 gather)
// with two rounds:
//
//   A  scatter: rank j stores its raw fp32 chunk d into rank d's raw slot
//      t = (j - d - 1) mod p (t = the hop at which the ring would have folded
//      it in), for every d != j;
//   B  the owner of chunk j replays the ring chain of its chunk locally, in
//      the ring's order and rounding:
//          S_0 = x[j+1][j];  m = Q(S_0)
//          S_t = dec(m) + x[j+1+t][j];  m = Q(S_t)    t = 1 .. p-1
//      (x[j+p] = its own chunk), keeps dec(m) (/p for Average) as its shard
//      and stores the final payload m into every peer's gather slot j;
//   C  every rank decodes the p-1 gathered payloads into its output.
//
// Two transports, chosen per call by size (comm.cu use_oneshot):
//
// Pair mode, the small end -- flag-in-data (the LL idea of NCCL's low-latency protocol): every 4-byte
// word crosses NVLink as an 8-byte (word, epoch) pair in one store (raw
// values go two pairs per 16-byte store), and the reader polls the pairs themselves until each
// carries this call's epoch -- no system-scope fence, no separate flag, no
// acquire round trip per step.  The wire carries twice the bytes, the right
// trade below a few MiB where latency, not bandwidth, is the cost.
//
// Flag mode, the upper end: raw words and payload bytes as they are, one
// system-scope release per CTA and phase (half the wire bytes).  The two
// modes use separate window regions, so calls may alternate freely.
//
// Only the wire traffic differs from the ring: (p-1) raw chunks out per rank
// instead of p-1 compressed ones.  Slot reuse needs no acks: a rank reaches
// the next call's phase A only after its phase C saw every peer's phase-B
// words for its range, which each peer wrote after consuming the raw words
// of that range, and a peer's gather slot is rewritten only after that peer
// has started the next call (its phase A), i.e. finished decoding this one.
// Epochs never repeat within 2^32 calls, so a stale pair never validates.
#pragma once

#include "ring_fused.cuh"

namespace hccx {

constexpr int kOsWarps = 8;

__device__ __forceinline__ void st_ll2(uint4* dst, uint32_t w0, uint32_t w1, uint32_t epoch) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(w0), "r"(epoch), "r"(w1),
               "r"(epoch)
               : "memory");
}

__device__ __forceinline__ void st_ll1(uint2* dst, uint32_t w, uint32_t epoch) {
  asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(dst), "r"(w), "r"(epoch) : "memory");
}

__device__ __forceinline__ uint2 ld_ll1(const uint2* src) {
  uint2 v;
  asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(src) : "memory");
  return v;
}

__device__ __forceinline__ uint2 wait_ll1(const FusedParams& P, const uint2* src, uint32_t epoch) {
  uint2 v = ld_ll1(src);
  if (v.y == epoch) return v;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t spins = 1;; ++spins) {
    v = ld_ll1(src);
    if (v.y == epoch) return v;
    if ((spins & 255u) == 0) {
      if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return v;
      if (globaltimer_ns() - t0 > P.timeout_ns) {
        if (P.err) atomicOr(P.err, kErrTimeout);
        return v;
      }
    }
  }
}

__device__ __forceinline__ uint4 ld_ll2(const uint4* src) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(src)
               : "memory");
  return v;
}

// Poll a pair-of-pairs until both carry `epoch` (bounded by the timeout;
// after a timeout, or once another wait of this rank timed out, the stale
// words are returned and the error word says so).
__device__ __forceinline__ uint4 wait_ll2(const FusedParams& P, const uint4* src, uint32_t epoch, bool need_hi) {
  uint4 v = ld_ll2(src);
  if (v.y == epoch && (!need_hi || v.w == epoch)) return v;
  const uint64_t t0 = globaltimer_ns();
  for (uint32_t spins = 1;; ++spins) {
    v = ld_ll2(src);
    if (v.y == epoch && (!need_hi || v.w == epoch)) return v;
    if ((spins & 255u) == 0) {
      if (P.err && (ldg_u32_coherent(P.err) & kErrTimeout)) return v;
      if (globaltimer_ns() - t0 > P.timeout_ns) {
        if (P.err) atomicOr(P.err, kErrTimeout);
        return v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Flag mode, for the upper end of the one-shot range: raw fp32 words and
// plain payload bytes (half the wire bytes of the pair mode), published per
// CTA with a system-scope release and waited for with acquire loads.
__device__ __forceinline__ uint32_t* os_flag(const FusedParams& P, int rank, int kind, int slot, uint32_t idx) {
  return reinterpret_cast<uint32_t*>(P.win[rank] + P.os_flag_off) +
         (static_cast<uint64_t>(kind) * P.p + slot) * kAckIdx + idx;
}

template <class Codec>
__device__ __forceinline__ void oneshot_flags_body(const FusedParams& P, const uint32_t cta, const uint32_t G) {
  __shared__ __align__(16) uint8_t stage[kOsWarps][kStageBytes];
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const int p = P.p, j = P.rank;
  const uint64_t c = P.n_chunk;
  const uint64_t GB = Codec::kGroupBytes;
  const uint64_t wire = Codec::wire_bytes(c);
  const uint64_t gc = (c + kGroupVals - 1) / kGroupVals;
  const uint64_t gpc = (gc + G - 1) / G;
  const uint64_t g0 = min(cta * gpc, gc), g1 = min(g0 + gpc, gc);
  const uint64_t v0 = min(g0 * kGroupVals, c), v1 = min(g1 * kGroupVals, c);
  const bool vec = P.vec_ok != 0;
  uint8_t* sm = stage[warp];
  uint32_t bad = 0;
  if constexpr (Codec::kNeedsInit) {
    Codec::kernel_init();
    __syncthreads();
  }
  auto raw_slot = [&](int rank, int t) {
    return reinterpret_cast<float*>(P.win[rank] + P.os_off + static_cast<uint64_t>(t) * P.os_raw_bytes);
  };
  auto ag_slot = [&](int rank, int src) {
    return P.win[rank] + P.os_ag_off + static_cast<uint64_t>(src) * P.os_ag_bytes;
  };

  // ---- A: raw scatter of this CTA's value range of every peer's chunk
  for (int q = 1; q < p; ++q) {
    const int d = (j + q) % p;
    const int t = (j - d - 1 + 2 * p) % p;
    const float* src = P.in + static_cast<uint64_t>(d) * c;
    float* dst = raw_slot(d, t);
    if (vec) {
      for (uint64_t i = v0 / 4 + threadIdx.x; i < v1 / 4; i += blockDim.x)
        reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
      for (uint64_t i = (v1 / 4) * 4 + threadIdx.x; i < v1; i += blockDim.x) dst[i] = src[i];
    } else {
      for (uint64_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) dst[i] = src[i];
    }
  }
  __syncthreads();  // every thread's stores precede the releases below (bar.sync + release cumulativity)
  if (threadIdx.x < static_cast<unsigned>(p - 1)) {
    const int d = (j + 1 + static_cast<int>(threadIdx.x)) % p;
    signal(os_flag(P, d, 0, (j - d - 1 + 2 * p) % p, cta), P.epoch);
  }

  // ---- B: replay the ring chain of chunk j for this CTA's groups
  if (threadIdx.x < static_cast<unsigned>(p - 1)) spin_ge(P, os_flag(P, j, 0, threadIdx.x, cta), P.epoch, 0xb00u);
  __syncthreads();
  for (uint64_t g = g0 + warp; g < g1; g += kOsWarps) {
    const uint64_t base = g * kGroupVals;
    const uint32_t live = static_cast<uint32_t>(c - base < kGroupVals ? c - base : kGroupVals);
    const uint32_t ll = lane_live(live, lane);
    typename Codec::Lane s;
    float v[8], loc[8];
    load_vals<false>(raw_slot(j, 0), base, live, true, lane, v);
    Codec::encode(v, s, bad, ll);
    for (int t = 1; t < p; ++t) {
      Codec::decode(s, v);
      const float* x = t < p - 1 ? raw_slot(j, t) : P.in + static_cast<uint64_t>(j) * c;
      load_vals<false>(x, base, live, t < p - 1 ? true : vec, lane, loc);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], loc[i]);  // arriving partial on the left
      Codec::encode(v, s, bad, ll);
    }
    Codec::decode(s, v);
    apply_div(v, P.div_mode, P.recip, P.divisor);
    store_vals(P.out + static_cast<uint64_t>(j) * c, base, live, vec, lane, v);
    // final payload -> every peer's gather slot j (4-byte stores; group
    // offsets are 4-byte multiples, the buffer's last group may end mid-word)
    Codec::to_stage(s, sm, lane);
    __syncwarp();
    const uint32_t nb = static_cast<uint32_t>(min(GB, wire - g * GB));
    for (int q = 1; q < p; ++q) {
      uint8_t* dst = ag_slot((j + q) % p, j) + g * GB;
      for (uint32_t w = lane; w < nb / 4; w += 32)
        reinterpret_cast<uint32_t*>(dst)[w] = reinterpret_cast<const uint32_t*>(sm)[w];
      for (uint32_t b = (nb / 4) * 4 + lane; b < nb; b += 32) dst[b] = sm[b];
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < static_cast<unsigned>(p - 1)) {
    const int d = (j + 1 + static_cast<int>(threadIdx.x)) % p;
    signal(os_flag(P, d, 1, j, cta), P.epoch);
  }

  // ---- C: decode every peer's shard (this CTA's groups of it)
  if (threadIdx.x < static_cast<unsigned>(p - 1)) {
    const int src = (j + 1 + static_cast<int>(threadIdx.x)) % p;
    spin_ge(P, os_flag(P, j, 1, src, cta), P.epoch, 0xc00u);
  }
  __syncthreads();
  for (int q = 1; q < p; ++q) {
    const int src = (j + q) % p;
    const uint8_t* pay = ag_slot(j, src);
    for (uint64_t g = g0 + warp; g < g1; g += kOsWarps) {
      const uint64_t base = g * kGroupVals;
      const uint32_t live = static_cast<uint32_t>(c - base < kGroupVals ? c - base : kGroupVals);
      typename Codec::Lane s;
      float v[8];
      group_load<Codec, false>(s, pay + g * GB, live, true, sm, lane);
      Codec::decode(s, v);
      apply_div(v, P.div_mode, P.recip, P.divisor);
      store_vals(P.out + static_cast<uint64_t>(src) * c, base, live, vec, lane, v);
    }
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

// ---------------------------------------------------------------------------
// Pair (LL) mode.
template <class Codec>
__device__ __forceinline__ void oneshot_ll_body(const FusedParams& P, const uint32_t cta, const uint32_t G) {
  __shared__ __align__(16) uint8_t stage[kOsWarps][kStageBytes];
  const int lane = static_cast<int>(lane_id()), warp = static_cast<int>(threadIdx.x >> 5);
  const int p = P.p, j = P.rank;
  const uint64_t c = P.n_chunk;
  const uint64_t GB = Codec::kGroupBytes;
  const uint64_t wire = Codec::wire_bytes(c);
  const uint64_t gc = (c + kGroupVals - 1) / kGroupVals;
  const uint64_t gpc = (gc + G - 1) / G;
  const uint64_t g0 = min(cta * gpc, gc), g1 = min(g0 + gpc, gc);
  const uint64_t v0 = min(g0 * kGroupVals, c), v1 = min(g1 * kGroupVals, c);
  const bool vec = P.vec_ok != 0;
  const uint32_t ep = P.epoch;
  uint8_t* sm = stage[warp];
  uint32_t bad = 0;
  if constexpr (Codec::kNeedsInit) {
    Codec::kernel_init();
    __syncthreads();
  }
  // raw slot t of `rank`: value i as the pair (bits, epoch) -> 8 bytes per value
  auto raw_slot = [&](int rank, int t) {
    return reinterpret_cast<uint4*>(P.win[rank] + P.os_ll_off + static_cast<uint64_t>(t) * P.os_ll_raw_bytes);
  };
  // gather slot of owner `src` at `rank`: payload word w as the pair (word,
  // epoch), one 8-byte store each (a group's words start at any word index)
  auto ag_slot = [&](int rank, int src) {
    return reinterpret_cast<uint2*>(P.win[rank] + P.os_ll_ag_off + static_cast<uint64_t>(src) * P.os_ll_ag_bytes);
  };

  // ---- A: raw scatter of this CTA's value range of every peer's chunk
  // (values in pairs: thread i stores values 2i, 2i+1 of the range)
  for (int q = 1; q < p; ++q) {
    const int d = (j + q) % p;
    const int t = (j - d - 1 + 2 * p) % p;
    const float* src = P.in + static_cast<uint64_t>(d) * c;
    uint4* dst = raw_slot(d, t);
    for (uint64_t i = v0 / 2 + threadIdx.x; 2 * i < v1; i += blockDim.x) {
      const uint32_t a = __float_as_uint(src[2 * i]);
      const uint32_t b = 2 * i + 1 < c ? __float_as_uint(src[2 * i + 1]) : 0u;
      st_ll2(dst + i, a, b, ep);
    }
  }

  // ---- B: replay the ring chain of chunk j for this CTA's groups
  for (uint64_t g = g0 + warp; g < g1; g += kOsWarps) {
    const uint64_t base = g * kGroupVals;
    const uint32_t live = static_cast<uint32_t>(c - base < kGroupVals ? c - base : kGroupVals);
    const uint32_t ll = lane_live(live, lane);
    typename Codec::Lane s;
    float v[8], loc[8];
    // this lane's 8 values of raw slot t: 4 pair-of-pairs, polled until valid
    auto load_raw = [&](int t, float (&o)[8]) {
      const uint4* r = raw_slot(j, t) + (base + 8 * lane) / 2;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (2u * k < ll) {
          const uint4 w = wait_ll2(P, r + k, ep, 2u * k + 1 < ll);
          o[2 * k] = __uint_as_float(w.x);
          o[2 * k + 1] = 2u * k + 1 < ll ? __uint_as_float(w.z) : 0.0f;
        } else {
          o[2 * k] = o[2 * k + 1] = 0.0f;
        }
      }
    };
    load_raw(0, v);
    Codec::encode(v, s, bad, ll);
    for (int t = 1; t < p; ++t) {
      Codec::decode(s, v);
      if (t < p - 1) {
        load_raw(t, loc);
      } else {
        load_vals<false>(P.in + static_cast<uint64_t>(j) * c, base, live, vec, lane, loc);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], loc[i]);  // arriving partial on the left
      Codec::encode(v, s, bad, ll);
    }
    Codec::decode(s, v);
    apply_div(v, P.div_mode, P.recip, P.divisor);
    store_vals(P.out + static_cast<uint64_t>(j) * c, base, live, vec, lane, v);
    // final payload -> every peer's gather slot j as (word, epoch) pairs;
    // the group's last bytes may end mid-word (zero padded)
    const uint32_t nb = static_cast<uint32_t>(min(GB, wire - g * GB));
    const uint32_t nw = (nb + 3) / 4;
    reinterpret_cast<uint32_t*>(sm)[nw > 0 ? nw - 1 : 0] = 0u;
    __syncwarp();
    Codec::to_stage(s, sm, lane);
    __syncwarp();
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(sm);
    const uint64_t wbase = g * GB / 4;  // GB is a multiple of 4 bytes
    for (int q = 1; q < p; ++q) {
      uint2* dst = ag_slot((j + q) % p, j) + wbase;
      for (uint32_t w = lane; w < nw; w += 32) st_ll1(dst + w, sw[w], ep);
    }
    __syncwarp();
  }

  // ---- C: decode every peer's shard (this CTA's groups of it)
  for (int q = 1; q < p; ++q) {
    const int src = (j + q) % p;
    const uint2* pay = ag_slot(j, src);
    for (uint64_t g = g0 + warp; g < g1; g += kOsWarps) {
      const uint64_t base = g * kGroupVals;
      const uint32_t live = static_cast<uint32_t>(c - base < kGroupVals ? c - base : kGroupVals);
      const uint32_t nb = static_cast<uint32_t>(min(GB, wire - g * GB));
      const uint32_t nw = (nb + 3) / 4;
      uint32_t* sw = reinterpret_cast<uint32_t*>(sm);
      const uint64_t wbase = g * GB / 4;
      for (uint32_t w = lane; w < nw; w += 32) sw[w] = wait_ll1(P, pay + wbase + w, ep).x;
      for (uint32_t w = nw + lane; w < GB / 4; w += 32) sw[w] = 0u;  // partial group: zero tail
      __syncwarp();
      typename Codec::Lane s;
      float v[8];
      Codec::from_stage(s, sm, lane);
      __syncwarp();
      Codec::decode(s, v);
      apply_div(v, P.div_mode, P.recip, P.divisor);
      store_vals(P.out + static_cast<uint64_t>(src) * c, base, live, vec, lane, v);
    }
  }
  if constexpr (Codec::kCheckFinite) {
    if (__any_sync(kFull, bad) && lane == 0 && P.err) atomicOr(P.err, kErrNonFinite);
  }
}

template <class Codec>
__device__ __forceinline__ void oneshot_body(const FusedParams& P, const uint32_t cta, const uint32_t G) {
  if (P.os_ll)
    oneshot_ll_body<Codec>(P, cta, G);
  else
    oneshot_flags_body<Codec>(P, cta, G);
}

template <class Codec>
__global__ void __launch_bounds__(kOsWarps * 32) oneshot_allreduce_kernel(const __grid_constant__ FusedParams P) {
  // launched with programmatic stream serialization (fused_launch.cuh): the
  // grid is scheduled while the previous kernel drains; nothing is touched
  // before that kernel has completed
  pdl_wait_and_release();
  oneshot_body<Codec>(P, blockIdx.x, gridDim.x);
}

// Virtual ranks (see ring_fused_vkernel): rank v = blockIdx.x / G.
template <class Codec>
__global__ void __launch_bounds__(kOsWarps * 32) oneshot_allreduce_vkernel(const __grid_constant__ VParams V) {
  const uint32_t v = blockIdx.x / V.G;
  oneshot_body<Codec>(V.r[v], blockIdx.x - v * V.G, V.G);
}

}  // namespace hccx
