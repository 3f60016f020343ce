// hcc_shim.cpp -- namespace hcc (the reference's C++ host API) over the C ABI
// of libhccx.so.  Pure host code: validation, exception mapping, byte
// accounting and the container format live here; every value computation is
// a call into include/hccx.h (sm_100a kernels).
//
// Reference behaviour mirrored (paths relative to /root/reference/proj):
//   CodecSpec / strings ............ src/codec.cpp:11-45
//   size law / container ........... src/codec.cpp:47-121
//   collectives + TraceEvent ........ src/collectives.cpp:113-248
//   SimClock ........................ src/netsim.cpp:77-106 (clock only)
//   layout + scheme builders ........ src/parallel3d.cpp:7-122
#include <algorithm>
#include <cstring>
#include <mutex>
#include <utility>

#include "hcc/hcc_b200.hpp"
#include "hcc/rng.hpp"
#include "hccx.h"

namespace hcc {

namespace {

int g_device = 0;

[[noreturn]] void raise(hccx_status_t st, const std::string& what) {
  const std::string msg = what + ": " + hccx_status_string(st);
  switch (st) {
    case HCCX_ERR_NONFINITE: throw NonFiniteInputError(msg);
    case HCCX_ERR_CORRUPT_PAYLOAD: throw CorruptPayloadError(msg);
    case HCCX_ERR_DATA_DEPENDENT_SIZE: throw DataDependentSizeError(msg);
    case HCCX_ERR_BAD_CHUNKING: throw BadChunkingError(msg);
    case HCCX_ERR_BAD_LAYOUT: throw BadLayoutError(msg);
    case HCCX_ERR_INVALID_SCHEME: throw InvalidSchemeError(msg);
    case HCCX_ERR_CONFIG: throw ConfigError("codec", msg);
    default: throw Error(msg);
  }
}

void check(hccx_status_t st, const std::string& what) {
  if (st != HCCX_OK) raise(st, what);
}

hccx_codec_t c_of(const CodecSpec& s) { return hccx_codec_t{static_cast<int32_t>(s.kind), s.rate_bits}; }

bool lossless(const CodecSpec& s) { return s.kind == CodecKind::LosslessPredictor; }

// Wire bytes of a ring collective: the size law, or under LosslessPredictor
// the device-sized hop messages (hccx_lossless_ring_wire).
std::uint64_t ring_wire(const CodecSpec& spec, const std::vector<const float*>& in, std::uint64_t n, int collective,
                        std::uint64_t law_msgs, std::uint64_t law_n) {
  if (!lossless(spec)) return law_msgs * wire_size_bytes(spec, law_n);
  std::uint64_t w = 0;
  check(hccx_lossless_ring_wire_host(in.data(), static_cast<int>(in.size()), n, collective, &w, g_device),
        "lossless wire accounting");
  return w;
}

std::uint64_t message_wire(const CodecSpec& spec, const FloatBuffer& buf) {
  if (!lossless(spec)) return wire_size_bytes(spec, buf.size());
  const float* two[2] = {buf.data(), buf.data()};
  std::uint64_t w = 0;  // allgather over 2 members = one hop of this buffer
  check(hccx_lossless_ring_wire_host(two, 2, buf.size(), 1, &w, g_device), "lossless wire accounting");
  return w / 2;
}

// one device group per communicator size, created on first use
hccx_group_t group_for(int p) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, hccx_group_t> groups;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(p, g_device);
  auto it = groups.find(key);
  if (it != groups.end()) return it->second;
  hccx_group_t g = nullptr;
  check(hccx_group_create(p, g_device, &g), "group_create");
  groups.emplace(key, g);
  return g;
}

std::vector<const float*> cptrs(const std::vector<FloatBuffer>& v) {
  std::vector<const float*> out;
  for (const auto& b : v) out.push_back(b.data());
  return out;
}

std::vector<float*> mptrs(std::vector<FloatBuffer>& v) {
  std::vector<float*> out;
  for (auto& b : v) out.push_back(b.data());
  return out;
}

// src/collectives.cpp:113-126
void commit(SimClock& clock, const Communicator& comm, double dur, std::uint64_t raw_total,
            std::uint64_t wire_total, int rounds, CommPath path, CollectiveKind kind) {
  clock.sync_to_max(comm.ranks);
  for (int r : comm.ranks) clock.advance(r, dur);
  const auto p = static_cast<std::uint64_t>(comm.size());
  TraceEvent e;
  e.path = path;
  e.collective = kind;
  e.comm_size = comm.size();
  e.raw_bytes = raw_total / p;
  e.wire_bytes = wire_total / p;
  e.duration_s = dur;
  e.round_count = rounds;
  clock.record(e);
}

// std::stoi with the reference's error mapping (src/codec.cpp:31-45)
int parse_rate(const std::string& s, const std::string& field, const std::string& whole) {
  try {
    return std::stoi(s);
  } catch (const std::exception&) {
    throw ConfigError(field, "bad rate in '" + whole + "'");
  }
}

}  // namespace

void set_device(int device) { g_device = device; }

// ------------------------------------------------------------------ codec --

CodecSpec CodecSpec::fixed_rate(int bits) {
  if (bits < 2 || bits > 32) throw InvalidSchemeError("fixed-rate bits must be in [2, 32], got " + std::to_string(bits));
  return {CodecKind::FixedRate, bits};
}

CodecSpec CodecSpec::zfp_rate(int bits) {
  if (bits < 3 || bits > 32) throw InvalidSchemeError("zfp-rate bits must be in [3, 32], got " + std::to_string(bits));
  return {CodecKind::ZfpRate, bits};
}

std::string to_string(const CodecSpec& spec) {
  switch (spec.kind) {
    case CodecKind::Identity: return "identity";
    case CodecKind::LosslessPredictor: return "lossless";
    case CodecKind::FixedRate: return "fixed-rate:" + std::to_string(spec.rate_bits);
    case CodecKind::ZfpRate: return "zfp-rate:" + std::to_string(spec.rate_bits);
  }
  return "unknown";
}

CodecSpec codec_spec_from_string(const std::string& s) {
  if (s == "identity") return CodecSpec::identity();
  if (s == "lossless") return CodecSpec::lossless();
  if (s.rfind("fixed-rate:", 0) == 0) return CodecSpec::fixed_rate(parse_rate(s.substr(11), "codec", s));
  if (s.rfind("zfp-rate:", 0) == 0) return CodecSpec::zfp_rate(parse_rate(s.substr(9), "codec", s));
  throw ConfigError("codec", "unknown codec '" + s + "' (expected identity | lossless | fixed-rate:N | zfp-rate:N)");
}

std::uint64_t wire_size_bytes(const CodecSpec& spec, std::uint64_t n) {
  std::uint64_t out = 0;
  check(hccx_wire_size_bytes(c_of(spec), n, &out), "wire_size_bytes");
  return out;
}

CompressedBuffer compress(const CodecSpec& spec, const FloatBuffer& buf) {
  check(hccx_codec_validate(c_of(spec)), "compress");
  CompressedBuffer out;
  out.codec = spec;
  out.original_len = buf.size();
  std::uint64_t cc = 0;
  check(hccx_chunk_count(c_of(spec), buf.size(), &cc), "compress");
  out.chunk_count = static_cast<std::uint32_t>(cc);
  if (lossless(spec)) {  // data-dependent size (codec_serial.cpp:42-55)
    out.payload.resize(hccx_lossless_max_bytes(buf.size()));
    std::uint64_t nb = 0;
    if (!buf.empty())
      check(hccx_lossless_compress_host(buf.data(), buf.size(), out.payload.data(), out.payload.size(), &nb,
                                        g_device),
            "compress");
    out.payload.resize(nb);
    return out;
  }
  out.payload.resize(wire_size_bytes(spec, buf.size()));
  if (!buf.empty())
    check(hccx_compress_host(c_of(spec), buf.data(), buf.size(), out.payload.data(), g_device), "compress");
  return out;
}

FloatBuffer decompress(const CompressedBuffer& cbuf) {
  std::uint64_t cc = 0;
  check(hccx_chunk_count(c_of(cbuf.codec), cbuf.original_len, &cc), "decompress");
  if (lossless(cbuf.codec)) {  // codec_serial.cpp:85-107
    if (cbuf.chunk_count != cc || cbuf.payload.size() < (cc + 7) / 8)
      throw CorruptPayloadError("predictor payload header mismatch");
    FloatBuffer out(cbuf.original_len);
    if (!out.empty())
      check(hccx_lossless_decompress_host(cbuf.payload.data(), cbuf.payload.size(), out.size(), out.data(), g_device),
            "decompress");
    return out;
  }
  if (cbuf.codec.kind != CodecKind::Identity && cbuf.chunk_count != cc)
    throw CorruptPayloadError("payload does not match block count");
  if (cbuf.payload.size() != wire_size_bytes(cbuf.codec, cbuf.original_len))
    throw CorruptPayloadError("payload size does not match the codec's size law");
  FloatBuffer out(cbuf.original_len);
  if (!out.empty())
    check(hccx_decompress_host(c_of(cbuf.codec), cbuf.payload.data(), cbuf.payload.size(), out.size(), out.data(),
                               g_device),
          "decompress");
  return out;
}

namespace serial {
CompressedBuffer compress(const CodecSpec& spec, const FloatBuffer& buf) { return hcc::compress(spec, buf); }
FloatBuffer decompress(const CompressedBuffer& cbuf) { return hcc::decompress(cbuf); }
}  // namespace serial

// "HCC1" | kind u8 | rate u8 | original_len u64 LE | chunk_count u32 LE | payload
std::vector<std::uint8_t> to_bytes(const CompressedBuffer& cbuf) {
  std::vector<std::uint8_t> out{'H', 'C', 'C', '1', static_cast<std::uint8_t>(cbuf.codec.kind),
                                static_cast<std::uint8_t>(cbuf.codec.rate_bits)};
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<std::uint8_t>(cbuf.original_len >> (8 * i)));
  for (int i = 0; i < 4; ++i) out.push_back(static_cast<std::uint8_t>(cbuf.chunk_count >> (8 * i)));
  out.insert(out.end(), cbuf.payload.begin(), cbuf.payload.end());
  return out;
}

CompressedBuffer from_bytes(const std::vector<std::uint8_t>& b) {
  if (b.size() < kContainerHeaderBytes) throw CorruptPayloadError("container shorter than header");
  if (!(b[0] == 'H' && b[1] == 'C' && b[2] == 'C' && b[3] == '1')) throw CorruptPayloadError("bad container magic");
  if (b[4] > 3) throw CorruptPayloadError("bad codec kind byte");
  CompressedBuffer c;
  c.codec.kind = static_cast<CodecKind>(b[4]);
  c.codec.rate_bits = b[5];
  if (c.codec.kind == CodecKind::FixedRate && (c.codec.rate_bits < 2 || c.codec.rate_bits > 32))
    throw CorruptPayloadError("bad fixed-rate bits in header");
  if (c.codec.kind == CodecKind::ZfpRate && (c.codec.rate_bits < 3 || c.codec.rate_bits > 32))
    throw CorruptPayloadError("bad zfp-rate bits in header");
  for (int i = 0; i < 8; ++i) c.original_len |= static_cast<std::uint64_t>(b[6 + i]) << (8 * i);
  for (int i = 0; i < 4; ++i) c.chunk_count |= static_cast<std::uint32_t>(b[14 + i]) << (8 * i);
  c.payload.assign(b.begin() + kContainerHeaderBytes, b.end());
  return c;
}

// -------------------------------------------------------------- comm path --

const char* to_string(CommPath p) {
  switch (p) {
    case CommPath::DpAllReduce: return "DpAllReduce";
    case CommPath::PpP2p: return "PpP2p";
    case CommPath::TpAllReduce: return "TpAllReduce";
    case CommPath::TpAllGather: return "TpAllGather";
    case CommPath::Zero1AllGather: return "Zero1AllGather";
    case CommPath::Zero1ReduceScatter: return "Zero1ReduceScatter";
  }
  return "unknown";
}

CommPath comm_path_from_string(const std::string& s) {
  for (CommPath p : kAllCommPaths)
    if (s == to_string(p)) return p;
  throw ConfigError("path", "unknown communication path '" + s + "'");
}

const char* to_string(CollectiveKind c) {
  switch (c) {
    case CollectiveKind::AllReduce: return "AllReduce";
    case CollectiveKind::AllGather: return "AllGather";
    case CollectiveKind::ReduceScatter: return "ReduceScatter";
    case CollectiveKind::P2P: return "P2P";
    case CollectiveKind::Broadcast: return "Broadcast";
  }
  return "unknown";
}

// ------------------------------------------------------------ topology --

Topology Topology::lassen_like(int n) { return Topology{n, 4, 75.0e9, 12.5e9, 2.0e-6, 5.0e-6, 400.0e9, 7.0e12}; }
Topology Topology::desk_2x2(int n) { return Topology{n, 2, 16.0e9, 1.25e9, 5.0e-6, 20.0e-6, 50.0e9, 1.0e12}; }
Topology Topology::b200_box(int g) { return Topology{1, g, 900.0e9, 900.0e9, 2.0e-6, 2.0e-6, 0.0, 0.0}; }
Topology Topology::preset(const std::string& name, int n) {
  if (name == "lassen-like") return lassen_like(n);
  if (name == "desk-2x2") return desk_2x2(n);
  if (name == "b200-box") return b200_box(8 * n);
  throw ConfigError("topology.preset", "unknown preset '" + name + "'");
}

double SimClock::max_time() const { return clock_.empty() ? 0.0 : *std::max_element(clock_.begin(), clock_.end()); }

void SimClock::advance(int rank, double dt) {
  if (dt < 0) throw Error("SimClock::advance: negative dt");
  clock_.at(rank) += dt;
}

void SimClock::sync_to_max(std::span<const int> ranks) {
  double t = 0.0;
  for (int r : ranks) t = std::max(t, clock_.at(r));
  for (int r : ranks) clock_.at(r) = t;
}

void SimClock::record(TraceEvent e) {
  e.step = step_;
  trace_.push_back(e);
}

void write_trace_csv(std::ostream& os, const std::vector<TraceEvent>& trace) {
  os << "step,path,collective,comm_size,raw_bytes,wire_bytes,duration_s\n";
  char buf[64];
  for (const auto& e : trace) {
    std::snprintf(buf, sizeof(buf), "%.9e", e.duration_s);
    os << e.step << ',' << to_string(e.path) << ',' << to_string(e.collective) << ',' << e.comm_size << ','
       << e.raw_bytes << ',' << e.wire_bytes << ',' << buf << '\n';
  }
}

// ------------------------------------------------------------ collectives --

FloatBuffer p2p(SimClock& clock, int src, int dst, const FloatBuffer& buf, const CodecSpec& spec, CommPath path) {
  if (src == dst) throw Error("p2p: src == dst");
  const std::uint64_t n = buf.size();
  const std::uint64_t wire = message_wire(spec, buf);
  FloatBuffer out(n);
  double dur = 0.0;
  if (n) check(hccx_group_p2p_host(group_for(2), buf.data(), out.data(), n, c_of(spec), &dur), "p2p");
  const int pair[2] = {src, dst};
  clock.sync_to_max(pair);
  clock.advance(src, dur);
  clock.advance(dst, dur);
  TraceEvent e;
  e.path = path;
  e.collective = CollectiveKind::P2P;
  e.comm_size = 2;
  e.raw_bytes = 4 * n;
  e.wire_bytes = wire;
  e.duration_s = dur;
  e.round_count = 1;
  clock.record(e);
  return out;
}

std::vector<FloatBuffer> ring_reduce_scatter(SimClock& clock, const Communicator& comm,
                                             const std::vector<FloatBuffer>& inputs, const CodecSpec& spec,
                                             CommPath path) {
  const int p = comm.size();
  if (p < 1 || static_cast<int>(inputs.size()) != p) throw Error("reduce_scatter: one input per member");
  const std::size_t n = inputs[0].size();
  if (n % p != 0)
    throw BadChunkingError("reduce_scatter: length " + std::to_string(n) + " not divisible by " + std::to_string(p));
  for (const auto& b : inputs)
    if (b.size() != n) throw BadChunkingError("reduce_scatter: ragged inputs");
  if (p == 1) return {inputs[0]};
  const std::uint64_t c = n / p;
  std::vector<FloatBuffer> shards(p, FloatBuffer(c));
  auto in = cptrs(inputs);
  auto out = mptrs(shards);
  double dur = 0.0;
  check(hccx_group_reduce_scatter_host(group_for(p), in.data(), out.data(), n, c_of(spec), &dur), "reduce_scatter");
  const std::uint64_t rounds = p - 1;
  commit(clock, comm, dur, rounds * p * 4 * c, ring_wire(spec, in, n, 0, rounds * p, c), p - 1,
         path, CollectiveKind::ReduceScatter);
  return shards;
}

std::vector<FloatBuffer> ring_allgather(SimClock& clock, const Communicator& comm,
                                        const std::vector<FloatBuffer>& shards, const CodecSpec& spec,
                                        CommPath path) {
  const int p = comm.size();
  if (p < 1 || static_cast<int>(shards.size()) != p) throw Error("allgather: one shard per member");
  const std::size_t c = shards[0].size();
  for (const auto& s : shards)
    if (s.size() != c) throw BadChunkingError("allgather: mismatched shard lengths");
  if (p == 1) return {shards[0]};
  std::vector<FloatBuffer> outs(p, FloatBuffer(c * p));
  auto in = cptrs(shards);
  auto out = mptrs(outs);
  double dur = 0.0;
  check(hccx_group_allgather_host(group_for(p), in.data(), out.data(), c, c_of(spec), &dur), "allgather");
  const std::uint64_t rounds = p - 1;
  commit(clock, comm, dur, rounds * p * 4 * c, ring_wire(spec, in, c, 1, rounds * p, c), p - 1,
         path, CollectiveKind::AllGather);
  return outs;
}

std::vector<FloatBuffer> allreduce(SimClock& clock, const Communicator& comm, const std::vector<FloatBuffer>& inputs,
                                   const CodecSpec& spec, CommPath path, ReduceMode mode) {
  const int p = comm.size();
  if (p < 1 || static_cast<int>(inputs.size()) != p) throw Error("allreduce: one input per member");
  const std::size_t n = inputs[0].size();
  if (n % p != 0)
    throw BadChunkingError("allreduce: length " + std::to_string(n) + " not divisible by " + std::to_string(p));
  for (const auto& b : inputs)
    if (b.size() != n) throw BadChunkingError("allreduce: ragged inputs");
  if (p == 1) return {inputs[0]};
  const std::uint64_t c = n / p;
  std::vector<FloatBuffer> outs(p, FloatBuffer(n));
  auto in = cptrs(inputs);
  auto out = mptrs(outs);
  double dur = 0.0;
  check(hccx_group_allreduce_host(group_for(p), in.data(), out.data(), n, c_of(spec),
                                  mode == ReduceMode::Average ? HCCX_AVERAGE : HCCX_SUM, &dur),
        "allreduce");
  const std::uint64_t rounds = p - 1;
  commit(clock, comm, dur, 2 * rounds * p * 4 * c, ring_wire(spec, in, n, 2, 2 * rounds * p, c),
         2 * (p - 1), path, CollectiveKind::AllReduce);
  return outs;
}

std::vector<FloatBuffer> broadcast(SimClock& clock, const Communicator& comm, int root, const FloatBuffer& buf,
                                   const CodecSpec& spec, CommPath path) {
  const int p = comm.size();
  if (root < 0 || root >= p) throw Error("broadcast: root out of range");
  if (p == 1) return {buf};
  const std::uint64_t n = buf.size();
  std::vector<FloatBuffer> outs(p, FloatBuffer(n));
  auto out = mptrs(outs);
  double dur = 0.0;
  if (n) check(hccx_group_broadcast_host(group_for(p), root, buf.data(), out.data(), n, c_of(spec), &dur), "broadcast");
  const std::uint64_t rounds = p - 1;
  commit(clock, comm, dur, rounds * 4 * n, rounds * message_wire(spec, buf), p - 1, path, CollectiveKind::Broadcast);
  return outs;
}

// ------------------------------------------------ layout and rate policy --

std::vector<int> ParallelLayout::dp_group(int rank) const {
  const Coord c = coord_of(rank);
  std::vector<int> out;
  for (int d = 0; d < dp; ++d) out.push_back(rank_of(d, c.p, c.t));
  return out;
}

std::vector<int> ParallelLayout::tp_group(int rank) const {
  const Coord c = coord_of(rank);
  std::vector<int> out;
  for (int t = 0; t < tp; ++t) out.push_back(rank_of(c.d, c.p, t));
  return out;
}

std::vector<int> ParallelLayout::pp_chain(int rank) const {
  const Coord c = coord_of(rank);
  std::vector<int> out;
  for (int s = 0; s < pp; ++s) out.push_back(rank_of(c.d, s, c.t));
  return out;
}

ParallelLayout build_layout(int dp, int pp, int tp, const Topology& topo) {
  if (dp < 1 || pp < 1 || tp < 1) throw BadLayoutError("parallel degrees must be >= 1");
  if (dp * pp * tp != topo.world_size())
    throw BadLayoutError("dp*pp*tp = " + std::to_string(dp * pp * tp) + " does not match world size " +
                         std::to_string(topo.world_size()));
  return ParallelLayout{dp, pp, tp};
}

SchemeTable scheme_no_compression() {
  SchemeTable t{"no-compression", {}};
  for (CommPath p : kAllCommPaths) t.paths[p] = CodecSpec::identity();
  return t;
}

SchemeTable scheme_naive(const CodecSpec& spec) {
  SchemeTable t;
  switch (spec.kind) {
    case CodecKind::Identity: t.name = "no-compression"; break;
    case CodecKind::LosslessPredictor: t.name = "naive-mpc"; break;
    case CodecKind::ZfpRate: t.name = "naive-zfpmode" + std::to_string(spec.rate_bits); break;
    default: t.name = "naive-zfp" + std::to_string(spec.rate_bits);
  }
  for (CommPath p : kAllCommPaths) t.paths[p] = spec;
  return t;
}

SchemeTable scheme_mz_hybrid(int dp_rate) {
  SchemeTable t{"mz-hybrid:" + std::to_string(dp_rate), {}};
  for (CommPath p : kAllCommPaths) t.paths[p] = CodecSpec::lossless();
  t.paths[CommPath::DpAllReduce] = CodecSpec::fixed_rate(dp_rate);
  return t;
}

SchemeTable scheme_z_hybrid(int mp_rate, int dp_rate) {
  if (mp_rate < dp_rate)
    throw InvalidSchemeError("z-hybrid requires mp_rate >= dp_rate, got mp=" + std::to_string(mp_rate) +
                             " dp=" + std::to_string(dp_rate));
  SchemeTable t{"z-hybrid:" + std::to_string(mp_rate) + "," + std::to_string(dp_rate), {}};
  for (CommPath p : kAllCommPaths) t.paths[p] = CodecSpec::fixed_rate(mp_rate);
  t.paths[CommPath::DpAllReduce] = CodecSpec::fixed_rate(dp_rate);
  return t;
}

SchemeTable scheme_from_name(const std::string& name) {
  if (name == "baseline" || name == "no-compression") return scheme_no_compression();
  if (name == "naive-mpc") return scheme_naive(CodecSpec::lossless());
  if (name.rfind("naive-zfp", 0) == 0) return scheme_naive(CodecSpec::fixed_rate(parse_rate(name.substr(9), "scheme", name)));
  if (name.rfind("mz-hybrid:", 0) == 0) return scheme_mz_hybrid(parse_rate(name.substr(10), "scheme", name));
  if (name.rfind("z-hybrid:", 0) == 0) {
    const auto comma = name.find(',', 9);
    if (comma != std::string::npos)
      return scheme_z_hybrid(parse_rate(name.substr(9, comma - 9), "scheme", name),
                             parse_rate(name.substr(comma + 1), "scheme", name));
  }
  throw ConfigError("scheme", "unknown scheme '" + name +
                                  "' (expected baseline | no-compression | naive-mpc | naive-zfpN | mz-hybrid:D | "
                                  "z-hybrid:M,D)");
}

}  // namespace hcc

// Synthetic inputs for the bench / tools: the reference's hcc::Rng streams
// (include/hcc/rng.hpp), so the GPU and the CPU reference see the same
// buffers for a seed.  mode 0: lo * normal() (the gradient-like bench input,
// lo = 1e-3); mode 1: uniform(lo, hi).
extern "C" __attribute__((visibility("default"))) void hcc_b200_fill(std::uint64_t seed, int mode, std::uint64_t n,
                                                                    float lo, float hi, float* out) {
  hcc::Rng rng(seed);
  if (mode == 1) {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.uniform(lo, hi);
  } else {
    for (std::uint64_t i = 0; i < n; ++i) out[i] = lo * rng.normal();
  }
}
