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

// Collective members run on the NVLink engine's single-process communicator
// (include/hccx.h hccx_mcomm_*), one per member->GPU map, grown on demand.
std::vector<int>& device_list() {
  static std::vector<int> devs = [] {
    std::vector<int> d;
    if (const char* e = std::getenv("HCC_B200_DEVICES")) {
      std::string s(e);
      for (size_t pos = 0; pos < s.size();) {
        const size_t comma = s.find(',', pos);
        const std::string tok = s.substr(pos, comma == std::string::npos ? std::string::npos : comma - pos);
        if (!tok.empty()) d.push_back(std::stoi(tok));
        if (comma == std::string::npos) break;
        pos = comma + 1;
      }
    }
    if (d.empty()) {
      const int n = hccx_device_count();
      for (int i = 0; i < (n > 0 ? n : 1); ++i) d.push_back(i);
    }
    return d;
  }();
  return devs;
}


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

std::uint64_t message_wire(const CodecSpec& spec, const FloatBuffer& buf) {
  if (!lossless(spec)) return wire_size_bytes(spec, buf.size());
  const float* two[2] = {buf.data(), buf.data()};
  std::uint64_t w = 0;  // allgather over 2 members = one hop of this buffer
  check(hccx_lossless_ring_wire_host(two, 2, buf.size(), 1, &w, g_device), "lossless wire accounting");
  return w / 2;
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

// std::stoi with the reference's error mapping (src/codec.cpp:31-45)
int parse_rate(const std::string& s, const std::string& field, const std::string& whole) {
  try {
    return std::stoi(s);
  } catch (const std::exception&) {
    throw ConfigError(field, "bad rate in '" + whole + "'");
  }
}

}  // namespace

void set_device(int device) {
  g_device = device;
  device_list() = {device};
}
void set_devices(const std::vector<int>& devices) {
  if (devices.empty()) throw Error("set_devices: empty device list");
  g_device = devices[0];
  device_list() = devices;
}

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

void Topology::validate() const {
  auto need = [](bool ok, const char* field, const char* what) {
    if (!ok) throw ConfigError(field, what);
  };
  need(num_nodes >= 1, "topology.num_nodes", "must be >= 1");
  need(gpus_per_node >= 1, "topology.gpus_per_node", "must be >= 1");
  need(intra_bw > 0, "topology.intra_bw", "must be > 0");
  need(inter_bw > 0, "topology.inter_bw", "must be > 0");
  need(intra_lat > 0, "topology.intra_lat", "must be > 0");
  need(inter_lat > 0, "topology.inter_lat", "must be > 0");
  need(codec_bw > 0, "topology.codec_bw", "must be > 0");
  need(compute_flops > 0, "topology.compute_flops", "must be > 0");
}

Topology Topology::lassen_like(int n) { return Topology{n, 4, 75.0e9, 12.5e9, 2.0e-6, 5.0e-6, 400.0e9, 7.0e12}; }
Topology Topology::desk_2x2(int n) { return Topology{n, 2, 16.0e9, 1.25e9, 5.0e-6, 20.0e-6, 50.0e9, 1.0e12}; }
// codec_bw: fixed-rate r8 compress on one B200, 4.05e12 uncompressed B/s
// (bench.py N=1, profiles/r02_bench_n1.json); compute_flops: fp32 CUDA-core
// peak, 148 SMs x 128 lanes x 2 x 1.965 GHz (the toy trainer's matmuls are
// fp32); intra: NVLink 5, 900 GB/s per direction, ~2 us flag latency.
Topology Topology::b200_box(int g) { return Topology{1, g, 900.0e9, 900.0e9, 2.0e-6, 2.0e-6, 4.05e12, 74.4e12}; }
Topology Topology::preset(const std::string& name, int n) {
  if (name == "lassen-like") return lassen_like(n);
  if (name == "desk-2x2") return desk_2x2(n);
  if (name == "b200-box") return b200_box(8 * n);
  throw ConfigError("topology.preset", "unknown preset '" + name + "' (expected lassen-like | desk-2x2 | b200-box)");
}

LinkClass link_class(const Topology& topo, int a, int b) {
  if (a == b) return LinkClass::SelfLoop;
  return topo.node_of(a) == topo.node_of(b) ? LinkClass::IntraNode : LinkClass::InterNode;
}

double transfer_time(const Topology& topo, std::uint64_t bytes, LinkClass link) {
  if (link == LinkClass::SelfLoop) return 0.0;
  const bool intra = link == LinkClass::IntraNode;
  return (intra ? topo.intra_lat : topo.inter_lat) + static_cast<double>(bytes) / (intra ? topo.intra_bw : topo.inter_bw);
}

double codec_time(const Topology& topo, std::uint64_t raw_bytes, const CodecSpec& spec) {
  return spec.kind == CodecKind::Identity ? 0.0 : static_cast<double>(raw_bytes) / topo.codec_bw;
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

namespace {

std::vector<int> member_devices(const std::vector<int>& ranks) {
  const auto& devs = device_list();
  std::vector<int> out;
  for (int r : ranks) out.push_back(devs[static_cast<size_t>(r) % devs.size()]);
  return out;
}

hccx_mcomm_t mcomm_for(const std::vector<int>& devices, std::uint64_t max_n) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::pair<hccx_mcomm_t, std::uint64_t>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = cache[devices];
  if (slot.first && slot.second >= max_n) return slot.first;
  if (slot.first) hccx_mcomm_destroy(slot.first);
  slot = {nullptr, 0};
  const std::uint64_t cap = std::max<std::uint64_t>({max_n, 2 * slot.second, 1u << 16});
  hccx_mcomm_t m = nullptr;
  check(hccx_mcomm_create(static_cast<int>(devices.size()), devices.data(), cap, &m), "mcomm_create");
  slot = {m, cap};
  return m;
}

// The reference's per-collective cost record (src/collectives.cpp:9-14).
struct PhaseCost {
  double duration = 0;
  std::uint64_t raw_total = 0, wire_total = 0;
  int rounds = 0;
};

// Ring reduce-scatter cost (src/collectives.cpp:34-64): every round's
// duration is its slowest hop; msg(round, j) = payload member j sends.
template <class Msg>
PhaseCost rs_cost(const SimClock& clock, const Communicator& comm, const CodecSpec& spec, std::uint64_t chunk,
                  Msg&& msg) {
  const int p = comm.size();
  const std::uint64_t raw_msg = 4 * chunk;
  const Topology& t = clock.topology();
  PhaseCost cost;
  for (int round = 0; round < p - 1; ++round) {
    double round_dur = 0;
    for (int j = 0; j < p; ++j) {
      const std::uint64_t payload = msg(round, j);
      const double hop = codec_time(t, raw_msg, spec) +
                         transfer_time(t, payload, link_class(t, comm.ranks[j], comm.ranks[(j + 1) % p])) +
                         codec_time(t, raw_msg, spec);
      round_dur = std::max(round_dur, hop);
      cost.raw_total += raw_msg;
      cost.wire_total += payload;
    }
    cost.duration += round_dur;
  }
  cost.rounds = p - 1;
  return cost;
}

// Ring allgather cost (src/collectives.cpp:93-109): shard c, compressed once
// at its origin, forwarded by member j in round (j - c) mod p.
template <class Shard>
PhaseCost ag_cost(const SimClock& clock, const Communicator& comm, const CodecSpec& spec, std::uint64_t chunk,
                  Shard&& shard) {
  const int p = comm.size();
  const std::uint64_t raw_msg = 4 * chunk;
  const Topology& t = clock.topology();
  PhaseCost cost;
  for (int round = 0; round < p - 1; ++round) {
    double round_dur = 0;
    for (int j = 0; j < p; ++j) {
      const std::uint64_t payload = shard(((j - round) % p + p) % p);
      double hop = transfer_time(t, payload, link_class(t, comm.ranks[j], comm.ranks[(j + 1) % p])) +
                   codec_time(t, raw_msg, spec);
      if (round == 0) hop += codec_time(t, raw_msg, spec);
      round_dur = std::max(round_dur, hop);
      cost.raw_total += raw_msg;
      cost.wire_total += payload;
    }
    cost.duration += round_dur;
  }
  cost.rounds = p - 1;
  return cost;
}

// Per-message payload bytes: the size law, or the device-sized messages of
// the LosslessPredictor ring (hccx_lossless_ring_hops).
std::vector<std::uint64_t> lossless_hops(const std::vector<const float*>& in, std::uint64_t n, int collective) {
  const int p = static_cast<int>(in.size());
  std::vector<std::uint64_t> hop(static_cast<size_t>(p) * p + p, 0);
  check(hccx_lossless_ring_hops_host(in.data(), p, n, collective, hop.data(), g_device), "lossless wire accounting");
  return hop;
}

// src/collectives.cpp:113-126, plus the measured device time.
void commit(SimClock& clock, const Communicator& comm, const PhaseCost& cost, double device_s, CommPath path,
            CollectiveKind kind) {
  clock.sync_to_max(comm.ranks);
  for (int r : comm.ranks) clock.advance(r, cost.duration);
  const auto p = static_cast<std::uint64_t>(comm.size());
  TraceEvent e;
  e.path = path;
  e.collective = kind;
  e.comm_size = comm.size();
  e.raw_bytes = cost.raw_total / p;
  e.wire_bytes = cost.wire_total / p;
  e.duration_s = cost.duration;
  e.round_count = cost.rounds;
  e.device_s = device_s;
  clock.record(e);
}

void check_ranks(const SimClock& clock, const Communicator& comm, const char* what) {
  if (comm.ranks.empty()) throw Error(std::string(what) + ": empty communicator");
  for (int r : comm.ranks)
    if (r < 0 || r >= clock.topology().world_size()) throw Error(std::string(what) + ": rank out of range");
}

}  // namespace

FloatBuffer p2p(SimClock& clock, int src, int dst, const FloatBuffer& buf, const CodecSpec& spec, CommPath path) {
  if (src == dst) throw Error("p2p: src == dst");
  const std::uint64_t n = buf.size();
  const std::uint64_t wire = message_wire(spec, buf);
  FloatBuffer out(n);
  double dev_s = 0.0;
  if (n) {
    hccx_mcomm_t m = mcomm_for(member_devices({src, dst}), n);
    check(hccx_mcomm_p2p_host(m, 0, 1, buf.data(), out.data(), n, c_of(spec), &dev_s), "p2p");
  }
  // src/collectives.cpp:133-151
  const Topology& t = clock.topology();
  const std::uint64_t raw = 4 * n;
  const double dur = codec_time(t, raw, spec) + transfer_time(t, wire, link_class(t, src, dst)) +
                     codec_time(t, raw, spec);
  const int pair[2] = {src, dst};
  clock.sync_to_max(pair);
  clock.advance(src, dur);
  clock.advance(dst, dur);
  TraceEvent e;
  e.path = path;
  e.collective = CollectiveKind::P2P;
  e.comm_size = 2;
  e.raw_bytes = raw;
  e.wire_bytes = wire;
  e.duration_s = dur;
  e.round_count = 1;
  e.device_s = dev_s;
  clock.record(e);
  return out;
}

std::vector<FloatBuffer> ring_reduce_scatter(SimClock& clock, const Communicator& comm,
                                             const std::vector<FloatBuffer>& inputs, const CodecSpec& spec,
                                             CommPath path) {
  check_ranks(clock, comm, "reduce_scatter");
  const int p = comm.size();
  if (static_cast<int>(inputs.size()) != p) throw Error("reduce_scatter: one input per member");
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
  double dev_s = 0.0;
  hccx_mcomm_t m = mcomm_for(member_devices(comm.ranks), n);
  check(hccx_mcomm_reduce_scatter_host(m, in.data(), out.data(), n, c_of(spec), &dev_s), "reduce_scatter");
  PhaseCost cost;
  if (lossless(spec)) {
    const auto hop = lossless_hops(in, n, 0);
    cost = rs_cost(clock, comm, spec, c, [&](int r, int j) { return hop[static_cast<size_t>(r) * p + j]; });
  } else {
    const std::uint64_t w = wire_size_bytes(spec, c);
    cost = rs_cost(clock, comm, spec, c, [&](int, int) { return w; });
  }
  commit(clock, comm, cost, dev_s, path, CollectiveKind::ReduceScatter);
  return shards;
}

std::vector<FloatBuffer> ring_allgather(SimClock& clock, const Communicator& comm,
                                        const std::vector<FloatBuffer>& shards, const CodecSpec& spec,
                                        CommPath path) {
  check_ranks(clock, comm, "allgather");
  const int p = comm.size();
  if (static_cast<int>(shards.size()) != p) throw Error("allgather: one shard per member");
  const std::size_t c = shards[0].size();
  for (const auto& s : shards)
    if (s.size() != c) throw BadChunkingError("allgather: mismatched shard lengths");
  if (p == 1) return {shards[0]};
  std::vector<FloatBuffer> outs(p, FloatBuffer(c * p));
  auto in = cptrs(shards);
  auto out = mptrs(outs);
  double dev_s = 0.0;
  hccx_mcomm_t m = mcomm_for(member_devices(comm.ranks), c * p);
  check(hccx_mcomm_allgather_host(m, in.data(), out.data(), c, c_of(spec), &dev_s), "allgather");
  PhaseCost cost;
  if (lossless(spec)) {
    const auto hop = lossless_hops(in, c, 1);
    cost = ag_cost(clock, comm, spec, c, [&](int s) { return hop[s]; });
  } else {
    const std::uint64_t w = wire_size_bytes(spec, c);
    cost = ag_cost(clock, comm, spec, c, [&](int) { return w; });
  }
  commit(clock, comm, cost, dev_s, path, CollectiveKind::AllGather);
  return outs;
}

std::vector<FloatBuffer> allreduce(SimClock& clock, const Communicator& comm, const std::vector<FloatBuffer>& inputs,
                                   const CodecSpec& spec, CommPath path, ReduceMode mode) {
  check_ranks(clock, comm, "allreduce");
  const int p = comm.size();
  if (static_cast<int>(inputs.size()) != p) throw Error("allreduce: one input per member");
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
  double dev_s = 0.0;
  hccx_mcomm_t m = mcomm_for(member_devices(comm.ranks), n);
  check(hccx_mcomm_allreduce_host(m, in.data(), out.data(), n, c_of(spec),
                                  mode == ReduceMode::Average ? HCCX_AVERAGE : HCCX_SUM, &dev_s),
        "allreduce");
  // src/collectives.cpp:219-246: RS cost + AG cost of the reduced shards
  PhaseCost rs, ag;
  if (lossless(spec)) {
    const auto hop = lossless_hops(in, n, 2);
    const size_t nrs = static_cast<size_t>(p - 1) * p;
    rs = rs_cost(clock, comm, spec, c, [&](int r, int j) { return hop[static_cast<size_t>(r) * p + j]; });
    ag = ag_cost(clock, comm, spec, c, [&](int s) { return hop[nrs + s]; });
  } else {
    const std::uint64_t w = wire_size_bytes(spec, c);
    rs = rs_cost(clock, comm, spec, c, [&](int, int) { return w; });
    ag = ag_cost(clock, comm, spec, c, [&](int) { return w; });
  }
  PhaseCost total;
  total.duration = rs.duration + ag.duration;
  total.raw_total = rs.raw_total + ag.raw_total;
  total.wire_total = rs.wire_total + ag.wire_total;
  total.rounds = rs.rounds + ag.rounds;
  commit(clock, comm, total, dev_s, path, CollectiveKind::AllReduce);
  return outs;
}

std::vector<FloatBuffer> broadcast(SimClock& clock, const Communicator& comm, int root, const FloatBuffer& buf,
                                   const CodecSpec& spec, CommPath path) {
  check_ranks(clock, comm, "broadcast");
  const int p = comm.size();
  if (root < 0 || root >= p) throw Error("broadcast: root out of range");
  if (p == 1) return {buf};
  const std::uint64_t n = buf.size();
  std::vector<FloatBuffer> outs(p, FloatBuffer(n));
  auto out = mptrs(outs);
  double dev_s = 0.0;
  if (n) {
    hccx_mcomm_t m = mcomm_for(member_devices(comm.ranks), n);
    check(hccx_mcomm_broadcast_host(m, root, buf.data(), out.data(), n, c_of(spec), &dev_s), "broadcast");
  }
  // By analogy with the allgather of one shard: the
  // root's payload crosses p-1 ring hops.
  const std::uint64_t w = message_wire(spec, buf);
  const Topology& t = clock.topology();
  const std::uint64_t raw = 4 * n;
  PhaseCost cost;
  for (int round = 0; round < p - 1; ++round) {
    const int j = ((root + round) % p + p) % p;
    double hop = transfer_time(t, w, link_class(t, comm.ranks[j], comm.ranks[(j + 1) % p])) + codec_time(t, raw, spec);
    if (round == 0) hop += codec_time(t, raw, spec);
    cost.duration += hop;
    cost.raw_total += raw;
    cost.wire_total += w;
  }
  cost.rounds = p - 1;  // commit() reports the per-rank share (total / p), like the group accounting
  commit(clock, comm, cost, dev_s, path, CollectiveKind::Broadcast);
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
