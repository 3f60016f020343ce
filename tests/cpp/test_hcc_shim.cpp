// test_hcc_shim.cpp -- the reference's own C++ test cases, run against the
// B200 drop-in (libhcc_b200.so over libhccx.so).  Cases follow
// /root/reference/proj/tests/test_codec.cpp, test_collectives.cpp and
// test_parallel3d.cpp; expected values that need arithmetic come from the CPU
// oracle (oracle/hcc_oracle.c, TEST INFRASTRUCTURE, pinned to the reference).
// Needs a GPU.  Exit status 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "hcc/collectives.hpp"
#include "hcc/parallel3d.hpp"

extern "C" {
void orc_fill(uint64_t seed, int mode, uint64_t n, float lo, float hi, float* out);
int orc_fr_compress(int rate, const float* in, uint64_t n, uint8_t* out);
void orc_fr_decompress(int rate, const uint8_t* in, uint64_t n, float* out);
uint64_t orc_wire_size(int kind, int rate, uint64_t n);
int orc_allreduce(int p, uint64_t n, const float* inputs, int kind, int rate, int average, float* out, uint64_t* acct);
int orc_reduce_scatter(int p, uint64_t n, const float* inputs, int kind, int rate, float* shards, uint64_t* acct);
int orc_allgather(int p, uint64_t c, const float* shards, int kind, int rate, float* out, uint64_t* acct);
double orc_block_bound(const float* v, uint64_t n, int rate);
uint64_t orc_pred_size(const float* in, uint64_t n);
uint64_t orc_pred_compress(const float* in, uint64_t n, uint8_t* out);
int orc_p2p(uint64_t n, const float* in, int kind, int rate, float* out, uint64_t* acct);
}

using namespace hcc;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                            \
  do {                                                                         \
    if (cond) {                                                                \
      ++g_pass;                                                                \
    } else {                                                                   \
      ++g_fail;                                                                \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                          \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static FloatBuffer fill(uint64_t seed, int mode, size_t n, float lo = -1.f, float hi = 1.f) {
  FloatBuffer v(n);
  if (n) orc_fill(seed, mode, n, lo, hi, v.data());
  return v;
}

static bool bit_equal(const FloatBuffer& a, const FloatBuffer& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 4 * a.size()) == 0);
}

static double max_abs(const FloatBuffer& a, const FloatBuffer& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(double(a[i]) - double(b[i])));
  return m;
}

static Communicator comm_of(int p) {
  Communicator c;
  for (int i = 0; i < p; ++i) c.ranks.push_back(i);
  return c;
}

static std::vector<FloatBuffer> inputs(uint64_t seed, int p, size_t n) {
  std::vector<FloatBuffer> v;
  for (int j = 0; j < p; ++j) v.push_back(fill(seed + 31 * j, 2, n));
  return v;
}

static std::vector<float> flat(const std::vector<FloatBuffer>& v) {
  std::vector<float> f;
  for (const auto& b : v) f.insert(f.end(), b.begin(), b.end());
  return f;
}

static void test_codec() {
  // test_codec.cpp:25-39
  CHECK(!throws<Error>([] { CodecSpec::fixed_rate(2); }));
  CHECK(throws<InvalidSchemeError>([] { CodecSpec::fixed_rate(1); }));
  CHECK(throws<InvalidSchemeError>([] { CodecSpec::fixed_rate(33); }));
  for (auto s : {CodecSpec::identity(), CodecSpec::lossless(), CodecSpec::fixed_rate(8), CodecSpec::fixed_rate(24)})
    CHECK(codec_spec_from_string(to_string(s)) == s);
  CHECK(throws<ConfigError>([] { codec_spec_from_string("zfp"); }));
  CHECK(throws<InvalidSchemeError>([] { codec_spec_from_string("fixed-rate:99"); }));
  // identity round trip + golden container (test_codec.cpp:41-58)
  const FloatBuffer one = {1.0f, -2.5f, 3.75f};
  CHECK(bit_equal(decompress(compress(CodecSpec::identity(), one)), one));
  const auto bytes = to_bytes(compress(CodecSpec::identity(), {1.0f}));
  const std::vector<uint8_t> golden = {'H', 'C', 'C', '1', 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                       0x00, 0x00, 0x80, 0x3F};
  CHECK(bytes == golden);
  // rate 8 payload (test_codec.cpp:103-108) and wire law (:110-129)
  CHECK(compress(CodecSpec::fixed_rate(8), fill(14, 2, 1024, -4, 4)).payload_bytes() == 1040u);
  CHECK(wire_size_bytes(CodecSpec::identity(), 100) == 400u);
  CHECK(wire_size_bytes(CodecSpec::fixed_rate(16), 64) == 129u);
  CHECK(wire_size_bytes(CodecSpec::fixed_rate(8), 65) == 130u);
  CHECK(wire_size_bytes(CodecSpec::fixed_rate(8), 0) == 0u);
  CHECK(throws<DataDependentSizeError>([] { wire_size_bytes(CodecSpec::lossless(), 10); }));
  for (int rate : {2, 8, 16, 24, 32})
    for (size_t n : {size_t{0}, size_t{1}, size_t{63}, size_t{64}, size_t{65}, size_t{1000000}}) {
      const auto x = fill(15 + rate + n, 2, n);
      const auto cb = compress(CodecSpec::fixed_rate(rate), x);
      CHECK(cb.payload_bytes() == wire_size_bytes(CodecSpec::fixed_rate(rate), n));
      // byte-exact vs the oracle restatement of hcc::compress
      std::vector<uint8_t> want(cb.payload.size() + 1);
      CHECK(orc_fr_compress(rate, x.data(), n, want.data()) == 0);
      CHECK(std::memcmp(want.data(), cb.payload.data(), cb.payload.size()) == 0);
      const auto back = decompress(cb);
      FloatBuffer wback(n + 1);
      orc_fr_decompress(rate, cb.payload.data(), n, wback.data());
      wback.resize(n);
      CHECK(bit_equal(back, wback));
    }
  // rate 32 powers of two (test_codec.cpp:131-137)
  FloatBuffer pw;
  for (int i = 0; i < 64; ++i) pw.push_back(std::ldexp(1.0f, -(i % 8)));
  CHECK(max_abs(decompress(compress(CodecSpec::fixed_rate(32), pw)), pw) <= std::ldexp(1.0, -30));
  // random blocks within the bound (test_codec.cpp:148-158)
  for (int rate : {8, 16, 24, 32})
    for (int t = 0; t < 50; ++t) {
      const auto x = fill(17000 + rate * 100 + t, 1, 64);
      CHECK(max_abs(decompress(compress(CodecSpec::fixed_rate(rate), x)), x) <=
            orc_block_bound(x.data(), 64, rate));
    }
  // zeros / denormals (test_codec.cpp:174-185), non-finite (:187-195)
  const FloatBuffer zeros(130, 0.0f);
  CHECK(bit_equal(decompress(compress(CodecSpec::fixed_rate(8), zeros)), zeros));
  FloatBuffer bad(64, 1.0f);
  bad[10] = std::numeric_limits<float>::quiet_NaN();
  CHECK(throws<NonFiniteInputError>([&] { compress(CodecSpec::fixed_rate(8), bad); }));
  bad[10] = std::numeric_limits<float>::infinity();
  CHECK(throws<NonFiniteInputError>([&] { compress(CodecSpec::fixed_rate(8), bad); }));
  // container round trip + malformed (test_codec.cpp:197-240)
  const auto cb = compress(CodecSpec::fixed_rate(12), fill(19, 2, 500, -2, 2));
  const auto parsed = from_bytes(to_bytes(cb));
  CHECK(parsed.codec == cb.codec && parsed.original_len == cb.original_len && parsed.payload == cb.payload);
  auto b = to_bytes(cb);
  auto t = b;
  t.resize(10);
  CHECK(throws<CorruptPayloadError>([&] { from_bytes(t); }));
  t = b;
  t[0] = 'X';
  CHECK(throws<CorruptPayloadError>([&] { from_bytes(t); }));
  t = b;
  t[4] = 7;
  CHECK(throws<CorruptPayloadError>([&] { from_bytes(t); }));
  auto shortp = cb;
  shortp.payload.pop_back();
  CHECK(throws<CorruptPayloadError>([&] { decompress(shortp); }));
  auto badcount = cb;
  badcount.chunk_count += 1;
  CHECK(throws<CorruptPayloadError>([&] { decompress(badcount); }));
  // serial namespace is the same device path
  CHECK(serial::compress(CodecSpec::fixed_rate(8), pw).payload == compress(CodecSpec::fixed_rate(8), pw).payload);
  // zfp-mode codec (addition): round trip within a loose relative bound
  const auto g = fill(5, 4, 4096, 1e-3f);
  const auto zb = decompress(compress(CodecSpec::zfp_rate(16), g));
  CHECK(max_abs(zb, g) < 1e-5);
}

static void test_collectives() {
  // test_collectives.cpp:67-75, 162-175: two-rank examples
  {
    SimClock clk(Topology::lassen_like(2));
    const std::vector<FloatBuffer> in = {{1.0f, 2.0f}, {3.0f, 4.0f}};
    const auto rs = ring_reduce_scatter(clk, comm_of(2), in, CodecSpec::identity(), CommPath::DpAllReduce);
    CHECK(rs[0] == FloatBuffer{4.0f} && rs[1] == FloatBuffer{6.0f});
    const auto ar = allreduce(clk, comm_of(2), in, CodecSpec::identity(), CommPath::DpAllReduce);
    CHECK((ar[0] == FloatBuffer{4.0f, 6.0f}) && (ar[1] == FloatBuffer{4.0f, 6.0f}));
    const auto av = allreduce(clk, comm_of(2), in, CodecSpec::identity(), CommPath::DpAllReduce, ReduceMode::Average);
    CHECK((av[0] == FloatBuffer{2.0f, 3.0f}));
  }
  // bit-exact vs the oracle for p in {2,3,4,8}, identity and fixed-rate
  for (int p : {2, 3, 4, 8})
    for (auto spec : {CodecSpec::identity(), CodecSpec::fixed_rate(4), CodecSpec::fixed_rate(8),
                      CodecSpec::fixed_rate(16)}) {
      const size_t n = 300 * p;
      const auto in = inputs(100 + p, p, n);
      const auto xf = flat(in);
      const int kind = static_cast<int>(spec.kind), rate = spec.rate_bits;
      SimClock clk(Topology::lassen_like(2));
      for (int avg = 0; avg < 2; ++avg) {
        const auto got = allreduce(clk, comm_of(p), in, spec, CommPath::DpAllReduce,
                                   avg ? ReduceMode::Average : ReduceMode::Sum);
        std::vector<float> want(n * p);
        uint64_t acct[3];
        CHECK(orc_allreduce(p, n, xf.data(), kind, rate, avg, want.data(), acct) == 0);
        CHECK(std::memcmp(flat(got).data(), want.data(), 4 * want.size()) == 0);
        const auto& e = clk.trace().back();
        CHECK(e.raw_bytes == acct[0] && e.wire_bytes == acct[1] && uint64_t(e.round_count) == acct[2]);
        CHECK(e.comm_size == p && e.collective == CollectiveKind::AllReduce && e.duration_s > 0);
      }
      const auto rs = ring_reduce_scatter(clk, comm_of(p), in, spec, CommPath::Zero1ReduceScatter);
      std::vector<float> wrs(n);
      uint64_t acct[3];
      CHECK(orc_reduce_scatter(p, n, xf.data(), kind, rate, wrs.data(), acct) == 0);
      CHECK(std::memcmp(flat(rs).data(), wrs.data(), 4 * n) == 0);
      CHECK(clk.trace().back().wire_bytes == acct[1]);
      std::vector<FloatBuffer> sh;
      for (const auto& b : in) sh.emplace_back(b.begin(), b.begin() + 100);
      const auto ag = ring_allgather(clk, comm_of(p), sh, spec, CommPath::Zero1AllGather);
      std::vector<float> wag(100 * p * p);
      CHECK(orc_allgather(p, 100, flat(sh).data(), kind, rate, wag.data(), acct) == 0);
      CHECK(std::memcmp(flat(ag).data(), wag.data(), 4 * wag.size()) == 0);
    }
  // agreement, trace accounting, wire shrink (test_collectives.cpp:205-246)
  {
    SimClock clk(Topology::lassen_like(2));
    const auto in = inputs(38, 4, 256 * 4);
    const auto out = allreduce(clk, comm_of(4), in, CodecSpec::fixed_rate(8), CommPath::DpAllReduce);
    for (int i = 1; i < 4; ++i) CHECK(bit_equal(out[0], out[i]));
    const auto& e = clk.trace()[0];
    CHECK(e.wire_bytes < e.raw_bytes && e.wire_bytes > e.raw_bytes / 8);
    CHECK(e.round_count == 6 && e.raw_bytes == 2u * 3 * 4 * 1024 / 4);
    for (int r = 1; r < 4; ++r) CHECK(clk.time(0) == clk.time(r));
  }
  // p2p == direct round trip (test_collectives.cpp:56-65)
  {
    SimClock clk(Topology::lassen_like(2));
    FloatBuffer ramp(64);
    for (int i = 0; i < 64; ++i) ramp[i] = float(i) / 64.0f - 0.5f;
    const auto got = p2p(clk, 0, 1, ramp, CodecSpec::fixed_rate(8), CommPath::PpP2p);
    CHECK(bit_equal(got, decompress(compress(CodecSpec::fixed_rate(8), ramp))));
    CHECK(clk.trace()[0].raw_bytes == 256 && clk.trace()[0].round_count == 1);
  }
  // errors and singletons (test_collectives.cpp:248-271)
  {
    SimClock clk(Topology::lassen_like(2));
    const std::vector<FloatBuffer> ragged = {{1.f, 2.f, 3.f}, {4.f, 5.f, 6.f}};
    CHECK(throws<BadChunkingError>(
        [&] { ring_reduce_scatter(clk, comm_of(2), ragged, CodecSpec::identity(), CommPath::DpAllReduce); }));
    CHECK(throws<BadChunkingError>(
        [&] { allreduce(clk, comm_of(2), ragged, CodecSpec::identity(), CommPath::DpAllReduce); }));
    const std::vector<FloatBuffer> mism = {{1.f, 2.f}, {3.f}};
    CHECK(throws<BadChunkingError>(
        [&] { ring_allgather(clk, comm_of(2), mism, CodecSpec::identity(), CommPath::TpAllGather); }));
    const std::vector<FloatBuffer> one = {{1.f, 2.f, 3.f}};
    const auto o = allreduce(clk, comm_of(1), one, CodecSpec::fixed_rate(8), CommPath::DpAllReduce);
    CHECK(bit_equal(o[0], one[0]) && clk.trace().empty() && clk.max_time() == 0.0);
    std::vector<FloatBuffer> big = {FloatBuffer(128, 3.0e38f), FloatBuffer(128, 3.0e38f)};
    CHECK(throws<NonFiniteInputError>(
        [&] { allreduce(clk, comm_of(2), big, CodecSpec::fixed_rate(8), CommPath::DpAllReduce); }));
  }
  // broadcast (addition)
  {
    SimClock clk(Topology::b200_box(8));
    const auto x = fill(9, 2, 1000);
    const auto out = broadcast(clk, comm_of(8), 3, x, CodecSpec::fixed_rate(8), CommPath::PpP2p);
    const auto want = decompress(compress(CodecSpec::fixed_rate(8), x));
    for (const auto& o : out) CHECK(bit_equal(o, want));
    std::ostringstream csv;
    write_trace_csv(csv, clk.trace());
    CHECK(csv.str().find("Broadcast") != std::string::npos);
  }
}

static void test_policy() {
  // test_parallel3d.cpp: layout groups, scheme builders
  const auto lay = build_layout(2, 3, 4, Topology::b200_box(24));
  CHECK((lay.tp_group(5) == std::vector<int>{4, 5, 6, 7}));
  CHECK((lay.dp_group(5) == std::vector<int>{5, 17}));
  CHECK((lay.pp_chain(5) == std::vector<int>{1, 5, 9}));
  CHECK(throws<BadLayoutError>([] { build_layout(2, 2, 2, Topology::b200_box(10)); }));
  const auto z = scheme_from_name("z-hybrid:16,4");
  CHECK(z.at(CommPath::DpAllReduce) == CodecSpec::fixed_rate(4));
  CHECK(z.at(CommPath::TpAllReduce) == CodecSpec::fixed_rate(16) && z.at(CommPath::PpP2p) == CodecSpec::fixed_rate(16));
  CHECK(scheme_from_name("mz-hybrid:8").at(CommPath::TpAllGather) == CodecSpec::lossless());
  CHECK(throws<InvalidSchemeError>([] { scheme_from_name("z-hybrid:4,16"); }));
  CHECK(throws<ConfigError>([] { scheme_from_name("zhybrid"); }));
  CHECK(comm_path_from_string("Zero1AllGather") == CommPath::Zero1AllGather);
  // hybrid policy drives the collectives: DP at rate 4 (Average), TP at 16
  SimClock clk(Topology::b200_box(4));
  const auto in = inputs(77, 4, 4096);
  allreduce(clk, comm_of(4), in, z.at(CommPath::DpAllReduce), CommPath::DpAllReduce, ReduceMode::Average);
  allreduce(clk, comm_of(4), in, z.at(CommPath::TpAllReduce), CommPath::TpAllReduce);
  CHECK(clk.trace()[0].wire_bytes < clk.trace()[1].wire_bytes);
}

static void test_lossless() {
  // test_codec.cpp:60-68 round trip of arbitrary bits
  for (size_t n : {size_t{0}, size_t{1}, size_t{63}, size_t{4096}, size_t{4097}, size_t{10000}}) {
    const auto x = fill(11 + n, 0, n);
    const auto cb = compress(CodecSpec::lossless(), x);
    CHECK(bit_equal(decompress(cb), x));
    std::vector<uint8_t> want(orc_pred_size(x.data(), n) + 1);
    CHECK(orc_pred_compress(x.data(), n, want.data()) == cb.payload.size());
    CHECK(std::memcmp(want.data(), cb.payload.data(), cb.payload.size()) == 0);
  }
  // :70-80 constant chunk: 3077 bytes
  const FloatBuffer ones(4096, 1.0f);
  const auto cb1 = compress(CodecSpec::lossless(), ones);
  CHECK(cb1.payload_bytes() == 3077u);
  CHECK(bit_equal(decompress(cb1), ones));
  // :95-100 sparse beats dense
  CHECK(compress(CodecSpec::lossless(), fill(13, 3, 1 << 16, 0.9f, 0)).payload_bytes() <
        compress(CodecSpec::lossless(), fill(13, 2, 1 << 16)).payload_bytes());
  // :237-239 truncated payload throws CorruptPayloadError
  auto cut = compress(CodecSpec::lossless(), fill(15, 2, 4096));
  cut.payload.resize(cut.payload.size() / 2);
  CHECK(throws<CorruptPayloadError>([&] { decompress(cut); }));
  // test_collectives.cpp:35-50 identity and lossless p2p are exact
  SimClock clk(Topology::b200_box(8));
  const auto buf = fill(35, 2, 5000);
  CHECK(bit_equal(p2p(clk, 1, 2, buf, CodecSpec::lossless(), CommPath::PpP2p), buf));
  uint64_t acct[3];
  FloatBuffer tmp(5000);
  orc_p2p(5000, buf.data(), 1, 0, tmp.data(), acct);
  CHECK(clk.trace().back().wire_bytes == acct[1]);
  // :189-203 lossless transparency, accounting equal to the oracle's
  for (int p : {2, 4}) {
    const auto in = inputs(37 + p, p, 32 * p * 100);
    SimClock c1(Topology::b200_box(8)), c2(Topology::b200_box(8));
    const auto id = allreduce(c1, comm_of(p), in, CodecSpec::identity(), CommPath::DpAllReduce);
    const auto mpc = allreduce(c2, comm_of(p), in, CodecSpec::lossless(), CommPath::DpAllReduce);
    for (int i = 0; i < p; ++i) CHECK(bit_equal(id[i], mpc[i]));
    CHECK(c1.trace()[0].raw_bytes == c2.trace()[0].raw_bytes);
    const auto f = flat(in);
    std::vector<float> out(f.size());
    uint64_t a[3];
    orc_allreduce(p, in[0].size(), f.data(), 1, 0, 0, out.data(), a);
    CHECK(c2.trace()[0].wire_bytes == a[1]);
    SimClock c3(Topology::b200_box(8));
    ring_reduce_scatter(c3, comm_of(p), in, CodecSpec::lossless(), CommPath::Zero1ReduceScatter);
    std::vector<float> sh(f.size() / p);
    orc_reduce_scatter(p, in[0].size(), f.data(), 1, 0, sh.data(), a);
    CHECK(c3.trace()[0].wire_bytes == a[1]);
  }
  // :275-292 deterministic replay
  const auto in = inputs(41, 4, 128);
  SimClock r1(Topology::b200_box(8)), r2(Topology::b200_box(8));
  const auto o1 = allreduce(r1, comm_of(4), in, CodecSpec::lossless(), CommPath::DpAllReduce);
  const auto o2 = allreduce(r2, comm_of(4), in, CodecSpec::lossless(), CommPath::DpAllReduce);
  CHECK(bit_equal(o1[0], o2[0]) && r1.trace()[0].wire_bytes == r2.trace()[0].wire_bytes);
}

int main() {
  test_codec();
  test_lossless();
  test_collectives();
  test_policy();
  std::printf("hcc shim tests: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
