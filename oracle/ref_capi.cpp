// ref_capi.cpp -- extern "C" shim over the UNMODIFIED reference library
// (hybridcomm, /root/reference/proj/src), compiled by oracle/build_ref.sh into
// oracle/_ref/libhcc_ref.so.  TEST INFRASTRUCTURE ONLY: it lets the Python
// tests pin the C restatement (oracle/hcc_oracle.c) against the reference
// itself, and lets bench.py time the reference's own CPU path
// (`--impl reference`, `cpu_baseline.kind == "reference"`).
//
// Nothing here re-implements reference logic; each entry point forwards to the
// reference API named in its comment (paths relative to /root/reference/proj).
#include <cstdint>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <vector>

#include "hcc/codec.hpp"
#include "hcc/collectives.hpp"
#include "hcc/errors.hpp"
#include "hcc/netsim.hpp"
#include "hcc/parallel3d.hpp"
#include "hcc/rng.hpp"
#include "hcc/toymodel.hpp"
#include "support/oracles.hpp"

namespace {

// Status codes match include/hccx.h.
int status_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const hcc::NonFiniteInputError&) {
    return 1;
  } catch (const hcc::CorruptPayloadError&) {
    return 2;
  } catch (const hcc::DataDependentSizeError&) {
    return 3;
  } catch (const hcc::BadChunkingError&) {
    return 4;
  } catch (const hcc::BadLayoutError&) {
    return 5;
  } catch (const hcc::InvalidSchemeError&) {
    return 6;
  } catch (const hcc::ConfigError&) {
    return 7;
  } catch (...) {
    return 99;
  }
}

hcc::CodecSpec spec_of(int kind, int rate) {
  switch (kind) {
    case 0: return hcc::CodecSpec::identity();
    case 1: return hcc::CodecSpec::lossless();
    default: return hcc::CodecSpec::fixed_rate(rate);
  }
}

// lassen_like has 4 GPUs per node (src/netsim.cpp:20-31); give the clock a
// world large enough for a p-member communicator.
hcc::SimClock make_clock(int p) { return hcc::SimClock(hcc::Topology::lassen_like((p + 3) / 4)); }

hcc::Communicator make_comm(int p) {
  hcc::Communicator c;
  for (int i = 0; i < p; ++i) c.ranks.push_back(i);
  return c;
}

std::vector<hcc::FloatBuffer> split(const float* in, int p, uint64_t n) {
  std::vector<hcc::FloatBuffer> v(static_cast<size_t>(p));
  for (int j = 0; j < p; ++j) v[j].assign(in + static_cast<uint64_t>(j) * n, in + static_cast<uint64_t>(j + 1) * n);
  return v;
}

void fill_acct(const hcc::SimClock& clk, uint64_t* acct) {
  acct[0] = acct[1] = acct[2] = 0;
  if (!clk.trace().empty()) {
    const auto& e = clk.trace().back();
    acct[0] = e.raw_bytes;
    acct[1] = e.wire_bytes;
    acct[2] = static_cast<uint64_t>(e.round_count);
  }
}

}  // namespace

extern "C" {

// hcc::compress / hcc::serial::compress (src/codec_omp.cpp:19, src/codec_serial.cpp:14).
// Writes the payload into `out` (capacity `cap`), returns status; *out_len = payload size.
int ref_compress(int kind, int rate, int serial, const float* in, uint64_t n, uint8_t* out,
                 uint64_t cap, uint64_t* out_len, uint32_t* chunk_count) {
  try {
    hcc::FloatBuffer buf(in, in + n);
    const auto spec = spec_of(kind, rate);
    const hcc::CompressedBuffer cb = serial ? hcc::serial::compress(spec, buf) : hcc::compress(spec, buf);
    *out_len = cb.payload.size();
    if (chunk_count) *chunk_count = cb.chunk_count;
    if (cb.payload.size() > cap) return 98;
    if (!cb.payload.empty()) std::memcpy(out, cb.payload.data(), cb.payload.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::decompress / hcc::serial::decompress (src/codec_omp.cpp:87, src/codec_serial.cpp:68).
int ref_decompress(int kind, int rate, int serial, const uint8_t* in, uint64_t in_len, uint64_t n,
                   uint32_t chunk_count, float* out) {
  try {
    hcc::CompressedBuffer cb;
    cb.codec = spec_of(kind, rate);
    cb.original_len = n;
    cb.chunk_count = chunk_count;
    cb.payload.assign(in, in + in_len);
    const hcc::FloatBuffer v = serial ? hcc::serial::decompress(cb) : hcc::decompress(cb);
    if (!v.empty()) std::memcpy(out, v.data(), 4 * v.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::wire_size_bytes (src/codec.cpp:47-61)
int ref_wire_size(int kind, int rate, uint64_t n, uint64_t* out) {
  try {
    *out = hcc::wire_size_bytes(spec_of(kind, rate), n);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::to_bytes (src/codec.cpp:89-100) of compress(spec, in).
int ref_container(int kind, int rate, const float* in, uint64_t n, uint8_t* out, uint64_t cap,
                  uint64_t* out_len) {
  try {
    const auto bytes = hcc::to_bytes(hcc::compress(spec_of(kind, rate), hcc::FloatBuffer(in, in + n)));
    *out_len = bytes.size();
    if (bytes.size() > cap) return 98;
    std::memcpy(out, bytes.data(), bytes.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::allreduce (src/collectives.cpp:202-248), all p members in one call.
int ref_allreduce(int p, uint64_t n, const float* inputs, int kind, int rate, int average,
                  float* out, uint64_t* acct) {
  try {
    auto clk = make_clock(p);
    const auto res = hcc::allreduce(clk, make_comm(p), split(inputs, p, n), spec_of(kind, rate),
                                    hcc::CommPath::DpAllReduce,
                                    average ? hcc::ReduceMode::Average : hcc::ReduceMode::Sum);
    for (int j = 0; j < p; ++j) std::memcpy(out + static_cast<uint64_t>(j) * n, res[j].data(), 4 * n);
    fill_acct(clk, acct);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// Timed forms for the bench's reference arm: the inputs are turned into the
// reference's value types once, outside the timed region, and only the
// reference library's own calls are timed (no marshalling copies).
// hcc::compress + hcc::decompress of n values, `reps` round trips; *secs =
// the median round trip.
int ref_time_codec(int kind, int rate, const float* in, uint64_t n, int reps, double* secs) {
  try {
    const hcc::FloatBuffer buf(in, in + n);
    const auto spec = spec_of(kind, rate);
    std::vector<double> t;
    for (int r = 0; r < reps; ++r) {
      const auto a = std::chrono::steady_clock::now();
      const hcc::CompressedBuffer cb = hcc::compress(spec, buf);
      const hcc::FloatBuffer back = hcc::decompress(cb);
      const auto b = std::chrono::steady_clock::now();
      if (back.size() != n) return 97;
      t.push_back(std::chrono::duration<double>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    *secs = t.empty() ? 0.0 : t[t.size() / 2];
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::allreduce of p members x n values (Sum), `reps` calls; *secs = median.
int ref_time_allreduce(int p, uint64_t n, const float* inputs, int kind, int rate, int reps, double* secs) {
  try {
    const auto ins = split(inputs, p, n);
    const auto comm = make_comm(p);
    const auto spec = spec_of(kind, rate);
    std::vector<double> t;
    for (int r = 0; r < reps; ++r) {
      auto clk = make_clock(p);
      const auto a = std::chrono::steady_clock::now();
      const auto res = hcc::allreduce(clk, comm, ins, spec, hcc::CommPath::DpAllReduce, hcc::ReduceMode::Sum);
      const auto b = std::chrono::steady_clock::now();
      if (static_cast<int>(res.size()) != p) return 97;
      t.push_back(std::chrono::duration<double>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    *secs = t.empty() ? 0.0 : t[t.size() / 2];
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::ring_reduce_scatter (src/collectives.cpp:154-181)
int ref_reduce_scatter(int p, uint64_t n, const float* inputs, int kind, int rate, float* shards,
                       uint64_t* acct) {
  try {
    auto clk = make_clock(p);
    const auto res = hcc::ring_reduce_scatter(clk, make_comm(p), split(inputs, p, n),
                                              spec_of(kind, rate), hcc::CommPath::Zero1ReduceScatter);
    const uint64_t c = n / static_cast<uint64_t>(p);
    for (int j = 0; j < p; ++j) std::memcpy(shards + static_cast<uint64_t>(j) * c, res[j].data(), 4 * c);
    fill_acct(clk, acct);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::ring_allgather (src/collectives.cpp:183-200)
int ref_allgather(int p, uint64_t c, const float* shards, int kind, int rate, float* out,
                  uint64_t* acct) {
  try {
    auto clk = make_clock(p);
    const auto res = hcc::ring_allgather(clk, make_comm(p), split(shards, p, c), spec_of(kind, rate),
                                         hcc::CommPath::Zero1AllGather);
    const uint64_t n = c * static_cast<uint64_t>(p);
    for (int j = 0; j < p; ++j) std::memcpy(out + static_cast<uint64_t>(j) * n, res[j].data(), 4 * n);
    fill_acct(clk, acct);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// hcc::p2p (src/collectives.cpp:130-152)
int ref_p2p(uint64_t n, const float* in, int kind, int rate, float* out, uint64_t* acct) {
  try {
    auto clk = make_clock(2);
    const auto res = hcc::p2p(clk, 0, 1, hcc::FloatBuffer(in, in + n), spec_of(kind, rate),
                              hcc::CommPath::PpP2p);
    if (!res.empty()) std::memcpy(out, res.data(), 4 * n);
    fill_acct(clk, acct);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// Buffer generators of tests/support/oracles.cpp:9-36 driven by hcc::Rng.
// mode: 0 bits, 1 finite, 2 uniform[lo,hi), 3 sparse(lo = zero fraction).
void ref_fill(uint64_t seed, int mode, uint64_t n, float lo, float hi, float* out) {
  hcc::Rng rng(seed);
  hcc::FloatBuffer b;
  switch (mode) {
    case 0: b = hcc::testing::random_bits_buffer(rng, n); break;
    case 1: b = hcc::testing::random_finite_buffer(rng, n); break;
    case 2: b = hcc::testing::uniform_buffer(rng, n, lo, hi); break;
    default: b = hcc::testing::sparse_buffer(rng, n, lo); break;
  }
  if (n) std::memcpy(out, b.data(), 4 * n);
}

// hcc::Trainer3D (src/toymodel.cpp:239-467) through run_experiment: the
// reference's 3D-parallel toy trainer on a one-node lassen_like topology of
// dp*pp*tp GPUs.  Outputs the step losses, the final eval loss, the
// assembled replica-0 model and raw/wire bytes per CommPath (enum order).
int ref_train(int num_blocks, int hidden, int width, int batch, int microbatches, int steps, uint64_t seed,
              float lr, int dp, int pp, int tp, const char* scheme, int zero, float* step_loss,
              int* steps_completed, float* final_eval, int* diverged, float* w1, float* w2, uint64_t* path_bytes) {
  try {
    hcc::ToyModelConfig cfg;
    cfg.num_blocks = num_blocks;
    cfg.hidden_dim = hidden;
    cfg.input_dim = width;
    cfg.batch_size = batch;
    cfg.microbatches = microbatches;
    cfg.steps = steps;
    cfg.seed = seed;
    cfg.learning_rate = lr;
    hcc::Topology topo = hcc::Topology::lassen_like(1);
    topo.gpus_per_node = dp * pp * tp;
    const auto layout = hcc::build_layout(dp, pp, tp, topo);
    hcc::Trainer3D trainer(cfg, layout, topo, hcc::scheme_from_name(scheme),
                           zero == 0 ? hcc::ZeroMode::Off : (zero == 1 ? hcc::ZeroMode::Replace
                                                                       : hcc::ZeroMode::Redundant));
    const auto met = trainer.run();
    for (std::size_t i = 0; i < met.step_loss.size(); ++i) step_loss[i] = met.step_loss[i];
    *steps_completed = met.steps_completed;
    *final_eval = met.final_eval_loss;
    *diverged = met.diverged ? 1 : 0;
    const auto model = trainer.assemble_replica(0);
    std::memcpy(w1, model.w1.data(), 4 * model.w1.size());
    std::memcpy(w2, model.w2.data(), 4 * model.w2.size());
    for (int k = 0; k < 12; ++k) path_bytes[k] = 0;
    for (const auto& [path, b] : met.bytes_by_path) {
      path_bytes[2 * static_cast<int>(path)] = b.raw;
      path_bytes[2 * static_cast<int>(path) + 1] = b.wire;
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

}  // extern "C"
