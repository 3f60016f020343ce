// capi.cu -- the extern "C" ABI of include/hccx.h for the codec and the
// single-device ring (virtual ranks).  The multi-process NVLink communicator
// lives in comm.cu.
//
// Every entry point validates like the reference (status codes mirror the
// exception hierarchy of proj/include/hcc/errors.hpp) and then only enqueues
// step kernels (step_kernel.cuh); there is no host-side compute path.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "hccx.h"
#include "hccx_internal.h"
#include "hccx_kernels.h"

using namespace hccx;

// ------------------------------------------------------------ helpers ----

namespace hccx {

namespace {
hccx_status_t report_cuda(cudaError_t e, const char* file, int line) {
  static const bool verbose = std::getenv("HCCX_VERBOSE") != nullptr;
  if (verbose) {
    int dev = -1;
    cudaGetDevice(&dev);
    std::fprintf(stderr, "hccx: CUDA failure at %s:%d (device %d, error %s: %s)\n", file, line, dev,
                 cudaGetErrorName(e), cudaGetErrorString(e));
  }
  return HCCX_ERR_CUDA;
}
}  // namespace

hccx_status_t cuda_fail(const char* file, int line) { return report_cuda(cudaPeekAtLastError(), file, line); }

hccx_status_t cuda_status(cudaError_t e) { return e == cudaSuccess ? HCCX_OK : report_cuda(e, "cuda_status", 0); }

hccx_status_t cuda_status_at(cudaError_t e, const char* file, int line) {
  return e == cudaSuccess ? HCCX_OK : report_cuda(e, file, line);
}

hccx_status_t check_codec(hccx_codec_t c) {
  switch (c.kind) {
    case HCCX_CODEC_IDENTITY:
    case HCCX_CODEC_LOSSLESS: return HCCX_OK;
    case HCCX_CODEC_FIXED_RATE:
      return (c.rate_bits >= 2 && c.rate_bits <= 32) ? HCCX_OK : HCCX_ERR_INVALID_SCHEME;
    case HCCX_CODEC_ZFP_RATE:
      return (c.rate_bits >= 3 && c.rate_bits <= 32) ? HCCX_OK : HCCX_ERR_INVALID_SCHEME;
    default: return HCCX_ERR_INVALID_ARGUMENT;
  }
}

// The lossless predictor is value-transparent; its device kernels move the
// raw bytes (identity) and only the wire accounting differs.
CodecSel sel_of(hccx_codec_t c) {
  if (c.kind == HCCX_CODEC_LOSSLESS) return CodecSel{0, 0};
  return CodecSel{c.kind, c.kind == HCCX_CODEC_IDENTITY ? 0 : c.rate_bits};
}

static bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

void finalize_params(StepParams& p, CodecSel c, int op) {
  bool vec = true, fast = true, tma = true;
  const uintptr_t fa = fast_align(c);
  for (int j = 0; j < p.njobs; ++j) {
    const StepJob& J = p.jobs[j];
    if (op == kOpEncode) {
      vec = vec && aligned(J.src, 32);
      fast = fast && aligned(J.dst, fa);
    } else {
      fast = fast && aligned(J.src, fa);
      tma = tma && aligned(J.src, 16);
      if (op == kOpDAR) fast = fast && aligned(J.dst, fa);
      if (op == kOpDecodeAdd) vec = vec && aligned(J.dst, 32);
      if (op == kOpDAR || op == kOpDecodeAdd) vec = vec && aligned(J.local, 32);
    }
    for (int o = 0; o < J.nouts; ++o) vec = vec && aligned(J.outs[o], 32);
  }
  p.vec_ok = vec ? 1 : 0;
  p.fast_ok = fast ? 1 : 0;
  p.tma_ok = tma ? 1 : 0;
}

void set_divisor(StepParams& p, int mode, int nranks) {
  p.div_mode = 0;
  p.recip = 1.0f;
  p.divisor = 1.0f;
  if (mode != HCCX_AVERAGE) return;
  p.divisor = static_cast<float>(nranks);
  if ((nranks & (nranks - 1)) == 0) {
    p.div_mode = 1;
    p.recip = 1.0f / static_cast<float>(nranks);
  } else {
    p.div_mode = 2;
  }
}

hccx_status_t run_step(CodecSel c, int op, StepParams& p, cudaStream_t s) {
  finalize_params(p, c, op);
  const cudaError_t e = launch_step(c, op, p, s);
  if (e != cudaSuccess) return HCCX_CUDA_FAIL;
  return HCCX_STATUS(cudaGetLastError());
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev_);
  if (dev >= 0 && dev != prev_) cudaSetDevice(dev);
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != prev_) cudaSetDevice(prev_);
}

hccx_status_t read_flag(uint32_t* d_err, cudaStream_t s) {
  if (cudaStreamSynchronize(s) != cudaSuccess) return HCCX_CUDA_FAIL;
  uint32_t h = 0;
  if (cudaMemcpy(&h, d_err, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return HCCX_CUDA_FAIL;
  if (h != 0 && cudaMemset(d_err, 0, 4) != cudaSuccess) return HCCX_CUDA_FAIL;
  if (h & kErrTimeout) return HCCX_ERR_TIMEOUT;
  if (h & kErrPeer) return HCCX_ERR_TIMEOUT;
  if (h & kErrNonFinite) return HCCX_ERR_NONFINITE;
  if (h & kErrCorrupt) return HCCX_ERR_CORRUPT_PAYLOAD;
  return HCCX_OK;
}

}  // namespace hccx

// ---------------------------------------------------------- size laws ----

extern "C" const char* hccx_status_string(hccx_status_t s) {
  switch (s) {
    case HCCX_OK: return "ok";
    case HCCX_ERR_NONFINITE: return "non-finite input value on a lossy path";
    case HCCX_ERR_CORRUPT_PAYLOAD: return "corrupt payload";
    case HCCX_ERR_DATA_DEPENDENT_SIZE: return "payload size is data-dependent for this codec";
    case HCCX_ERR_BAD_CHUNKING: return "buffer length does not fit the communicator";
    case HCCX_ERR_BAD_LAYOUT: return "bad parallel layout";
    case HCCX_ERR_INVALID_SCHEME: return "invalid codec/scheme parameters";
    case HCCX_ERR_CONFIG: return "configuration error";
    case HCCX_ERR_CUDA: return "CUDA error";
    case HCCX_ERR_INVALID_ARGUMENT: return "invalid argument";
    case HCCX_ERR_TIMEOUT: return "peer did not respond (timeout)";
    case HCCX_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

extern "C" int hccx_abi_version(void) { return HCCX_ABI_VERSION; }

extern "C" hccx_status_t hccx_codec_validate(hccx_codec_t codec) { return check_codec(codec); }

extern "C" hccx_status_t hccx_wire_size_bytes(hccx_codec_t codec, uint64_t n, uint64_t* bytes) {
  const hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (!bytes) return HCCX_ERR_INVALID_ARGUMENT;
  if (codec.kind == HCCX_CODEC_LOSSLESS) return HCCX_ERR_DATA_DEPENDENT_SIZE;
  *bytes = payload_bytes(sel_of(codec), n);
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_chunk_count(hccx_codec_t codec, uint64_t n, uint64_t* count) {
  const hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (!count) return HCCX_ERR_INVALID_ARGUMENT;
  switch (codec.kind) {
    case HCCX_CODEC_FIXED_RATE: *count = (n + 63) / 64; break;
    case HCCX_CODEC_LOSSLESS: *count = (n + 4095) / 4096; break;
    case HCCX_CODEC_ZFP_RATE: *count = (n + 3) / 4; break;
    default: *count = 0;
  }
  return HCCX_OK;
}

extern "C" uint64_t hccx_launch_count(void) { return launch_count(); }

extern "C" int hccx_device_count(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess ? n : 0;
}

// -------------------------------------------------------------- codec ----

extern "C" hccx_status_t hccx_compress(hccx_codec_t codec, const float* d_in, uint64_t n,
                                       uint8_t* d_out, uint32_t* d_err, void* stream) {
  HCCX_NVTX("hccx_compress");
  hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (codec.kind == HCCX_CODEC_LOSSLESS) return HCCX_ERR_UNSUPPORTED;
  if (n == 0) return HCCX_OK;
  if (!d_in || !d_out) return HCCX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (codec.kind == HCCX_CODEC_IDENTITY)
    return HCCX_STATUS(cudaMemcpyAsync(d_out, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
  StepParams p{};
  p.njobs = 1;
  p.n = n;
  p.jobs[0].src = d_in;
  p.jobs[0].dst = d_out;
  p.err = d_err;
  return run_step(sel_of(codec), kOpEncode, p, s);
}

extern "C" hccx_status_t hccx_decompress(hccx_codec_t codec, const uint8_t* d_in, uint64_t payload,
                                         uint64_t n, float* d_out, void* stream) {
  HCCX_NVTX("hccx_decompress");
  hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (codec.kind == HCCX_CODEC_LOSSLESS) return HCCX_ERR_UNSUPPORTED;
  if (payload != payload_bytes(sel_of(codec), n)) return HCCX_ERR_CORRUPT_PAYLOAD;
  if (n == 0) return HCCX_OK;
  if (!d_in || !d_out) return HCCX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (codec.kind == HCCX_CODEC_IDENTITY)
    return HCCX_STATUS(cudaMemcpyAsync(d_out, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
  StepParams p{};
  p.njobs = 1;
  p.n = n;
  p.jobs[0].src = d_in;
  p.jobs[0].outs[0] = d_out;
  p.jobs[0].nouts = 1;
  return run_step(sel_of(codec), kOpDecode, p, s);
}

extern "C" hccx_status_t hccx_flag_status(uint32_t* d_err, void* stream) {
  if (!d_err) return HCCX_ERR_INVALID_ARGUMENT;
  return read_flag(d_err, static_cast<cudaStream_t>(stream));
}

// --------------------------------------------------- host-buffer codec ----
// Slices of kSlice values (a multiple of the 256-value group, so slice
// payloads concatenate into the exact whole-buffer payload) cycle through
// kLanes streams: H2D(slice) -> kernel -> D2H(slice).  Copies of one slice
// overlap the kernel of the previous one on the copy engines.

namespace {

// Slices of the host pipeline: ~1/16 of the buffer (so filling and draining
// the copy pipeline costs ~1/16 of the transfer), between 256 Ki and 4 Mi
// values, a whole number of 256-value groups; kLanes streams overlap one
// slice's H2D with another's D2H.
constexpr uint64_t kSlice = uint64_t{1} << 22;  // largest slice: 4 Mi values = 16 MiB fp32
constexpr uint64_t kMinSlice = uint64_t{1} << 18;
constexpr int kLanes = 4;

uint64_t slice_for(uint64_t n) {
  uint64_t s = (n / 16 + 255) / 256 * 256;
  s = s < kMinSlice ? kMinSlice : (s > kSlice ? kSlice : s);
  return s;
}

struct HostPipe {
  int device = -1;
  cudaStream_t streams[kLanes] = {};
  float* d_vals[kLanes] = {};
  uint8_t* d_bytes[kLanes] = {};
  uint32_t* d_err = nullptr;
  uint64_t vals_cap = 0, bytes_cap = 0;
};

std::mutex g_pipe_mu;
std::vector<HostPipe*> g_pipes;

HostPipe* pipe_for(int device) {
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  for (HostPipe* p : g_pipes)
    if (p->device == device) return p;
  HostPipe* p = new HostPipe();
  p->device = device;
  for (int i = 0; i < kLanes; ++i) cudaStreamCreateWithFlags(&p->streams[i], cudaStreamNonBlocking);
  cudaMalloc(&p->d_err, 4);
  cudaMemset(p->d_err, 0, 4);
  g_pipes.push_back(p);
  return p;
}

hccx_status_t ensure_pipe(HostPipe* p, uint64_t vals, uint64_t bytes) {
  if (vals > p->vals_cap || bytes > p->bytes_cap) {
    for (int i = 0; i < kLanes; ++i) {
      cudaFree(p->d_vals[i]);
      cudaFree(p->d_bytes[i]);
      p->d_vals[i] = nullptr;
      p->d_bytes[i] = nullptr;
      if (cudaMalloc(&p->d_vals[i], 4 * vals + 64) != cudaSuccess) return HCCX_CUDA_FAIL;
      if (cudaMalloc(&p->d_bytes[i], bytes + 64) != cudaSuccess) return HCCX_CUDA_FAIL;
    }
    p->vals_cap = vals;
    p->bytes_cap = bytes;
  }
  return HCCX_OK;
}

std::mutex g_run_mu;  // one host pipeline run per process at a time

hccx_status_t host_codec(bool compress, hccx_codec_t codec, const void* h_in, uint64_t n, void* h_out,
                         int device) {
  const CodecSel c = sel_of(codec);
  DeviceGuard guard(device);
  std::lock_guard<std::mutex> lock(g_run_mu);
  HostPipe* p = pipe_for(device);
  const uint64_t step = slice_for(n);
  const uint64_t slice = n < step ? n : step;
  const uint64_t slice_bytes = payload_bytes(c, slice);
  hccx_status_t st = ensure_pipe(p, slice, slice_bytes);
  if (st != HCCX_OK) return st;
  const uint64_t gb = group_bytes(c);
  int lane = 0;
  for (uint64_t off = 0; off < n; off += step, lane = (lane + 1) % kLanes) {
    const uint64_t m = (n - off) < step ? (n - off) : step;
    const uint64_t boff = (off / 256) * gb;  // payload offset of this slice
    const uint64_t mb = payload_bytes(c, m);
    cudaStream_t s = p->streams[lane];
    StepParams sp{};
    sp.njobs = 1;
    sp.n = m;
    sp.err = p->d_err;
    if (compress) {
      if (cudaMemcpyAsync(p->d_vals[lane], static_cast<const float*>(h_in) + off, 4 * m,
                          cudaMemcpyHostToDevice, s) != cudaSuccess)
        return HCCX_CUDA_FAIL;
      sp.jobs[0].src = p->d_vals[lane];
      sp.jobs[0].dst = p->d_bytes[lane];
      if ((st = run_step(c, kOpEncode, sp, s)) != HCCX_OK) return st;
      if (cudaMemcpyAsync(static_cast<uint8_t*>(h_out) + boff, p->d_bytes[lane], mb,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return HCCX_CUDA_FAIL;
    } else {
      if (cudaMemcpyAsync(p->d_bytes[lane], static_cast<const uint8_t*>(h_in) + boff, mb,
                          cudaMemcpyHostToDevice, s) != cudaSuccess)
        return HCCX_CUDA_FAIL;
      sp.jobs[0].src = p->d_bytes[lane];
      sp.jobs[0].outs[0] = p->d_vals[lane];
      sp.jobs[0].nouts = 1;
      if ((st = run_step(c, kOpDecode, sp, s)) != HCCX_OK) return st;
      if (cudaMemcpyAsync(static_cast<float*>(h_out) + off, p->d_vals[lane], 4 * m,
                          cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return HCCX_CUDA_FAIL;
    }
  }
  for (int i = 0; i < kLanes; ++i)
    if (cudaStreamSynchronize(p->streams[i]) != cudaSuccess) return HCCX_CUDA_FAIL;
  return read_flag(p->d_err, p->streams[0]);
}

}  // namespace

extern "C" hccx_status_t hccx_compress_host(hccx_codec_t codec, const float* h_in, uint64_t n,
                                            uint8_t* h_out, int device) {
  HCCX_NVTX("hccx_compress_host");
  hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (codec.kind == HCCX_CODEC_LOSSLESS) return HCCX_ERR_UNSUPPORTED;
  if (n == 0) return HCCX_OK;
  if (!h_in || !h_out) return HCCX_ERR_INVALID_ARGUMENT;
  return host_codec(true, codec, h_in, n, h_out, device);
}

extern "C" hccx_status_t hccx_decompress_host(hccx_codec_t codec, const uint8_t* h_in, uint64_t payload,
                                              uint64_t n, float* h_out, int device) {
  HCCX_NVTX("hccx_decompress_host");
  hccx_status_t st = check_codec(codec);
  if (st != HCCX_OK) return st;
  if (codec.kind == HCCX_CODEC_LOSSLESS) return HCCX_ERR_UNSUPPORTED;
  if (payload != payload_bytes(sel_of(codec), n)) return HCCX_ERR_CORRUPT_PAYLOAD;
  if (n == 0) return HCCX_OK;
  if (!h_in || !h_out) return HCCX_ERR_INVALID_ARGUMENT;
  return host_codec(false, codec, h_in, n, h_out, device);
}

// ----------------------------------------- single-device ring (group) ----

struct hccx_group {
  int p = 0;
  int device = 0;
  uint8_t* ws = nullptr;
  uint64_t ws_bytes = 0;
  uint32_t* d_err = nullptr;
  // *_host variants: staging buffers kept across calls (grown on demand)
  std::vector<float*> hbuf;
  std::vector<uint64_t> hcap;
};

namespace {

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

hccx_status_t group_ws(hccx_group* g, uint64_t need) {
  if (need <= g->ws_bytes) return HCCX_OK;
  if (g->ws) cudaFree(g->ws);
  g->ws = nullptr;
  g->ws_bytes = 0;
  if (cudaMalloc(&g->ws, need) != cudaSuccess) return HCCX_CUDA_FAIL;
  g->ws_bytes = need;
  return HCCX_OK;
}

// Ring reduce-scatter on p device buffers (src/collectives.cpp:27-66).
// Round t: member j sends Q(chunk (j-1-t) mod p); j+1 computes
// dec(msg) + local and -- except in the last round -- re-encodes it as its
// own round-(t+1) message (that is the chunk it sends next).  The last round
// either re-encodes into the allgather slot (allreduce, `ag_slots`, writing
// the owner's decoded copy / divisor into out[d] chunk d) or stores the
// fp32 sum (reduce_scatter, `shards`).
hccx_status_t ring_rs(hccx_group* g, CodecSel c, const float* const* in, uint64_t n, float* const* out,
                      float* const* shards, uint8_t** ag_slots_out, int mode, cudaStream_t s) {
  const int p = g->p;
  const uint64_t cn = n / p;
  const uint64_t stride = align_up(payload_bytes(c, cn), 256);
  hccx_status_t st = group_ws(g, 2 * static_cast<uint64_t>(p) * stride + 256);
  if (st != HCCX_OK) return st;
  uint8_t* bank[2] = {g->ws, g->ws + static_cast<uint64_t>(p) * stride};
  auto slot = [&](int b, int j) { return bank[b] + static_cast<uint64_t>(j) * stride; };
  auto chunk = [&](int j) { return ((j % p) + p) % p; };

  StepParams sp{};
  sp.n = cn;
  sp.err = g->d_err;
  sp.njobs = p;
  for (int j = 0; j < p; ++j) {
    sp.jobs[j].src = in[j] + static_cast<uint64_t>(chunk(j - 1)) * cn;
    sp.jobs[j].dst = slot(0, j);
  }
  if ((st = run_step(c, kOpEncode, sp, s)) != HCCX_OK) return st;
  int cur = 0;
  for (int t = 1; t <= p - 2; ++t) {
    StepParams dp{};
    dp.n = cn;
    dp.err = g->d_err;
    dp.njobs = p;
    for (int d = 0; d < p; ++d) {
      dp.jobs[d].src = slot(cur, chunk(d - 1));
      dp.jobs[d].local = in[d] + static_cast<uint64_t>(chunk(d - 1 - t)) * cn;
      dp.jobs[d].dst = slot(1 - cur, d);
    }
    if ((st = run_step(c, kOpDAR, dp, s)) != HCCX_OK) return st;
    cur = 1 - cur;
  }
  StepParams fp{};
  fp.n = cn;
  fp.err = g->d_err;
  fp.njobs = p;
  set_divisor(fp, mode, p);
  for (int d = 0; d < p; ++d) {
    fp.jobs[d].src = slot(cur, chunk(d - 1));
    fp.jobs[d].local = in[d] + static_cast<uint64_t>(d) * cn;
    if (shards) {
      fp.jobs[d].dst = shards[d];
    } else {
      fp.jobs[d].dst = slot(1 - cur, d);
      fp.jobs[d].outs[0] = out[d] + static_cast<uint64_t>(d) * cn;
      fp.jobs[d].nouts = 1;
    }
  }
  if ((st = run_step(c, shards ? kOpDecodeAdd : kOpDAR, fp, s)) != HCCX_OK) return st;
  if (ag_slots_out)
    for (int d = 0; d < p; ++d) ag_slots_out[d] = slot(1 - cur, d);
  return HCCX_OK;
}

// Allgather delivery: every member receives dec(slot[c]) at chunk c, except
// `skip_owner` members that already hold their own chunk.
hccx_status_t ring_ag_deliver(hccx_group* g, CodecSel c, uint8_t* const* slots, uint64_t cn,
                              float* const* out, bool skip_owner, int mode, cudaStream_t s) {
  const int p = g->p;
  StepParams sp{};
  sp.n = cn;
  sp.err = g->d_err;
  sp.njobs = p;
  set_divisor(sp, mode, p);
  for (int cc = 0; cc < p; ++cc) {
    sp.jobs[cc].src = slots[cc];
    int k = 0;
    for (int i = 0; i < p; ++i) {
      if (skip_owner && i == cc) continue;
      sp.jobs[cc].outs[k++] = out[i] + static_cast<uint64_t>(cc) * cn;
    }
    sp.jobs[cc].nouts = k;
  }
  return run_step(c, kOpDecode, sp, s);
}

hccx_status_t check_group(hccx_group* g, hccx_codec_t codec) {
  if (!g) return HCCX_ERR_INVALID_ARGUMENT;
  return check_codec(codec);
}

}  // namespace

extern "C" hccx_status_t hccx_group_create(int p, int device, hccx_group_t* out) {
  if (!out || p < 1 || p > kMaxJobs) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(device);
  hccx_group* g = new hccx_group();
  g->p = p;
  g->device = device;
  if (cudaMalloc(&g->d_err, 4) != cudaSuccess || cudaMemset(g->d_err, 0, 4) != cudaSuccess) {
    delete g;
    return HCCX_CUDA_FAIL;
  }
  *out = g;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_destroy(hccx_group_t g) {
  if (!g) return HCCX_OK;
  DeviceGuard guard(g->device);
  cudaFree(g->ws);
  cudaFree(g->d_err);
  for (float* b : g->hbuf) cudaFree(b);
  delete g;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_allreduce(hccx_group_t g, const float* const* d_in, float* const* d_out,
                                              uint64_t n, hccx_codec_t codec, int mode, void* stream) {
  HCCX_NVTX("hccx_group_allreduce");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  const int p = g->p;
  if (n % static_cast<uint64_t>(p) != 0) return HCCX_ERR_BAD_CHUNKING;
  DeviceGuard guard(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p == 1 || n == 0) {  // src/collectives.cpp:217-219: returned untouched, not quantized
    for (int j = 0; j < p; ++j)
      if (d_out[j] != d_in[j] && n &&
          cudaMemcpyAsync(d_out[j], d_in[j], 4 * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return HCCX_CUDA_FAIL;
    return HCCX_OK;
  }
  const CodecSel c = sel_of(codec);
  uint8_t* slots[kMaxJobs];
  if ((st = ring_rs(g, c, d_in, n, d_out, nullptr, slots, mode, s)) != HCCX_OK) return st;
  return ring_ag_deliver(g, c, slots, n / p, d_out, true, mode, s);
}

extern "C" hccx_status_t hccx_group_reduce_scatter(hccx_group_t g, const float* const* d_in,
                                                   float* const* d_shard, uint64_t n, hccx_codec_t codec,
                                                   void* stream) {
  HCCX_NVTX("hccx_group_reduce_scatter");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  const int p = g->p;
  if (n % static_cast<uint64_t>(p) != 0) return HCCX_ERR_BAD_CHUNKING;
  DeviceGuard guard(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p == 1 || n == 0) {
    if (n && cudaMemcpyAsync(d_shard[0], d_in[0], 4 * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    return HCCX_OK;
  }
  return ring_rs(g, sel_of(codec), d_in, n, nullptr, d_shard, nullptr, HCCX_SUM, s);
}

extern "C" hccx_status_t hccx_group_allgather(hccx_group_t g, const float* const* d_shard, float* const* d_out,
                                              uint64_t shard_n, hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_group_allgather");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  const int p = g->p;
  DeviceGuard guard(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p == 1 || shard_n == 0) {
    if (shard_n &&
        cudaMemcpyAsync(d_out[0], d_shard[0], 4 * shard_n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    return HCCX_OK;
  }
  const CodecSel c = sel_of(codec);
  const uint64_t stride = align_up(payload_bytes(c, shard_n), 256);
  if ((st = group_ws(g, static_cast<uint64_t>(p) * stride + 256)) != HCCX_OK) return st;
  uint8_t* slots[kMaxJobs];
  StepParams sp{};
  sp.n = shard_n;
  sp.err = g->d_err;
  sp.njobs = p;
  for (int j = 0; j < p; ++j) {
    slots[j] = g->ws + static_cast<uint64_t>(j) * stride;
    sp.jobs[j].src = d_shard[j];
    sp.jobs[j].dst = slots[j];
  }
  if ((st = run_step(c, kOpEncode, sp, s)) != HCCX_OK) return st;
  return ring_ag_deliver(g, c, slots, shard_n, d_out, false, HCCX_SUM, s);
}

extern "C" hccx_status_t hccx_group_broadcast(hccx_group_t g, int root, const float* d_in, float* const* d_out,
                                              uint64_t n, hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_group_broadcast");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  const int p = g->p;
  if (root < 0 || root >= p) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return HCCX_OK;
  if (p == 1) {
    if (d_out[0] != d_in && cudaMemcpyAsync(d_out[0], d_in, 4 * n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return HCCX_CUDA_FAIL;
    return HCCX_OK;
  }
  const CodecSel c = sel_of(codec);
  if ((st = group_ws(g, align_up(payload_bytes(c, n), 256) + 256)) != HCCX_OK) return st;
  StepParams sp{};
  sp.n = n;
  sp.err = g->d_err;
  sp.njobs = 1;
  sp.jobs[0].src = d_in;
  sp.jobs[0].dst = g->ws;
  if ((st = run_step(c, kOpEncode, sp, s)) != HCCX_OK) return st;
  // Decode once per group into all p outputs (kMaxOuts >= kMaxJobs >= p).
  StepParams dp{};
  dp.n = n;
  dp.err = g->d_err;
  dp.njobs = 1;
  dp.jobs[0].src = g->ws;
  for (int i = 0; i < p; ++i) dp.jobs[0].outs[i] = d_out[i];
  dp.jobs[0].nouts = p;
  return run_step(c, kOpDecode, dp, s);
}

extern "C" hccx_status_t hccx_group_p2p(hccx_group_t g, const float* d_in, float* d_out, uint64_t n,
                                        hccx_codec_t codec, void* stream) {
  HCCX_NVTX("hccx_group_p2p");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  DeviceGuard guard(g->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) return HCCX_OK;
  const CodecSel c = sel_of(codec);
  if (c.kind == 0) return HCCX_STATUS(cudaMemcpyAsync(d_out, d_in, 4 * n, cudaMemcpyDeviceToDevice, s));
  if ((st = group_ws(g, align_up(payload_bytes(c, n), 256) + 256)) != HCCX_OK) return st;
  StepParams sp{};
  sp.n = n;
  sp.err = g->d_err;
  sp.njobs = 1;
  sp.jobs[0].src = d_in;
  sp.jobs[0].dst = g->ws;
  if ((st = run_step(c, kOpEncode, sp, s)) != HCCX_OK) return st;
  StepParams dp{};
  dp.n = n;
  dp.err = g->d_err;
  dp.njobs = 1;
  dp.jobs[0].src = g->ws;
  dp.jobs[0].outs[0] = d_out;
  dp.jobs[0].nouts = 1;
  return run_step(c, kOpDecode, dp, s);
}

extern "C" hccx_status_t hccx_group_status(hccx_group_t g, void* stream) {
  if (!g) return HCCX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(g->device);
  return read_flag(g->d_err, static_cast<cudaStream_t>(stream));
}

// ----------------------------------------- host-buffer group variants ----

namespace {

// The group's staging buffers for one *_host call: slot k of the call is
// the group's k-th cached buffer, reallocated only when it must grow (no
// allocator traffic in steady state).
struct DevBufs {
  hccx_group* g;
  size_t next = 0;
  explicit DevBufs(hccx_group* grp) : g(grp) {}
  float* add(uint64_t n) {
    const size_t k = next++;
    if (g->hbuf.size() <= k) {
      g->hbuf.resize(k + 1, nullptr);
      g->hcap.resize(k + 1, 0);
    }
    if (g->hcap[k] < n || !g->hbuf[k]) {
      cudaFree(g->hbuf[k]);
      g->hbuf[k] = nullptr;
      g->hcap[k] = 0;
      float* p = nullptr;
      if (cudaMalloc(&p, 4 * (n ? n : 1)) != cudaSuccess) return nullptr;
      g->hbuf[k] = p;
      g->hcap[k] = n;
    }
    return g->hbuf[k];
  }
};

template <class F>
hccx_status_t timed_run(hccx_group* g, double* secs, F&& body) {
  cudaStream_t s = nullptr;
  cudaEvent_t a = nullptr, b = nullptr;
  if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return HCCX_CUDA_FAIL;
  cudaEventRecord(a, s);
  hccx_status_t st = body(s);
  cudaEventRecord(b, s);
  if (st == HCCX_OK) st = hccx_group_status(g, s);
  float ms = 0.0f;
  if (cudaEventSynchronize(b) == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
  if (secs) *secs = ms * 1e-3;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return st;
}

hccx_status_t h2d(float* d, const float* h, uint64_t n) {
  return n ? HCCX_STATUS(cudaMemcpy(d, h, 4 * n, cudaMemcpyHostToDevice)) : HCCX_OK;
}
hccx_status_t d2h(float* h, const float* d, uint64_t n) {
  return n ? HCCX_STATUS(cudaMemcpy(h, d, 4 * n, cudaMemcpyDeviceToHost)) : HCCX_OK;
}

}  // namespace

extern "C" hccx_status_t hccx_group_allreduce_host(hccx_group_t g, const float* const* h_in, float* const* h_out,
                                                   uint64_t n, hccx_codec_t codec, int mode, double* secs) {
  HCCX_NVTX("hccx_group_allreduce_host");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(g->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  DeviceGuard guard(g->device);
  DevBufs B(g);
  std::vector<float*> din(g->p), dout(g->p);
  for (int j = 0; j < g->p; ++j) {
    if (!(din[j] = B.add(n)) || !(dout[j] = B.add(n))) return HCCX_CUDA_FAIL;
    if ((st = h2d(din[j], h_in[j], n)) != HCCX_OK) return st;
  }
  st = timed_run(g, secs, [&](cudaStream_t s) {
    return hccx_group_allreduce(g, din.data(), dout.data(), n, codec, mode, s);
  });
  if (st != HCCX_OK) return st;
  for (int j = 0; j < g->p; ++j)
    if ((st = d2h(h_out[j], dout[j], n)) != HCCX_OK) return st;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_reduce_scatter_host(hccx_group_t g, const float* const* h_in,
                                                        float* const* h_shard, uint64_t n, hccx_codec_t codec,
                                                        double* secs) {
  HCCX_NVTX("hccx_group_reduce_scatter_host");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  if (n % static_cast<uint64_t>(g->p) != 0) return HCCX_ERR_BAD_CHUNKING;
  DeviceGuard guard(g->device);
  const uint64_t c = n / g->p;
  DevBufs B(g);
  std::vector<float*> din(g->p), dsh(g->p);
  for (int j = 0; j < g->p; ++j) {
    if (!(din[j] = B.add(n)) || !(dsh[j] = B.add(c))) return HCCX_CUDA_FAIL;
    if ((st = h2d(din[j], h_in[j], n)) != HCCX_OK) return st;
  }
  st = timed_run(g, secs, [&](cudaStream_t s) {
    return hccx_group_reduce_scatter(g, din.data(), dsh.data(), n, codec, s);
  });
  if (st != HCCX_OK) return st;
  for (int j = 0; j < g->p; ++j)
    if ((st = d2h(h_shard[j], dsh[j], g->p == 1 ? n : c)) != HCCX_OK) return st;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_allgather_host(hccx_group_t g, const float* const* h_shard, float* const* h_out,
                                                   uint64_t shard_n, hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_group_allgather_host");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  DeviceGuard guard(g->device);
  const uint64_t n = shard_n * g->p;
  DevBufs B(g);
  std::vector<float*> dsh(g->p), dout(g->p);
  for (int j = 0; j < g->p; ++j) {
    if (!(dsh[j] = B.add(shard_n)) || !(dout[j] = B.add(n))) return HCCX_CUDA_FAIL;
    if ((st = h2d(dsh[j], h_shard[j], shard_n)) != HCCX_OK) return st;
  }
  st = timed_run(g, secs, [&](cudaStream_t s) {
    return hccx_group_allgather(g, dsh.data(), dout.data(), shard_n, codec, s);
  });
  if (st != HCCX_OK) return st;
  for (int j = 0; j < g->p; ++j)
    if ((st = d2h(h_out[j], dout[j], n)) != HCCX_OK) return st;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_broadcast_host(hccx_group_t g, int root, const float* h_in, float* const* h_out,
                                                   uint64_t n, hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_group_broadcast_host");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  DeviceGuard guard(g->device);
  DevBufs B(g);
  float* din = B.add(n);
  std::vector<float*> dout(g->p);
  if (!din) return HCCX_CUDA_FAIL;
  for (int j = 0; j < g->p; ++j)
    if (!(dout[j] = B.add(n))) return HCCX_CUDA_FAIL;
  if ((st = h2d(din, h_in, n)) != HCCX_OK) return st;
  st = timed_run(g, secs, [&](cudaStream_t s) {
    return hccx_group_broadcast(g, root, din, dout.data(), n, codec, s);
  });
  if (st != HCCX_OK) return st;
  for (int j = 0; j < g->p; ++j)
    if ((st = d2h(h_out[j], dout[j], n)) != HCCX_OK) return st;
  return HCCX_OK;
}

extern "C" hccx_status_t hccx_group_p2p_host(hccx_group_t g, const float* h_in, float* h_out, uint64_t n,
                                             hccx_codec_t codec, double* secs) {
  HCCX_NVTX("hccx_group_p2p_host");
  hccx_status_t st = check_group(g, codec);
  if (st != HCCX_OK) return st;
  DeviceGuard guard(g->device);
  DevBufs B(g);
  float* din = B.add(n);
  float* dout = B.add(n);
  if (!din || !dout) return HCCX_CUDA_FAIL;
  if ((st = h2d(din, h_in, n)) != HCCX_OK) return st;
  st = timed_run(g, secs, [&](cudaStream_t s) { return hccx_group_p2p(g, din, dout, n, codec, s); });
  if (st != HCCX_OK) return st;
  return d2h(h_out, dout, n);
}
