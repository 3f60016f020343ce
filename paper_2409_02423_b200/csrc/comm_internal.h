// comm_internal.h -- the NVLink communicator's state, shared by comm.cu
// (windows, fused-kernel collectives, single-process communicators) and
// lossless_comm.cu (LosslessPredictor collectives with framed messages).
#pragma once
#include <cstdint>

#include "hccx.h"
#include "lossless_msg.h"
#include "ring_fused.cuh"

struct hccx_comm {
  int rank = 0, p = 0, device = 0;
  uint64_t chunk_cap = 0;   // values per slot (multiple of one segment)
  uint64_t slot_bytes = 0;  // payload capacity per slot (worst codec: 257 B / 64 values)
  uint32_t max_seg = 0;
  uint64_t rs_off = 0, ag_off = 0, pp_off = 0, flag_off = 0, win_bytes = 0;
  uint64_t os_cap = 0;  // one-shot allreduce: values per chunk
  uint64_t os_off = 0, os_ag_off = 0, os_flag_off = 0, os_raw_bytes = 0, os_ag_bytes = 0;
  uint64_t os_ll_off = 0, os_ll_ag_off = 0, os_ll_raw_bytes = 0, os_ll_ag_bytes = 0;
  uint8_t* win = nullptr;
  uint8_t* peers[hccx::kMaxRanks] = {};
  bool connected = false;
  uint32_t* d_err = nullptr;
  uint32_t epoch = 0;                  // collectives
  uint32_t last_rs = 0, last_ag = 0;   // epoch of the last collective that used rs / ag slots
  uint32_t send_ep[hccx::kMaxRanks] = {};    // p2p / broadcast messages sent to rank d
  uint32_t recv_ep[hccx::kMaxRanks] = {};    // ... received from rank s
  uint64_t* d_trace = nullptr;         // optional CTA-0 timeline (hccx_comm_trace_enable)
  uint64_t trace_cap = 0;
  // Slot geometry (codec, values per slot) of the last use of each slot
  // class; a change makes the next sender wait for every receiver CTA's ack
  // (FusedParams::credit_all).
  uint64_t geo_rs = 0, geo_ag = 0;
  uint64_t geo_pp[hccx::kMaxRanks] = {};     // per destination (send side)
  uint32_t max_grid = 0;               // CTAs per rank shared by all ranks (single-process comms)
  bool ipc = true;                     // peers[] opened with cudaIpcOpenMemHandle (closed on destroy)
  // bytes this rank pushed in its last collective: codec payloads (the
  // reference's wire accounting) and whole frames (payload + message header)
  uint64_t last_payload = 0, last_frame = 0;
  uint64_t last_recv = 0;  // framed payload bytes received (LosslessPredictor collectives)
  // LosslessPredictor collectives (grown on demand, this device): encoder
  // scratch, byte accounting (payload pushed, message bytes pushed, payload
  // received), the reduce-scatter work copy
  hccx::MsgScratch ll_msg;
  unsigned long long* ll_acct = nullptr;
  float* ll_work = nullptr;
  uint64_t ll_work_cap = 0;
  uint8_t* ll_stage = nullptr;  // whole framed message: root staging / receiver reassembly
  uint64_t ll_stage_cap = 0;
};

namespace hccx {

// Message frame at the start of a slot for framed (data-dependent size)
// messages: [u64 container bytes][HCC1 container header, 18 B
// (proj/src/codec.cpp:89-99)][pad][payload at kFrameBytes].
constexpr uint64_t kFrameBytes = 32;

uint64_t comm_timeout_ns();

}  // namespace hccx
