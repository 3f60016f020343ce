"""Timeline of CTA 0 of the fused NVLink kernel (run under torchrun)."""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec, _lib  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402
from paper_2409_02423_b200.codec import codec_spec_from_string  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, p = dist.get_rank(), dist.get_world_size()
n = int(os.environ.get("TRACE_N", str(1 << 26)))
op = os.environ.get("TRACE_OP", "ar")
spec = codec_spec_from_string(os.environ.get("TRACE_CODEC", "fixed-rate:8"))
comm = D.NvlinkComm(n)
x = torch.randn(n, device="cuda") * 1e-3
out = torch.empty_like(x)
for _ in range(3):
    comm.allreduce(x, spec, 0, out)
torch.cuda.synchronize()
cap = 1 << 16
_lib.hccx_comm_trace_enable(comm.h, cap)
dist.barrier()
reps = int(os.environ.get("TRACE_REPS", "1"))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
if op == "ar":
    for _ in range(reps):
        comm.allreduce(x, spec, 0, out)
elif op == "pp":
    for _ in range(reps):
        comm.p2p(x, 0, 1, spec, out if rank == 1 else None)
elif op == "ag":
    for _ in range(reps):
        comm.allgather(x[: n // p].contiguous(), spec, out)
elif op == "rs":
    for _ in range(reps):
        comm.reduce_scatter(x, spec)
ev1.record()
torch.cuda.synchronize()
ev_us = ev0.elapsed_time(ev1) * 1e3
try:
    comm.status()
    print(f"rank {rank} {op}: ok", flush=True)
except Exception as e:
    print(f"rank {rank} {op}: {e}", flush=True)
buf = (C.c_uint64 * cap)()
nw = C.c_uint64()
_lib.hccx_comm_trace_read(comm.h, buf, cap, C.byref(nw))
acc = {k: buf[4096 + k] for k in range(24)}
if buf[4095]:
    print(f"rank {rank}: pipeline wait timed out: cta {buf[4095] >> 32} who {hex(buf[4095] & 0xffffffff)}", flush=True)
names = {0: "prod_total", 1: "prod_wait_empty", 2: "prod_wait_flag", 8: "push_total", 9: "push_wait_tfull",
         10: "push_wait_read", 11: "push_publish", 12: "push_credit", 13: "push_issue", 14: "push_ack", 15: "push_signal", 16: "comp_total", 17: "comp_wait_full",
         18: "comp_wait_tile", 19: "comp_compute"}
import json as _json
with open(f"gpurun_out/ctas_r{rank}_{op}.json", "w") as fh:
    _json.dump([[buf[8192 + 2 * b], buf[8193 + 2 * b], buf[16384 + b]] for b in range(1024) if buf[8192 + 2 * b]], fh)
spans = [(buf[8192 + 2 * b], buf[8193 + 2 * b]) for b in range(1024) if buf[8192 + 2 * b] and buf[8193 + 2 * b]]
with open(f"gpurun_out/acc_r{rank}_{op}.txt", "w") as fh:
    if spans:
        t0 = min(a for a, _ in spans)
        starts = sorted(a - t0 for a, _ in spans)
        ends = sorted(b - t0 for _, b in spans)
        fh.write(f"r{rank} {op} events_us {ev_us:.1f} ctas {len(spans)} start_max_us {starts[-1] / 1e3:.1f} "
                 f"end_min_us {ends[0] / 1e3:.1f} end_med_us {ends[len(ends) // 2] / 1e3:.1f} "
                 f"end_max_us {ends[-1] / 1e3:.1f}\n")
    for k, nm in names.items():
        fh.write(f"r{rank} {op} {nm:18s} {acc[k] / 1.9e3:10.1f} us (@1.9GHz)\n")
cnt = buf[0]
ev = sorted((buf[2 + 2 * i], buf[1 + 2 * i]) for i in range(min(cnt, (cap - 1) // 2)))
if ev:
    t0 = ev[0][0]
    lines = [f"rank {rank} n={n} op={op} events={cnt}"]
    for t, tag in ev[:400]:
        e, ph, sg = tag >> 32, (tag >> 16) & 0xffff, tag & 0xffff
        lines.append(f"r{rank} {(t - t0) / 1e3:9.2f}us ev{e:2d} ph{ph} k{sg}")
    with open(f"gpurun_out/trace_r{rank}_{op}.txt", "w") as f:
        f.write("\n".join(lines) + "\n")
_lib.hccx_comm_trace_enable(comm.h, 0)
comm.close()
dist.destroy_process_group()
