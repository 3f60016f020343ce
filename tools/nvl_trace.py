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
if op == "ar":
    comm.allreduce(x, spec, 0, out)
elif op == "pp":
    comm.p2p(x, 0, 1, spec, out if rank == 1 else None)
elif op == "ag":
    comm.allgather(x[: n // p].contiguous(), spec, out)
buf = (C.c_uint64 * cap)()
nw = C.c_uint64()
_lib.hccx_comm_trace_read(comm.h, buf, cap, C.byref(nw))
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
