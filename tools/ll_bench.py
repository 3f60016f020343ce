"""LosslessPredictor collectives on the NVLink engine (csrc/lossless_comm.cu),
run under torchrun: allreduce / p2p of smooth (compressible) and random
fp32 at several sizes; device time per call (CUDA events, max over ranks)
and the payload bytes this rank pushed.  HCCX_LL_PROFILE=1 adds a per-stage
breakdown on stderr.

  torchrun --nproc-per-node N tools/ll_bench.py [n ...]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, p = dist.get_rank(), dist.get_world_size()
sizes = [int(a) for a in sys.argv[1:]] or [1 << 20, 1 << 22, 1 << 24]
K = int(os.environ.get("LL_K", "5"))
spec = CodecSpec.lossless()
comm = D.NvlinkComm(max(sizes))
s = torch.cuda.current_stream()


def data(kind, n):
    if kind == "smooth":
        t = torch.arange(n, device="cuda", dtype=torch.float32)
        x = torch.sin(t * 1e-4 + rank) * 1e-2
        return (x * 4096).round() / 4096
    return torch.randn(n, device="cuda")


def timed(fn):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / K], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


for n in sizes:
    n -= n % p
    for kind in ("smooth", "random"):
        x = data(kind, n)
        out = torch.empty_like(x)
        ms = timed(lambda: comm.allreduce(x, spec, 0, out))
        pay, frame = comm.wire_bytes()
        row = {"op": "allreduce", "data": kind, "p": p, "values": n, "us": round(ms * 1e3, 1),
               "algbw_GBps": round(4 * n / (ms * 1e-3) / 1e9, 2), "payload_pushed": pay, "frame_pushed": frame}
        ms = timed(lambda: comm.p2p(x, 0, 1, spec, out))
        row2 = {"op": "p2p", "data": kind, "p": p, "values": n, "us": round(ms * 1e3, 1),
                "GBps": round(4 * n / (ms * 1e-3) / 1e9, 2)}
        if rank == 0:
            print(json.dumps(row), flush=True)
            print(json.dumps(row2), flush=True)
comm.status()
comm.close()
dist.destroy_process_group()
