"""Small-message allreduce latency (BASELINE config 3's low end): per size,
the one-shot path, the ring, and NCCL's allreduce, device time per call (max
over ranks), run under torchrun.  Rank 0 prints one JSON line per size.

  SMALL_SIZES=4096,65536 SMALL_RATE=8 torchrun --nproc-per-node N tools/nvl_small.py
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
sizes = [int(s) for s in os.environ.get(
    "SMALL_SIZES", ",".join(str(1 << k) for k in range(12, 25, 2))).split(",")]  # bytes
rate = int(os.environ.get("SMALL_RATE", "8"))
K = int(os.environ.get("SMALL_K", "50"))
spec = CodecSpec.fixed_rate(rate)
comm = D.NvlinkComm(max(sizes) // 4 + 64 * p)
s = torch.cuda.current_stream()


def timed(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e6))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    us = torch.tensor([a.elapsed_time(b) * 1e3 / K], device="cuda")
    dist.all_reduce(us, op=dist.ReduceOp.MAX)
    return round(float(us.item()), 2)


for nbytes in sizes:
    n = max(nbytes // 4, p)
    n -= n % p
    x = torch.randn(n, device="cuda") * 1e-3
    out = torch.empty_like(x)
    row = {"p": p, "bytes": 4 * n, "rate": rate}
    for mode, env in (("oneshot_us", str(1 << 40)), ("ring_us", "0")):
        os.environ["HCCX_ONESHOT_BYTES"] = env
        row[mode] = timed(lambda: comm.allreduce(x, spec, 0, out))
    os.environ.pop("HCCX_ONESHOT_BYTES", None)
    row["default_us"] = timed(lambda: comm.allreduce(x, spec, 0, out))
    y = x.clone()
    row["nccl_us"] = timed(lambda: dist.all_reduce(y))
    comm.status()
    if rank == 0:
        print(json.dumps(row), flush=True)
comm.close()
dist.destroy_process_group()
