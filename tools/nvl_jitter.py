"""Per-call device-time distribution of the NVLink allreduce (torchrun, N
GPUs): JITTER_BYTES per rank, JITTER_RATE, JITTER_CALLS calls each bracketed
by its own events; prints min/median/p90/max over calls (max over ranks)."""
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
sizes = [int(s) for s in os.environ.get("JITTER_BYTES", str(64 << 20)).split(",")]
rate = int(os.environ.get("JITTER_RATE", "8"))
calls = int(os.environ.get("JITTER_CALLS", "40"))
comm = D.NvlinkComm(max(sizes) // 4)
for nbytes in sizes:
    n = nbytes // 4 - (nbytes // 4) % p
    x = torch.randn(n, device="cuda") * 1e-3
    out = torch.empty_like(x)
    spec = CodecSpec.fixed_rate(rate)
    for _ in range(3):
        comm.allreduce(x, spec, 0, out)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(calls + 1)]
    torch.cuda._sleep(int(2e6))
    ev[0].record()
    for i in range(calls):
        comm.allreduce(x, spec, 0, out)
        ev[i + 1].record()
    torch.cuda.synchronize()
    t = torch.tensor([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(calls)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ts = sorted(t.tolist())
    comm.status()
    if rank == 0:
        print(f"p={p} bytes={nbytes} r{rate}: min {ts[0]:.1f} med {ts[len(ts) // 2]:.1f} p90 {ts[int(len(ts) * 0.9)]:.1f} "
              f"max {ts[-1]:.1f} us; slow calls (>1.5x med): {[round(v) for v in t.tolist() if v > 1.5 * ts[len(ts) // 2]]}",
              flush=True)
comm.close()
dist.destroy_process_group()
