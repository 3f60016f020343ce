"""Interleaved A/B of fused-allreduce variants selected per call by env
(HCCX_DEBUG knobs, HCCX_STEP_SEGS, ...), run under torchrun:

  AB="HCCX_DEBUG=0;HCCX_DEBUG=128" torchrun --nproc-per-node N tools/nvl_ab.py [n] [rounds]
  (AB_RATE=R picks the rate, AB_CODEC=zfp the ZFP-mode codec)

Each round times K back-to-back allreduces per variant (CUDA events, max
over ranks); rank 0 prints the per-variant median ms and GB/s.
"""
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 5
K = int(os.environ.get("AB_K", "10"))
spec = (CodecSpec.zfp_rate(int(os.environ.get("AB_RATE", "8"))) if os.environ.get("AB_CODEC") == "zfp"
        else CodecSpec.fixed_rate(int(os.environ.get("AB_RATE", "8"))))
variants = [v for v in os.environ.get("AB", "HCCX_DEBUG=0").split(";") if v]
comm = D.NvlinkComm(n)
x = torch.randn(n, device="cuda") * 1e-3
out = torch.empty_like(x)
s = torch.cuda.current_stream()


def apply(v):
    for kv in v.split(","):
        k, val = kv.split("=", 1)
        os.environ[k] = val


res = {v: [] for v in variants}
for r in range(rounds + 1):
    for v in variants:
        apply(v)
        for _ in range(2):
            comm.allreduce(x, spec, 0, out)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(1e6))
        a.record(s)
        for _ in range(K):
            comm.allreduce(x, spec, 0, out)
        b.record(s)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / K], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        if r:
            res[v].append(float(ms.item()))
comm.status()
if rank == 0:
    for v, ts in res.items():
        ts.sort()
        med = ts[len(ts) // 2]
        print(f"p={p} n={n} [{v}] median {med:.4f} ms  {4 * n / (med * 1e-3) / 1e9:.1f} GB/s  (min {ts[0]:.4f})",
              flush=True)
comm.close()
dist.destroy_process_group()
