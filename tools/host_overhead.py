"""Host-side enqueue cost per small allreduce call (4 KiB): hccx through NvlinkComm, through raw ctypes, and NCCL; the GPU is kept busy so the host never waits (run under torchrun)."""
import os, sys, time, json
import torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2409_02423_b200 import CodecSpec
from paper_2409_02423_b200 import dist as D
local = int(os.environ.get("LOCAL_RANK", "0")); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, p = dist.get_rank(), dist.get_world_size()
spec = CodecSpec.fixed_rate(8)
comm = D.NvlinkComm(1 << 20)
x = torch.randn(1024, device="cuda"); out = torch.empty_like(x)
for _ in range(20): comm.allreduce(x, spec, 0, out)
torch.cuda.synchronize(); dist.barrier()
torch.cuda._sleep(int(2e8))  # ~100 ms: the host never waits for the GPU below
t0 = time.perf_counter()
for _ in range(200): comm.allreduce(x, spec, 0, out)
t1 = time.perf_counter()
torch.cuda.synchronize(); dist.barrier()
y = x.clone()
for _ in range(20): dist.all_reduce(y)
torch.cuda.synchronize(); dist.barrier()
torch.cuda._sleep(int(2e8))
t2 = time.perf_counter()
for _ in range(200): dist.all_reduce(y)
t3 = time.perf_counter()
torch.cuda.synchronize()
import ctypes as C
from paper_2409_02423_b200 import _lib
codec = spec.c()
s = torch.cuda.current_stream().cuda_stream
torch.cuda._sleep(int(2e8))
t4 = time.perf_counter()
for _ in range(200): _lib.hccx_allreduce(comm.h, x.data_ptr(), out.data_ptr(), 1024, codec, 0, s)
t5 = time.perf_counter()
torch.cuda.synchronize()
if rank == 0:
    print(json.dumps({"p": p, "hccx_host_us_per_call": round((t1-t0)/200*1e6, 2), "nccl_host_us_per_call": round((t3-t2)/200*1e6, 2), "raw_ctypes_us": round((t5-t4)/200*1e6,2)}))
comm.close(); dist.destroy_process_group()
