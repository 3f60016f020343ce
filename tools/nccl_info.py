"""NCCL's own record of the uncompressed baseline: communicator init lines
and the algorithm / protocol it picks for the 256 MiB fp32 allreduce of
BASELINE config 2 (NCCL_DEBUG=INFO, SUBSYS INIT,TUNING,NVLS), plus its
algbw.  Run under torchrun; rank 0 prints one summary line.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_info.py
"""
import os

os.environ["NCCL_DEBUG"] = "INFO"  # the image exports NCCL_DEBUG=VERSION
os.environ["NCCL_DEBUG_SUBSYS"] = "INIT,TUNING,NVLS,GRAPH"
os.environ["NCCL_DEBUG_FILE"] = f"/tmp/nccl_info.{os.environ.get('RANK', '0')}.log"

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, world = dist.get_rank(), dist.get_world_size()
n = 1 << 26
y = torch.ones(n, device="cuda")
for _ in range(5):
    dist.all_reduce(y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    dist.all_reduce(y)
b.record()
torch.cuda.synchronize()
ms = torch.tensor([a.elapsed_time(b) / 20], device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
dist.destroy_process_group()
if rank == 0:
    with open(os.environ["NCCL_DEBUG_FILE"], errors="replace") as f:
        lines = [ln.rstrip() for ln in f]
    out = os.environ.get("NCCL_INFO_OUT", "gpurun_out/nccl_info.txt")
    with open(out, "w") as f:
        f.write(f"# NCCL allreduce 256 MiB fp32, p={world}: {ms.item():.4f} ms = "
                f"{4 * n / (ms.item() * 1e-3) / 1e9:.1f} GB/s algbw\n")
        f.write("\n".join(lines) + "\n")
    print(f"nccl p={world}: {ms.item():.4f} ms, log -> {out}")
