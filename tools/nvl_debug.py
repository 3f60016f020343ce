"""Debug driver for the NVLink engine: each op once, status after each."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, p = dist.get_rank(), dist.get_world_size()
comm = D.NvlinkComm(1 << 20)
print(f"rank {rank} connected", flush=True)
for spec in (CodecSpec.identity(), CodecSpec.fixed_rate(8)):
    for n_per in (64, 4096):
        x = torch.arange(n_per * p, dtype=torch.float32, device="cuda") * (rank + 1)
        for name, fn in [("ar", lambda: comm.allreduce(x, spec)), ("rs", lambda: comm.reduce_scatter(x, spec)),
                         ("ag", lambda: comm.allgather(x[:n_per].contiguous(), spec)),
                         ("bc", lambda: comm.broadcast(x, 0, spec)), ("pp", lambda: comm.p2p(x, 0, p - 1, spec))]:
            t0 = time.time()
            try:
                fn()
                comm.status()
                r = "ok"
            except Exception as e:
                r = f"ERR {e}"
            print(f"rank {rank} {spec} n_per={n_per} {name}: {r} ({time.time() - t0:.2f}s)", flush=True)
            dist.barrier()
comm.close()
dist.destroy_process_group()
