"""NVLink traffic of the compressed allreduce, measured by the hardware:
NVML NVLink counters (field values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX
and COUNT_XMIT/RCV_BYTES, summed over the GPU's links) read before and after
K allreduces on every rank, against the wire bytes the engine claims
(2(p-1)W per rank for the ring) -- and the same for NCCL's
uncompressed allreduce.  Run under torchrun; rank 0 prints one JSON line per
case with every rank's measured bytes per call.

  torchrun --nproc-per-node N tools/nvlink_bytes.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import CodecSpec  # noqa: E402
from paper_2409_02423_b200 import dist as D  # noqa: E402
from paper_2409_02423_b200.codec import wire_size_bytes  # noqa: E402

import pynvml as N  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, p = dist.get_rank(), dist.get_world_size()
N.nvmlInit()
vis = os.environ.get("CUDA_VISIBLE_DEVICES")
h = N.nvmlDeviceGetHandleByIndex(int(vis.split(",")[local]) if vis else local)
# NVML NVLink counters: throughput (KiB) and byte counters, per link (scope
# = link index), summed over the links that answer
FIELDS = {"data_tx": (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 1024),
          "data_rx": (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024),
          "raw_tx": (N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, 1024),
          "raw_rx": (N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX, 1024),
          "xmit_bytes": (N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, 1),
          "rcv_bytes": (N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1)}
LINKS = 18
STATUS = {}


def counters():
    out = {}
    for name, (fid, _unit) in FIELDS.items():
        total, ok = 0, 0
        try:
            vals = N.nvmlDeviceGetFieldValues(h, [(fid, link) for link in range(LINKS)])
            for v in vals:
                STATUS.setdefault(name, set()).add(int(v.nvmlReturn))
                if v.nvmlReturn == 0:
                    total += int(v.value.ullVal)
                    ok += 1
        except Exception as e:  # noqa: BLE001
            STATUS.setdefault(name, set()).add(str(e)[:40])
        out[name] = total if ok else None
    return out


n = int(os.environ.get("NB_N", str(1 << 26)))
n -= n % (64 * p)
K = int(os.environ.get("NB_K", "20"))
comm = D.NvlinkComm(n)
x = torch.randn(n, device="cuda") * 1e-3
out = torch.empty_like(x)
os.environ["HCCX_ONESHOT_BYTES"] = "0"  # the ring at every size


def measure(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    a = counters()
    for _ in range(K):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    b = counters()
    per = {}
    for k, (_fid, unit) in FIELDS.items():
        if isinstance(a[k], int) and isinstance(b[k], int):
            per[k + "_bytes_per_call"] = round((b[k] - a[k]) * unit / K)
    per["nvml_status"] = {k: sorted(str(x) for x in v) for k, v in STATUS.items()}
    return per


rows = []
for rate in (8, 4, 16):
    spec = CodecSpec.fixed_rate(rate)
    c = n // p
    W = wire_size_bytes(spec, c)
    m = measure(lambda: comm.allreduce(x, spec, 0, out))
    rows.append({"case": f"hccx allreduce r{rate}", "claimed_wire_bytes_per_rank": 2 * (p - 1) * W, **m})
y = x.clone()
m = measure(lambda: dist.all_reduce(y))
rows.append({"case": "nccl allreduce (uncompressed)", "ring_bytes_per_rank_2(p-1)/p*4n": 2 * (p - 1) * 4 * n // p, **m})
gathered = [None] * p
dist.all_gather_object(gathered, rows)
if rank == 0:
    for i, r in enumerate(rows):
        print(json.dumps({"p": p, "n_values_per_rank": n, "case": r["case"],
                          "claimed": {k: v for k, v in r.items() if k.startswith(("claimed", "ring"))},
                          "per_rank": [{k: v for k, v in g[i].items() if k.endswith("per_call") or k == "nvml_status"}
                                       for g in gathered]}), flush=True)
comm.close()
dist.destroy_process_group()
