"""The p = 8 ring (north_star's rank count) on whatever box this is: one
single-process communicator with 8 members spread over the GPUs (two per GPU
on a 4-GPU box: neighbours alternate between virtual ranks of one launch and
NVLink peers).  Times the 256 MiB-per-rank r8 allreduce (device time, events
on member 0's device after every device synchronised) and checks sampled
blocks against the CPU oracle.  NOT an 8xB200 number: two ranks share each
GPU's HBM and SMs.

  python tools/p8_on_box.py [values_per_rank] [reps]
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2409_02423_b200 import _lib  # noqa: E402
import oracle_lib as O  # noqa: E402  (checker)

p = 8
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n -= n % (64 * p)
g = torch.cuda.device_count()
devices = [j * g // p for j in range(p)]
h = C.c_void_p()
assert _lib.hccx_mcomm_create(p, (C.c_int * p)(*devices), n, C.byref(h)) == 0
xs, ys = [], []
for j in range(p):
    gen = torch.Generator(device=f"cuda:{devices[j]}").manual_seed(11 + j)
    xs.append(torch.randn(n, device=f"cuda:{devices[j]}", generator=gen) * 1e-3)
    ys.append(torch.empty(n, device=f"cuda:{devices[j]}"))
pin, _k1 = _lib.ptr_array([x.data_ptr() for x in xs])
pout, _k2 = _lib.ptr_array([y.data_ptr() for y in ys])
codec = _lib.Codec(2, 8)


def sync_all():
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)


for _ in range(2):
    assert _lib.hccx_mcomm_allreduce(h, pin, pout, n, codec, 0, None) == 0
sync_all()
times = []
for _ in range(reps):
    sync_all()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(devices[0]):
        a.record()
    assert _lib.hccx_mcomm_allreduce(h, pin, pout, n, codec, 0, None) == 0
    sync_all()
    with torch.cuda.device(devices[0]):
        b.record()
    b.synchronize()
    times.append(a.elapsed_time(b))
assert _lib.hccx_mcomm_status(h, None) == 0
# sampled parity: 64 blocks per chunk, the oracle allreduce of those blocks
c = n // p
rng = np.random.default_rng(3)
idx = np.concatenate([k * c + 64 * rng.choice(c // 64, 8, replace=False) for k in range(p)])
cols = (idx[:, None] + np.arange(64)[None, :]).reshape(-1)
xin = np.stack([x[torch.from_numpy(cols).to(x.device)].cpu().numpy() for x in xs])
want, _ = O.allreduce(xin, "fixed-rate", 8, False)
got = np.stack([y[torch.from_numpy(cols).to(y.device)].cpu().numpy() for y in ys])
ok = all(got[j].tobytes() == want[j].tobytes() for j in range(p))
ms = sorted(times)[len(times) // 2]
print(json.dumps({"p": p, "devices": devices, "values_per_rank": n, "rate": 8, "ms": round(ms, 4),
                  "GBps_per_rank": round(4 * n / (ms * 1e-3) / 1e9, 1), "sampled_bit_exact": ok,
                  "note": "two ranks per GPU: shared HBM/SMs, not an 8xB200 number"}))
_lib.hccx_mcomm_destroy(h)
