"""The NVLink engine's fused allreduce as virtual ranks on ONE GPU
(hccx_mcomm with every member on cuda:0): a single-process, single-launch
form of ring_fused_kernel that ncu can replay.  Per-CTA work (phases,
segments, codec bodies, pushes, flags) is the multi-GPU kernel's; the p ranks
share one GPU's HBM and SMs (148 / p CTAs each), so absolute times differ
from one rank per GPU.

  python tools/fused_virtual.py [p] [values_per_rank] [reps]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 24)
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rate = int(os.environ.get("FV_RATE", "8"))
os.environ.setdefault("HCCX_ONESHOT_BYTES", "0")
n -= n % (64 * p)
h = C.c_void_p()
devs = (C.c_int * p)(*([0] * p))
assert _lib.hccx_mcomm_create(p, devs, n, C.byref(h)) == 0
g = torch.Generator(device="cuda").manual_seed(5)
xs = [torch.randn(n, device="cuda", generator=g) * 1e-3 for _ in range(p)]
ys = [torch.empty_like(x) for x in xs]
a, _ka = _lib.ptr_array([x.data_ptr() for x in xs])
b, _kb = _lib.ptr_array([y.data_ptr() for y in ys])
codec = _lib.Codec(2, rate)
for _ in range(reps):
    assert _lib.hccx_mcomm_allreduce(h.value, a, b, n, codec, 0, None) == 0
assert _lib.hccx_mcomm_status(h.value, None) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(torch.cuda.default_stream())
for _ in range(reps):
    assert _lib.hccx_mcomm_allreduce(h.value, a, b, n, codec, 0, None) == 0
e1.record(torch.cuda.default_stream())
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"virtual allreduce p={p} n={n}/rank r{rate}: {ms:.4f} ms per call ({4 * n * p / (ms * 1e-3) / 1e9:.1f} GB/s "
      f"of member buffers)")
_lib.hccx_mcomm_destroy(h.value)
