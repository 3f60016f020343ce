"""One ZFP-mode compress + decompress at 2^24 r8 after two warm-up pairs (an
ncu target: --launch-skip 4 --launch-count 2 on the step kernels)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
rate = int(os.environ.get("ZFP_RATE", "8"))
n = 1 << 24
codec = _lib.Codec(3, rate)
w = C.c_uint64()
_lib.hccx_wire_size_bytes(codec, n, C.byref(w))
x = torch.randn(n, device="cuda") * 1e-3
p = torch.empty(w.value, dtype=torch.uint8, device="cuda")
y = torch.empty(n, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    assert _lib.hccx_compress(codec, x.data_ptr(), n, p.data_ptr(), None, s) == 0
    assert _lib.hccx_decompress(codec, p.data_ptr(), w.value, n, y.data_ptr(), s) == 0
torch.cuda.synchronize()
print("ok")
