"""Small driver for ncu: a few compress/decompress launches at the BASELINE
config-1 size (2^24 values, rate 8 by default)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_02423_b200 import _lib  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rate = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 24
codec = _lib.Codec(kind, rate)
w = C.c_uint64()
assert _lib.hccx_wire_size_bytes(codec, n, C.byref(w)) == 0
torch.cuda.set_device(0)
xs = [torch.randn(n, device="cuda") * 1e-3 for _ in range(3)]
ps = [torch.empty(w.value, dtype=torch.uint8, device="cuda") for _ in range(3)]
ys = [torch.empty(n, device="cuda") for _ in range(3)]
s = torch.cuda.current_stream().cuda_stream
for i in range(6):
    assert _lib.hccx_compress(codec, xs[i % 3].data_ptr(), n, ps[i % 3].data_ptr(), None, s) == 0
    assert _lib.hccx_decompress(codec, ps[i % 3].data_ptr(), w.value, n, ys[i % 3].data_ptr(), s) == 0
torch.cuda.synchronize()
print("ok", n, rate)
