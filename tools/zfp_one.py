import ctypes as C, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2409_02423_b200 import _lib
torch.cuda.set_device(0)
n = 1 << 24
codec = _lib.Codec(3, 8)
w = C.c_uint64(); _lib.hccx_wire_size_bytes(codec, n, C.byref(w))
x = torch.randn(n, device="cuda") * 1e-3
p = torch.empty(w.value, dtype=torch.uint8, device="cuda")
y = torch.empty(n, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.hccx_compress(codec, x.data_ptr(), n, p.data_ptr(), None, s)
    _lib.hccx_decompress(codec, p.data_ptr(), w.value, n, y.data_ptr(), s)
torch.cuda.synchronize()
print("ok")
